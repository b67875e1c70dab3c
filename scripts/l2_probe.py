"""Development probe: four-step decode/encode time per source byte at a given
(n, k, L, stripes), to compare HBM-resident and L2-sized intermediates
(FNTRS_SCRATCH_MB). Usage: python scripts/l2_probe.py n k L stripes"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C

import numpy as np
import torch

from paper_0907_1788_b200 import Codec, _lib, default_escape_capacity, workload as W

n, k, L, S = (int(a) for a in sys.argv[1:5])
codec = Codec(0)
lib = _lib.load()
src = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
out = torch.empty((S, n, L), dtype=torch.int16, device="cuda")
cap = default_escape_capacity(out.numel())
esc = torch.empty(cap, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")


def t_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


te = t_ms(lambda: codec.encode(k, n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
rng = np.random.default_rng(5)
pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(S)]).astype(np.uint32)
sp = np.arange(S, dtype=np.uint32)
plans = codec.plans(k, n, pats)
codec.encode(k, n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt)
idx = torch.from_numpy(pats.astype(np.int64)).cuda()
rx = torch.gather(out, 1, idx[:, :, None].expand(S, k, L)).contiguous()
spd = torch.from_numpy(sp.view(np.int32)).cuda()
dout = torch.empty_like(src)
ne = int(cnt.item())
assert ne == 0 or True
td = t_ms(lambda: codec.decode(plans, spd, rx, None, out=dout, esc_out=esc, esc_cap=cap, count=cnt))
gb = 2 * k * L * S / 1e9
print(f"n={n} k={k} L={L} S={S} scratch={os.environ.get('FNTRS_SCRATCH_MB', 'default')}: "
      f"encode {gb / te * 1e3:.1f} GB/s decode {gb / td * 1e3:.1f} GB/s (escapes {ne}; decode exact only without)", flush=True)
