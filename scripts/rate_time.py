"""Device timing of encode/decode for arbitrary (k, n) shapes (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
from paper_0907_1788_b200 import Codec, _lib, workload as W, default_escape_capacity

codec = Codec(0)
lib = _lib.load()


def t_ms(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for arg in sys.argv[1:]:
    k, n, L, S = (int(x) for x in arg.split(","))
    src = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
    lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
    out = torch.empty((S, n, L), dtype=torch.int16, device="cuda")
    cap = default_escape_capacity(out.numel())
    esc = torch.empty(cap, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    te = t_ms(lambda: codec.encode(k, n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
    rng = np.random.default_rng(1)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(16)]).astype(np.uint32)
    sp = (np.arange(S) % 16).astype(np.uint32)
    plans = codec.plans(k, n, pats)
    codec.encode(k, n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt)
    rx, rxe = W.received_packets(out, esc, cnt, pats, sp, n)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    dout = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
    td = t_ms(lambda: codec.decode(plans, spd, rx, rxe, out=dout, esc_out=esc, esc_cap=cap, count=cnt))
    ok = torch.equal(dout, src)
    gb = 2 * k * L * S / 1e9
    print(f"k={k} n={n} L={L} S={S}: encode {gb/te*1e3:.1f} GB/s | decode {gb/td*1e3:.1f} GB/s | ok={ok}", flush=True)
