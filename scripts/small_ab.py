import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
from paper_0907_1788_b200 import Codec, _lib, workload as W, default_escape_capacity
codec = Codec(0); lib = _lib.load()
def t_ms(fn, reps=50):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for (k, n, L, S) in [(1024, 2048, 512, 1), (2048, 4096, 1024, 1), (128, 256, 2048, 1), (1024, 2048, 512, 8)]:
    src = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
    lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
    rng = np.random.default_rng(1)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(S)]).astype(np.uint32)
    sp = torch.arange(S, dtype=torch.int32, device="cuda")
    for fast in (1, 0):
        lib.fntrs_gpu_set_fast_path(codec.ctx, fast)
        out, oe, cnt = codec.encode(k, n, src)
        te = t_ms(lambda: codec.encode(k, n, src, out=out, esc_out=oe, count=cnt))
        plans = codec.plans(k, n, pats)
        rx, rxe = W.received_packets(out, oe, cnt, pats, np.arange(S, dtype=np.uint32), n)
        dec, de, dc = codec.decode(plans, sp, rx, rxe)
        td = t_ms(lambda: codec.decode(plans, sp, rx, rxe, out=dec, esc_out=de, count=dc))
        print(f"k={k} n={n} L={L} S={S} fast={fast}: encode {te*1e3:.1f} us decode {td*1e3:.1f} us ok={torch.equal(dec, src)}")
