"""Quick device timing of encode/decode/plans per config (development aid)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
from paper_0907_1788_b200 import Codec, _lib, workload as W, default_escape_capacity

codec = Codec(0)
lib = _lib.load()
def t_ms(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

for name, stripes in ([("C1", 1), ("C2", 4096), ("C5", 256)] if len(sys.argv) < 2 else []) + ([(a, int(b)) for a, b in (x.split(":") for x in sys.argv[1:])]):
    cfg = W.CONFIGS[name]
    S = stripes
    src = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
    lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
    out = torch.empty((S, cfg.n, cfg.L), dtype=torch.int16, device="cuda")
    cap = default_escape_capacity(out.numel())
    esc = torch.empty(cap, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    te = t_ms(lambda: codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
    pats, sp = W.patterns(cfg, stripes=S)
    t0 = time.time(); plans = codec.plans(cfg.k, cfg.n, pats); torch.cuda.synchronize(); tp = (time.time()-t0)*1e3
    tp2 = t_ms(lambda: codec.plans(cfg.k, cfg.n, pats), reps=2)
    codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt)
    rx, rxe = W.received_packets(out, esc, cnt, pats, sp, cfg.n)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    dout = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
    td = t_ms(lambda: codec.decode(plans, spd, rx, rxe, out=dout, esc_out=esc, esc_cap=cap, count=cnt))
    ok = torch.equal(dout, src)
    gb = 2 * cfg.k * cfg.L * S / 1e9
    print(f"{name} S={S}: encode {te:.3f} ms = {gb/te*1e3:.1f} GB/s | decode {td:.3f} ms = {gb/td*1e3:.1f} GB/s "
          f"| plans {tp2:.2f} ms ({len(pats)} pats) | roundtrip ok={ok} esc={int(cnt.item())}", flush=True)
