import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_0907_1788_b200 import Codec, workload as W
codec = Codec(0)
for name in ["C5", "C2", "C4"]:
    cfg = W.CONFIGS[name]
    pats, sp = W.patterns(cfg)
    pp = torch.from_numpy(pats.astype(np.int32)).pin_memory()
    for i in range(6):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); s.record()
        p = codec.plans(cfg.k, cfg.n, pp)
        e.record(); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(name, i, f"gpu {s.elapsed_time(e):.3f} ms  host-call {1e3*(t1-t0):.3f} ms  total {1e3*(t2-t0):.3f} ms")
        p.close()
