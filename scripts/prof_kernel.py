import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
from paper_0907_1788_b200 import Codec, _lib, workload as W, default_escape_capacity
codec = Codec(0); lib = _lib.load()
name = sys.argv[1]; S = int(sys.argv[2]); what = sys.argv[3]
cfg = W.CONFIGS[name]
src = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
out = torch.empty((S, cfg.n, cfg.L), dtype=torch.int16, device="cuda")
cap = default_escape_capacity(out.numel()); esc = torch.empty(cap, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
sysm = what.startswith("sys")  # sysenc / sysdec: the systematic pair
for _ in range(2): codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt, systematic=sysm)
if what in ("dec", "sysdec"):
    pats, sp = W.patterns(cfg, stripes=S)
    plans = codec.plans(cfg.k, cfg.n, pats)
    rx, rxe = W.received_packets(out, esc, cnt, pats, sp, cfg.n)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    dout = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
    for _ in range(2): codec.decode(plans, spd, rx, rxe, out=dout, esc_out=esc, esc_cap=cap, count=cnt, systematic=sysm)
torch.cuda.synchronize(); print("ok")
