"""A/B of the streamed (one persistent launch, L2 rings) vs batched four-step
kernels: identical outputs, device times (development aid).
  python scripts/stream_ab.py C4:256 C3:1 [R,D ...]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0907_1788_b200 import Codec, _lib, default_escape_capacity, escapes_to_numpy, workload as W  # noqa: E402

codec = Codec(0)
lib = _lib.load()


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


specs = [a for a in sys.argv[1:] if ":" in a]
rds = [a for a in sys.argv[1:] if "," in a] or [None]
for spec in specs:
    name, S = spec.split(":")
    S = int(S)
    cfg = W.CONFIGS[name]
    src = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
    lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
    cap = default_escape_capacity(S * cfg.n * cfg.L)
    pats, sp = W.patterns(cfg, stripes=S)
    plans = codec.plans(cfg.k, cfg.n, pats)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    gb = 2 * cfg.k * cfg.L * S / 1e9
    ref = None
    for mode, rd in [("batched", None)] + [("stream", r) for r in rds]:
        os.environ["FNTRS_STREAM"] = "0" if mode == "batched" else "1"
        if rd:
            os.environ["FNTRS_STREAM_RD"] = rd
        else:
            os.environ.pop("FNTRS_STREAM_RD", None)
        out = torch.empty((S, cfg.n, cfg.L), dtype=torch.int16, device="cuda")
        esc = torch.empty(cap, dtype=torch.int64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        te = t_ms(lambda: codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
        enc_esc = escapes_to_numpy(esc, cnt)
        rx, rxe = W.received_packets(out, esc, cnt, pats, sp, cfg.n)
        dout = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
        desc = torch.empty(cap, dtype=torch.int64, device="cuda")
        dcnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        td = t_ms(lambda: codec.decode(plans, spd, rx, rxe, out=dout, esc_out=desc, esc_cap=cap, count=dcnt))
        ok = torch.equal(dout, src)
        if ref is None:
            ref = (out.clone(), enc_esc)
            same = True
        else:
            same = torch.equal(out, ref[0]) and np.array_equal(enc_esc, ref[1])
        print(f"{name} S={S} {mode:8s} R,D={rd or 'default'}: encode {te:8.3f} ms = {gb / te * 1e3:7.1f} GB/s | "
              f"decode {td:8.3f} ms = {gb / td * 1e3:7.1f} GB/s | roundtrip={ok} same_as_batched={same} "
              f"esc={len(enc_esc)}", flush=True)
        del out, esc, rx, dout
        torch.cuda.empty_cache()
