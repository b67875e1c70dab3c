"""Development probe: does encode throughput depend on the footprint or on the
run length?  Times one config's encode (a) on S stripes in one call, (b) as
S/c calls of c stripes over the same buffers, (c) c stripes repeated S/c times
on one buffer.  Usage: python scripts/enc_probe.py C5 2048 256"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import subprocess

import torch

from paper_0907_1788_b200 import Codec, _lib, default_escape_capacity, workload as W

name, S, c = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = W.CONFIGS[name]
codec = Codec(0)
lib = _lib.load()
src = torch.empty((S, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
out = torch.empty((S, cfg.n, cfg.L), dtype=torch.int16, device="cuda")
cap = default_escape_capacity(out.numel())
esc = torch.empty(cap, dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


gb = 2 * cfg.k * cfg.L * S / 1e9
t = timed(lambda: codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
print(f"{name} one call S={S}: {t:.2f} ms = {gb / t * 1e3:.1f} GB/s escapes={int(cnt.item())}", flush=True)


def chunks():
    for i in range(0, S, c):
        codec.encode(cfg.k, cfg.n, src[i:i + c], out=out[i:i + c], esc_out=esc, esc_cap=cap, count=cnt)


t = timed(chunks)
print(f"{name} {S // c} calls of {c}: {t:.2f} ms = {gb / t * 1e3:.1f} GB/s", flush=True)


def same():
    for i in range(0, S, c):
        codec.encode(cfg.k, cfg.n, src[:c], out=out[:c], esc_out=esc, esc_cap=cap, count=cnt)


t = timed(same)
print(f"{name} {S // c} calls of {c} on one buffer: {t:.2f} ms = {gb / t * 1e3:.1f} GB/s", flush=True)
# zero source: no escapes at all
src.zero_()
t = timed(lambda: codec.encode(cfg.k, cfg.n, src, out=out, esc_out=esc, esc_cap=cap, count=cnt))
print(f"{name} zero source S={S}: {t:.2f} ms = {gb / t * 1e3:.1f} GB/s escapes={int(cnt.item())}", flush=True)
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                      "--format=csv"], capture_output=True, text=True).stdout)
