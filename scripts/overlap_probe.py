"""Does running independent encode and decode chunks concurrently (two
streams) beat running them back to back? (development probe)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0907_1788_b200 import Codec, _lib, default_escape_capacity, workload as W  # noqa: E402

codec = Codec(0)
lib = _lib.load()
cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
chunk = min(S, 8192)
k, n, L = cfg.k, cfg.n, cfg.L
src = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
lib.fntrs_gpu_fill_symbols(W.SEED, 0, src.numel(), C.c_void_p(src.data_ptr()), None)
enc = torch.empty((S, n, L), dtype=torch.int16, device="cuda")
cap = default_escape_capacity(chunk * n * L)
nch = S // chunk
ee = [torch.empty(cap, dtype=torch.int64, device="cuda") for _ in range(nch)]
ec = torch.zeros(nch, dtype=torch.int64, device="cuda")
for c in range(nch):
    codec.encode(k, n, src[c * chunk:(c + 1) * chunk], out=enc[c * chunk:(c + 1) * chunk], esc_out=ee[c], esc_cap=cap,
                 count=ec[c:c + 1])
pats, sp = W.patterns(cfg, stripes=S)
plans = codec.plans(k, n, pats)
rx = torch.empty((S, k, L), dtype=torch.int16, device="cuda")
rxe = []
for c in range(nch):
    a, b = c * chunk, (c + 1) * chunk
    r, e = W.received_packets(enc[a:b], ee[c], ec[c:c + 1], pats, sp[a:b], n)
    rx[a:b].copy_(r)
    rxe.append(e)
spd = torch.from_numpy(sp.astype(np.int32)).cuda()
dec = torch.empty((chunk, k, L), dtype=torch.int16, device="cuda")
dcap = default_escape_capacity(chunk * k * L)
de = torch.empty(dcap, dtype=torch.int64, device="cuda")
dc = torch.zeros(1, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def enc_all(st):
    for c in range(nch):
        codec.encode(k, n, src[c * chunk:(c + 1) * chunk], out=enc[c * chunk:(c + 1) * chunk], esc_out=ee[c],
                     esc_cap=cap, count=ec[c:c + 1], stream=st)


dec2 = torch.empty((chunk, k, L), dtype=torch.int16, device="cuda")
de2 = torch.empty(dcap, dtype=torch.int64, device="cuda")
dc2 = torch.zeros(1, dtype=torch.int64, device="cuda")


def dec_all(st):
    for c in range(nch):
        a, b = c * chunk, (c + 1) * chunk
        codec.decode(plans, spd[a:b], rx[a:b], rxe[c], out=dec2, esc_out=de2, esc_cap=dcap, count=dc2, stream=st)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def serial():
    enc_all(torch.cuda.current_stream())
    dec_all(torch.cuda.current_stream())


def overlapped():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        enc_all(s1)
    with torch.cuda.stream(s2):
        dec_all(s2)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    cur.wait_event(e1)
    cur.wait_event(e2)


te = timed(lambda: enc_all(torch.cuda.current_stream()))
td = timed(lambda: dec_all(torch.cuda.current_stream()))
ts = timed(serial)
to = timed(overlapped)
gb = 2 * k * L * S / 1e9
print(f"{cfg.name} S={S}: encode {te:.2f} ms, decode {td:.2f} ms, serial {ts:.2f} ms ({gb / ts * 1e3:.1f} GB/s), "
      f"overlapped {to:.2f} ms ({gb / to * 1e3:.1f} GB/s), gain {100 * (ts / to - 1):.1f} %")
