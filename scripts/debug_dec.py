import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
from oracle_bind import Oracle, gather_received
from paper_0907_1788_b200 import Codec, workload as W, escapes_to_numpy
orc = Oracle(); codec = Codec(0)
for (k, n, L, S) in [(128, 256, 64, 40)]:
    src = W.symbols(W.SEED, 0, S * k * L).reshape(S, k, L)
    out, oe, cnt = codec.encode(k, n, torch.from_numpy(src.view(np.int16)).cuda())
    torch.cuda.synchronize()
    ge = escapes_to_numpy(oe, cnt)
    want, we = orc.encode_stripes(k, n, src)
    print("enc data eq", np.array_equal(out.cpu().numpy().view(np.uint16), want), "esc got", ge[:10], "want", we[:10], int(cnt.item()))
for (k, n, L, S) in [(2, 4, 8, 1), (4, 8, 8, 1), (8, 16, 16, 1), (128, 256, 64, 1), (128, 256, 64, 2)]:
    src = W.symbols(W.SEED, 0, S * k * L).reshape(S, k, L)
    enc, esc = orc.encode_stripes(k, n, src)
    rng = np.random.default_rng(1)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(S)]).astype(np.uint32)
    sp = np.arange(S, dtype=np.uint32)
    rx, rxe = gather_received(enc, esc, pats, sp)
    plans = codec.plans(k, n, pats)
    a, ap, ps, af = plans.export(0)
    st, oa, oap, ops, oaf = orc.build_plan(1 << (n-1).bit_length(), pats[0])
    print("plan eq", np.array_equal(a, oa), np.array_equal(ap, oap), np.array_equal(af, oaf))
    dec, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), torch.from_numpy(rx.view(np.int16)).cuda(), None)
    got = dec.cpu().numpy().view(np.uint16)
    bad = np.argwhere(got != src)
    print(k, n, L, S, "dec mismatches", len(bad), bad[:5].tolist(), "esc", int(dc.item()))
    if len(bad) and n <= 16:
        print("pats", pats[0], "src col0", src[0, :, 0], "got", got[0, :, 0])
