import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from oracle_bind import Oracle
from paper_0907_1788_b200 import Codec, workload as W
orc = Oracle(); codec = Codec(0)
for (k, n, L, S) in [(2, 4, 8, 1), (4, 8, 8, 1), (8, 16, 16, 1), (128, 256, 64, 1), (128, 256, 64, 2)]:
    src = W.symbols(W.SEED, 0, S * k * L).reshape(S, k, L)
    out, oe, cnt = codec.encode(k, n, torch.from_numpy(src.view(np.int16)).cuda())
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint16)
    want, _ = orc.encode_stripes(k, n, src)
    bad = np.argwhere(got != want)
    print(k, n, L, S, "mismatches", len(bad), bad[:5].tolist())
    if len(bad) and n <= 16:
        print("src col0", src[0, :, 0]); print("got col0", got[0, :, 0]); print("want col0", want[0, :, 0])
        x = np.zeros((n, 1), dtype=np.uint32); x[:k, 0] = src[0, :, 0]
        f = codec.fnt(torch.from_numpy(np.pad(x, ((0, 0), (0, 0))).view(np.int32)).cuda()).cpu().numpy().view(np.uint32)
        print("fnt col0", f[:, 0])
