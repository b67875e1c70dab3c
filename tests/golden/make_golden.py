"""Generate tests/golden/reference_vectors.npz from the reference library
itself (oracle/_ref/libfntrs_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Each case is seeded; arrays are uint32. Kinds:
  enc_{n}_{k}   codec::encode_nonsystematic        src -> out
  dec_{n}_{k}   codec::decode_nonsystematic (Fast)  pos, val (arbitrary values) -> out
  senc_{n}_{k}  codec::encode_systematic            src -> out
  sdec_{n}_{k}  codec::decode_systematic            pos, val -> out
  plan_{n}_{k}  interp::build_plan                  pos -> a, ap (1/A'(x_i)), afnt (bit-reversed)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bind import RefLib  # noqa: E402

P = 65537
SHAPES = [(8, 3), (16, 5), (64, 32), (100, 37), (256, 128), (300, 200), (1000, 600), (2048, 1024), (4096, 2048),
          (4096, 700)]


def main():
    assert RefLib.available(), "build oracle/_ref first (make -C oracle ref)"
    ref = RefLib()
    rng = np.random.default_rng(0x0907_1788)
    out = {}
    for n, k in SHAPES:
        nd = 1 << (n - 1).bit_length()
        src = rng.integers(0, P, k).astype(np.uint32)
        src[rng.integers(0, k)] = 65536
        st, enc = ref.encode(k, n, src)
        assert st == 0
        out[f"enc_{n}_{k}__src"], out[f"enc_{n}_{k}__out"] = src, enc[:n]
        pos = np.sort(rng.choice(n, k, replace=False)).astype(np.uint32)
        val = rng.integers(0, P, k).astype(np.uint32)
        st, dec = ref.decode(k, n, pos, val, path=1)
        assert st == 0
        out[f"dec_{n}_{k}__pos"], out[f"dec_{n}_{k}__val"], out[f"dec_{n}_{k}__out"] = pos, val, dec[:k]
        st, senc = ref.encode_systematic(k, n, src)
        assert st == 0
        out[f"senc_{n}_{k}__src"], out[f"senc_{n}_{k}__out"] = src, senc[:n]
        st, sdec = ref.decode_systematic(k, n, pos, val)
        assert st == 0
        out[f"sdec_{n}_{k}__pos"], out[f"sdec_{n}_{k}__val"], out[f"sdec_{n}_{k}__out"] = pos, val, sdec[:k]
        st, a, ap, ps, af = ref.build_plan(nd, pos)
        assert st == 0
        out[f"plan_{nd}_{k}__pos"], out[f"plan_{nd}_{k}__a"] = pos, a.astype(np.uint32)
        out[f"plan_{nd}_{k}__ap"], out[f"plan_{nd}_{k}__afnt"] = ap.astype(np.uint32), af.astype(np.uint32)
    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
