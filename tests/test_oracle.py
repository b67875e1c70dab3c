"""Pin the oracle (oracle/fntrs_oracle.c) before trusting it.

1. Every golden vector / known answer frozen in the reference's own unit
   tests for this path (file:line cited per case).
2. Agreement with the reference library itself (oracle/_ref, built from
   /root/reference/proj/src) on seeded random inputs, when it is built.
3. Agreement with the committed fixtures in tests/golden/ (made from the
   reference library by tests/golden/make_golden.py).
"""
import os

import numpy as np
import pytest

P = 65537


# ---------------------------------------------------------------- field ----
def test_field_golden(oracle):  # proj/tests/test_field.cpp:13-111
    o = oracle
    assert o.add(0, 123) == 123 and o.add(65536, 1) == 0
    assert o.add(40000, 40000) == 14463 and o.add(65536, 65536) == 65535
    assert o.sub(5, 7) == 65535 and o.sub(0, 65536) == 1 and o.sub(123, 123) == 0
    assert o.mul(1, 999) == 999 and o.mul(65536, 65536) == 1 and o.mul(256, 256) == 65536
    assert o.mul(65536, 2) == 65535 and o.mul(0, 65536) == 0
    for a, b, want in [(65343, 18073, 32836), (38415, 7635, 20450), (39801, 35634, 48154),
                       (39767, 19995, 46281), (50749, 2163, 61149), (58208, 41206, 61259)]:
        assert o.mul(a, b) == want
    assert o.pow(3, 65536) == 1 and o.pow(3, 32768) == 65536 and o.pow(7, 0) == 1 and o.pow(0, 5) == 0
    assert o.pow(12345, 67890) == 17777 and o.pow(65536, 3) == 65536 and o.pow(40000, 65535) == 10694
    for a, want in [(1, 1), (2, 32769), (65536, 65536), (3, 21846), (12345, 31651), (65535, 32768)]:
        assert o.inv(a) == want
    assert o.root(1) == (0, 1) and o.root(2) == (0, 65536) and o.root(4) == (0, 65281)
    assert o.root(8) == (0, 4096) and o.root(65536) == (0, 3)
    assert o.root(0)[0] == 3 and o.root(3)[0] == 3 and o.root(131072)[0] == 3  # InvalidTransformSize
    # survey values r_16 = 64, r_32 = 65529, r_256 = 282, r_2048 = 61869, r_4096 = 54449, r_16384 = 81
    for n, r in [(16, 64), (32, 65529), (256, 282), (2048, 61869), (4096, 54449), (16384, 81)]:
        assert o.root(n) == (0, r)
    rng = np.random.default_rng(1)
    a = rng.integers(0, P, 3000)
    b = rng.integers(0, P, 3000)
    for x, y in zip(a, b):
        assert o.mul(int(x), int(y)) == (int(x) * int(y)) % P
        assert o.add(int(x), int(y)) == (int(x) + int(y)) % P
        assert o.sub(int(x), int(y)) == (int(x) - int(y)) % P


# ------------------------------------------------------------ transform ----
def test_transform_golden(oracle):  # proj/tests/test_transform.cpp:42-71
    o = oracle
    assert list(o.fnt([1, 2])) == [3, 65536]
    assert list(o.fnt([3, 65536], inverse=True)) == [1, 2]
    assert list(o.fnt([9, 0, 0, 0])) == [9, 9, 9, 9]
    assert list(o.fnt([0, 1, 0, 0])) == [1, 65281, 65536, 256]
    want = [36, 50109, 1020, 48061, 65533, 17468, 64509, 15420]
    assert list(o.fnt(list(range(1, 9)))) == want
    assert list(o.fnt(want, inverse=True)) == list(range(1, 9))
    assert list(o.naive_dft(1, [42])) == [42]
    assert list(o.naive_dft(65536, [1, 2])) == [3, 65536]


def test_transform_vs_naive_and_roundtrip(oracle):  # test_transform.cpp:73-95
    rng = np.random.default_rng(2)
    for e in range(0, 11):
        n = 1 << e
        a = rng.integers(0, P, n).astype(np.uint32)
        r = oracle.root(n)[1]
        assert np.array_equal(oracle.fnt(a), oracle.naive_dft(r, a))
        assert np.array_equal(oracle.fnt(a, True), oracle.naive_dft(r, a, True))
    for e in range(0, 17):
        n = 1 << e
        a = rng.integers(0, P, n).astype(np.uint32)
        assert np.array_equal(oracle.fnt(oracle.fnt(a), True), a)


def test_geom_step5_equivalence(oracle):  # test_geom.cpp:74-82: negative direction = reversed list
    # geom_eval(a) on the size-8 chirp equals fnt_forward for a full-size polynomial
    a = [11, 22, 33, 44, 55, 66, 77, 88]
    assert list(oracle.fnt(a)) == [396, 26903, 11220, 4375, 65493, 61074, 54229, 38546]


# ----------------------------------------------------------------- plan ----
def test_plan_golden(oracle):  # proj/tests/test_interp.cpp:41-70
    st, a, ap, ps, af = oracle.build_plan(2, [0, 1])
    assert st == 0 and list(a) == [65536, 0, 1] and list(ap) == [32769, 32768]
    st, a, ap, ps, af = oracle.build_plan(4, [0])
    assert st == 0 and list(a) == [65536, 1] and list(ap) == [1]
    st, a, ap, ps, af = oracle.build_plan(8, [0, 2, 5])
    assert st == 0 and list(a) == [16, 61169, 4351, 1]
    assert list(ap) == [oracle.inv(4337), oracle.inv(61712), oracle.inv(3600)]
    # validation (test_interp.cpp:72-82)
    assert oracle.build_plan(8, [1, 3, 1])[0] == 7   # DuplicatePosition
    assert oracle.build_plan(8, [1, 8])[0] == 8      # PositionOutOfRange
    assert oracle.build_plan(12, [1])[0] == 3        # InvalidTransformSize


def test_interpolate_golden(oracle):  # test_interp.cpp:83-100
    assert list(oracle.interpolate(8, [3], [321])[1]) == [321]
    assert list(oracle.interpolate(4, [0, 2], [12, 65535])[1]) == [5, 7]
    assert list(oracle.interpolate(8, [0, 2, 5], [1000, 2000, 3000])[1]) == [46905, 62038, 23131]
    st, out = oracle.lagrange([1, 65536], [12, 65535])
    assert st == 0 and list(out) == [5, 7]


# ---------------------------------------------------------------- codec ----
def test_codec_golden(oracle):  # proj/tests/test_codec.cpp:60-112
    nd = __import__("ctypes").c_uint32()
    assert oracle.lib.orc_code_params(3, 6, nd) == 0 and nd.value == 8
    assert oracle.lib.orc_code_params(0, 4, nd) == 4 and oracle.lib.orc_code_params(5, 4, nd) == 4
    assert oracle.lib.orc_code_params(1, 65537, nd) == 4
    assert list(oracle.encode(1, 5, [77])[1]) == [77] * 5
    assert list(oracle.encode(2, 4, [5, 7])[1]) == [12, 63750, 65535, 1797]
    assert list(oracle.decode(2, 4, [0, 2], [12, 65535])[1]) == [5, 7]
    assert oracle.decode(2, 4, [0], [1])[0] == 10        # NotEnoughSymbols
    assert oracle.decode(2, 4, [1, 1], [5, 6])[0] == 7   # DuplicatePosition
    assert oracle.decode(2, 4, [0, 4], [5, 6])[0] == 8   # PositionOutOfRange


def _subsets(n, s):
    from itertools import combinations
    return combinations(range(n), s)


def test_codec_mds_exhaustive(oracle):  # test_codec.cpp:192-224; acceptance.cpp:85-132
    rng = np.random.default_rng(3)
    for n, k in [(4, 2), (8, 4), (8, 5), (16, 12)]:
        src = rng.integers(0, P, k).astype(np.uint32)
        enc = oracle.encode(k, n, src)[1]
        count = 0
        for s in range(k, n + 1):
            for keep in _subsets(n, s):
                keep = np.array(keep, dtype=np.uint32)
                st, got = oracle.decode(k, n, keep, enc[keep])
                assert st == 0 and np.array_equal(got, src), (n, k, keep)
                count += 1
        from math import comb
        assert count == sum(comb(n, s) for s in range(k, n + 1))


def test_codec_k_lowest_and_top_value(oracle):  # test_codec.cpp:238-247, 333-339
    rng = np.random.default_rng(19)
    src = rng.integers(0, P, 3).astype(np.uint32)
    enc = oracle.encode(3, 9, src)[1].copy()
    enc[8] = (enc[8] + 1) % P
    keep = np.array([1, 3, 5, 8], dtype=np.uint32)
    assert np.array_equal(oracle.decode(3, 9, keep, enc[keep])[1], src)
    src = np.array([65536, 65536, 65536], dtype=np.uint32)
    enc = oracle.encode(3, 7, src)[1]
    keep = np.array([2, 4, 6], dtype=np.uint32)
    assert np.array_equal(oracle.decode(3, 7, keep, enc[keep])[1], src)


def test_escape_rule(oracle):  # proj/tests/test_shardio.cpp:70-87
    v = np.array([5, 65536, 7], dtype=np.uint32)
    words = np.zeros(3, dtype=np.uint16)
    esc = np.zeros(3, dtype=np.uint32)
    ne = oracle.lib.orc_escape_split(v, 3, words, esc)
    assert ne == 1 and list(words) == [5, 0, 7] and list(esc[:1]) == [1]


def test_randomized_fast_equals_lagrange(oracle):  # acceptance.cpp:134-191 (scaled: 150 instances)
    rng = np.random.default_rng(4)
    for _ in range(150):
        n = int(rng.integers(2, 257))
        k = int(rng.integers(1, n + 1))
        src = rng.integers(0, P, k).astype(np.uint32)
        enc = oracle.encode(k, n, src)[1]
        keep = np.sort(rng.choice(n, size=int(rng.integers(k, n + 1)), replace=False)).astype(np.uint32)
        st, got = oracle.decode(k, n, keep, enc[keep])
        assert st == 0 and np.array_equal(got, src)
        nd = 1 << (n - 1).bit_length()
        r = oracle.root(nd)[1]
        xs = [oracle.pow(r, int(z)) for z in keep[:k]]
        st, lag = oracle.lagrange(xs, enc[keep[:k]])
        if not (n == nd and keep.size == n):
            assert np.array_equal(lag, src)


def test_batched_stripes_roundtrip(oracle):
    from paper_0907_1788_b200 import workload as W
    from oracle_bind import gather_received
    k, n, L, S = 8, 16, 6, 3
    src = W.symbols(W.SEED, 0, S * k * L).reshape(S, k, L)
    enc, esc = oracle.encode_stripes(k, n, src)
    pats = np.stack([np.sort(np.random.default_rng(s).choice(n, k, replace=False)) for s in range(S)]).astype(np.uint32)
    sp = np.arange(S, dtype=np.uint32)
    rx, rx_esc = gather_received(enc, esc, pats, sp)
    dec, desc = oracle.decode_stripes(k, n, pats, sp, rx, rx_esc)
    assert np.array_equal(dec, src) and desc.size == 0


# ------------------------------------------------------- systematic ----
def test_systematic_golden(oracle):  # proj/tests/test_codec.cpp:112-136,164-190
    assert list(oracle.encode_systematic(2, 4, [5, 7])[1]) == [5, 7, 65032, 65030]
    assert list(oracle.encode_systematic(4, 8, [100, 200, 300, 400])[1]) == [
        100, 200, 300, 400, 33256, 17912, 53593, 3200]
    assert list(oracle.encode_systematic(1, 6, [9])[1]) == [9] * 6
    rng = np.random.default_rng(100)
    for k, n in [(1, 6), (2, 4), (4, 8), (5, 13), (300, 700)]:
        src = rng.integers(0, P, k).astype(np.uint32)
        st, enc = oracle.encode_systematic(k, n, src)
        assert st == 0 and enc.size == n and np.array_equal(enc[:k], src)
    src = np.array([100, 200, 300, 400], dtype=np.uint32)
    enc = oracle.encode_systematic(4, 8, src)[1]
    for keep in ([0, 1, 2, 3, 6], [2, 3, 4, 5, 6, 7]):
        keep = np.array(keep, dtype=np.uint32)
        st, got = oracle.decode_systematic(4, 8, keep, enc[keep])
        assert st == 0 and np.array_equal(got, src)
    assert oracle.encode_systematic(3, 2, [1, 2, 3])[0] == 4  # SizeMismatch
    assert oracle.decode_systematic(2, 4, [0], [1])[0] == 10  # NotEnoughSymbols


def test_systematic_matches_reference_library(oracle, ref):  # codec.cpp:151-196
    rng = np.random.default_rng(17)
    for _ in range(60):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, n + 1))
        src = rng.integers(0, P, k).astype(np.uint32)
        so, eo = oracle.encode_systematic(k, n, src)
        sr, er = ref.encode_systematic(k, n, src)
        assert so == sr == 0 and np.array_equal(eo, er[:n]), (k, n)
        cnt = int(rng.integers(k, n + 1))
        pos = rng.choice(n, cnt, replace=False).astype(np.uint32)
        vals = rng.integers(0, P, cnt).astype(np.uint32)  # arbitrary values: k-lowest rule and prefix shortcut
        do, dr = oracle.decode_systematic(k, n, pos, vals), ref.decode_systematic(k, n, pos, vals)
        assert do[0] == dr[0] == 0 and np.array_equal(do[1], dr[1][:k]), (k, n)
        got = oracle.decode_systematic(k, n, pos, eo[pos])[1]
        assert np.array_equal(got, src)
    for args in [(2, 4, [0], [1]), (2, 4, [1, 1], [5, 6]), (2, 4, [0, 4], [5, 6])]:
        assert oracle.decode_systematic(*args)[0] == ref.decode_systematic(*args)[0]


# -------------------------------------------------- oracle vs reference ----
def test_oracle_matches_reference_library(oracle, ref):
    rng = np.random.default_rng(5)
    for e in range(0, 13):
        n = 1 << e
        a = rng.integers(0, P, n).astype(np.uint32)
        assert np.array_equal(oracle.fnt(a), ref.fnt(a)[1])
        assert np.array_equal(oracle.fnt(a, True), ref.fnt(a, True)[1])
    for n, k in [(8, 3), (64, 32), (256, 128), (1024, 512), (2048, 1024), (4096, 2048), (100, 37)]:
        nd = 1 << (n - 1).bit_length()
        pos = np.sort(rng.choice(n, k, replace=False)).astype(np.uint32)
        ro = oracle.build_plan(nd, pos)
        rr = ref.build_plan(nd, pos)
        assert ro[0] == rr[0] == 0
        assert np.array_equal(ro[1], rr[1]) and np.array_equal(ro[2], rr[2])
        assert ro[3] == rr[3] and np.array_equal(ro[4], rr[4])
        src = rng.integers(0, P, k).astype(np.uint32)
        eo, er = oracle.encode(k, n, src)[1], ref.encode(k, n, src)[1]
        assert np.array_equal(eo, er)
        vals = rng.integers(0, P, k).astype(np.uint32)  # arbitrary received values, not a codeword
        assert np.array_equal(oracle.decode(k, n, pos, vals)[1], ref.decode(k, n, pos, vals, path=1)[1])
    # error classes agree
    for args in [(2, 4, [0], [1]), (2, 4, [1, 1], [5, 6]), (2, 4, [0, 4], [5, 6])]:
        assert oracle.decode(*args)[0] == ref.decode(*args)[0]


def test_mul_low_split_matches_reference(oracle, ref):  # interp.cpp:133-134, poly.cpp:139-169
    """2k > 65536: no product transform fits, the reference splits the product."""
    rng = np.random.default_rng(33)
    for n, k in [(65536, 32769), (40000, 33000)]:
        pos = np.sort(rng.choice(n, k, replace=False)).astype(np.uint32)
        vals = rng.integers(0, P, k).astype(np.uint32)  # arbitrary received values
        so, go = oracle.decode(k, n, pos, vals)
        sr, gr = ref.decode(k, n, pos, vals, path=1)
        assert so == sr == 0 and np.array_equal(go, gr[:k])
        assert ref.build_plan(1 << (n - 1).bit_length(), pos)[3] == 0  # product_size 0


def test_oracle_matches_reference_stripes(oracle, ref):
    from paper_0907_1788_b200 import workload as W
    from oracle_bind import gather_received
    k, n, L, S = 64, 128, 16, 2
    src = W.symbols(123, 0, S * k * L).reshape(S, k, L)
    eo, esco = oracle.encode_stripes(k, n, src)
    er, escr = ref.encode_stripes(k, n, src, threads=2)
    assert np.array_equal(eo, er) and np.array_equal(esco, escr)
    pats = np.stack([np.sort(np.random.default_rng(7 + s).choice(n, k, replace=False)) for s in range(S)]).astype(np.uint32)
    sp = np.arange(S, dtype=np.uint32)
    rx, rxe = gather_received(eo, esco, pats, sp)
    do, deo = oracle.decode_stripes(k, n, pats, sp, rx, rxe)
    dr, der = ref.decode_stripes(k, n, pats, sp, rx, rxe, path=0, threads=2)
    assert np.array_equal(do, dr) and np.array_equal(deo, der) and np.array_equal(do, src)


# ------------------------------------------------------------- fixtures ----
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="fixtures not generated")
def test_oracle_matches_golden_fixtures(oracle):
    g = np.load(GOLDEN)
    for name in sorted({k.split("__")[0] for k in g.files}):
        kind, n, k = name.split("_")[0], int(name.split("_")[1]), int(name.split("_")[2])
        if kind == "enc":
            assert np.array_equal(oracle.encode(k, n, g[name + "__src"])[1], g[name + "__out"]), name
        elif kind == "dec":
            st, out = oracle.decode(k, n, g[name + "__pos"], g[name + "__val"])
            assert st == 0 and np.array_equal(out, g[name + "__out"]), name
        elif kind == "plan":
            st, a, ap, ps, af = oracle.build_plan(n, g[name + "__pos"])
            assert np.array_equal(a, g[name + "__a"]) and np.array_equal(ap, g[name + "__ap"])
            assert np.array_equal(af, g[name + "__afnt"]), name
        elif kind == "senc":
            assert np.array_equal(oracle.encode_systematic(k, n, g[name + "__src"])[1], g[name + "__out"]), name
        elif kind == "sdec":
            st, out = oracle.decode_systematic(k, n, g[name + "__pos"], g[name + "__val"])
            assert st == 0 and np.array_equal(out, g[name + "__out"]), name
        else:
            raise AssertionError(name)


# ------------------------------------------- systematic convolution form ----
@pytest.mark.parametrize("k,n,seed", [(4, 8, 1), (8, 16, 2), (5, 16, 3), (16, 32, 4), (3, 13, 5), (32, 64, 6)])
def test_systematic_convolution_identity(oracle, k, n, seed):
    """The identity the fused systematic kernels (codec_dec.cu MODE 3 / 4) compute:
    P(r^j) = A(r^j) r^-j (c (*) G')[j] with c[z] = v_z / A'(r^z) on the k lowest
    received positions and G'[e] = 1 / (1 - r^-e), G'[0] = 0 (cyclic, size N),
    checked against the oracle's encode_systematic / decode_systematic, i.e.
    interpolate + re-evaluate (proj/src/codec.cpp:151-196)."""
    o = oracle
    N = 1
    while N < n:
        N <<= 1
    st, r = o.root(N)
    assert st == 0
    rng = np.random.default_rng(seed)
    src = rng.integers(0, 65537, k).astype(np.uint32)
    st, cw = o.encode_systematic(k, n, src)
    assert st == 0

    def conv_eval(pos, vals):
        xs = [pow(r, int(z), P) for z in pos]
        def A(x):
            a = 1
            for xi in xs:
                a = a * (x - xi) % P
            return a
        c = np.zeros(N, dtype=np.uint32)
        for z, v, xi in zip(pos, vals, xs):
            d = 1
            for xl in xs:
                if xl != xi:
                    d = d * (xi - xl) % P
            c[z] = int(v) * pow(d, P - 2, P) % P
        g = np.array([0] + [pow((1 - pow(r, N - e, P)) % P, P - 2, P) for e in range(1, N)], dtype=np.uint32)
        ch, gh = o.fnt(c), o.fnt(g)
        h = o.fnt(np.array([int(a) * int(b) % P for a, b in zip(ch, gh)], dtype=np.uint32), inverse=True)
        return [A(pow(r, j, P)) * pow(r, (N - j) % N, P) % P * int(h[j]) % P for j in range(N)]

    # encode: parity rows k..n-1 from the source at positions 0..k-1
    ev = conv_eval(list(range(k)), src)
    assert [int(x) for x in cw[k:]] == ev[k:n]
    # decode: erased rows < k from the k lowest of a random received subset
    recv = np.sort(rng.choice(n, size=min(n, k + 2), replace=False))
    use = recv[:k]
    st, want = o.decode_systematic(k, n, recv, cw[recv])
    assert st == 0 and np.array_equal(want, cw[:k])
    ev = conv_eval(list(use), cw[use])
    got = [int(cw[j]) if j in set(use.tolist()) else ev[j] for j in range(k)]
    assert got == [int(x) for x in want]
