"""GPU parity of the systematic codec (proj/src/codec.cpp:151-196) against the
oracle restatement (oracle/fntrs_oracle.c: orc_encode_systematic /
orc_decode_systematic, itself pinned to the reference library and the
reference's frozen examples in tests/test_oracle.py). Bit-exact everywhere.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = 65537


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0907_1788_b200 import Codec
    return Codec(0)


def dev_u16(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).cuda()


def dev_esc(e):
    if e is None or len(e) == 0:
        return None
    return torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint64).view(np.int64)).cuda()


def split(vals):
    """uint32 field values -> uint16 words + ascending escape indices."""
    flat = vals.reshape(-1)
    esc = np.nonzero(flat == 65536)[0].astype(np.uint64)
    return np.where(vals == 65536, 0, vals).astype(np.uint16), esc


def joined(out, oe, cnt):
    from paper_0907_1788_b200 import escapes_to_numpy
    v = out.cpu().numpy().view(np.uint16).astype(np.uint32)
    e = escapes_to_numpy(oe, cnt).astype(np.int64)
    v.reshape(-1)[e] = 65536
    return v


def source(S, k, L, seed):
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 65536, (S, k, L)).astype(np.uint32)
    idx = rng.choice(v.size, size=min(3, v.size), replace=False)
    v.reshape(-1)[idx] = 65536  # the top field value travels as an escape
    return v


def columns(S, L, seed, limit=12):
    cells = [(s, c) for s in range(S) for c in range(L)]
    if len(cells) <= limit:
        return cells
    rng = np.random.default_rng(seed)
    return [cells[i] for i in rng.choice(len(cells), limit, replace=False)]


SYS_SHAPES = [  # (k, n, L, stripes): general kernels, fused N <= 4096 kernels, four-step N >= 8192
    (1, 6, 8, 2), (2, 4, 16, 3), (4, 8, 8, 2), (5, 13, 7, 2), (300, 700, 8, 1), (8, 8, 16, 2),
    (64, 128, 64, 3), (128, 256, 64, 4), (100, 256, 32, 2), (1024, 2048, 64, 1), (2048, 4096, 32, 1),
    (700, 2048, 32, 1), (4096, 8192, 64, 1), (8192, 16384, 64, 1),
    # many tiles per persistent CTA (fused MODE 1 / 2 at n_domain 256 and 4096)
    (128, 256, 64, 1200), (2048, 4096, 16, 200),
    # fused conv-form kernels (MODE 3 / 4) at every n_domain 32..1024, HALFK and not
    (16, 32, 32, 3), (10, 32, 32, 3), (20, 64, 32, 3), (32, 64, 64, 2), (40, 128, 32, 2),
    (256, 512, 32, 2), (200, 512, 32, 2), (512, 1024, 16, 2), (300, 1024, 16, 2),
]


@pytest.mark.parametrize("k,n,L,S", SYS_SHAPES)
def test_encode_systematic_matches_oracle(codec, oracle, k, n, L, S):
    src = source(S, k, L, seed=k * 7 + n)
    w, e = split(src)
    out, oe, cnt = codec.encode_systematic(k, n, dev_u16(w), dev_esc(e))
    got = joined(out, oe, cnt)
    assert got.shape == (S, n, L)
    assert np.array_equal(got[:, :k, :], src)  # the source rows, verbatim
    for s, c in columns(S, L, seed=n):
        st, want = oracle.encode_systematic(k, n, src[s, :, c])
        assert st == 0 and np.array_equal(got[s, :, c], want), (s, c)


def _patterns(S, n, k, seed):
    rng = np.random.default_rng(seed)
    pats = [np.arange(k)]  # stripe 0: the systematic prefix (reference's verbatim-copy case)
    pats += [np.sort(rng.choice(n, k, replace=False)) for _ in range(1, S)]
    if S > 2:  # stripe 1: parity only (no row < k received; every output row is computed)
        pats[1] = np.arange(n - k, n)
    return np.stack(pats).astype(np.uint32), np.arange(S, dtype=np.uint32)


@pytest.mark.parametrize("k,n,L,S", SYS_SHAPES)
def test_decode_systematic_matches_oracle(codec, oracle, k, n, L, S):
    src = source(S, k, L, seed=k + 3 * n)
    w, e = split(src)
    out, oe, cnt = codec.encode_systematic(k, n, dev_u16(w), dev_esc(e))
    enc = joined(out, oe, cnt)
    pats, sp = _patterns(max(S, 2), n, k, seed=n + 1)
    pats, sp = pats[:S], sp[:S]
    plans = codec.plans(k, n, pats)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    rx = np.stack([enc[s][pats[sp[s]]] for s in range(S)])  # [S, k, L]
    rw, re = split(rx)
    dec, de, dc = codec.decode_systematic(plans, spd, dev_u16(rw), dev_esc(re))
    assert np.array_equal(joined(dec, de, dc), src)
    # arbitrary received values (not codewords): the oracle's k-lowest interpolation
    rng = np.random.default_rng(k)
    junk = rng.integers(0, P, rx.shape).astype(np.uint32)
    jw, je = split(junk)
    dec, de, dc = codec.decode_systematic(plans, spd, dev_u16(jw), dev_esc(je))
    got = joined(dec, de, dc)
    for s, c in columns(S, L, seed=k + 1):
        st, want = oracle.decode_systematic(k, n, pats[sp[s]], junk[s, :, c])
        assert st == 0 and np.array_equal(got[s, :, c], want), (s, c)


def test_systematic_reference_interface(codec):  # proj/tests/test_codec.cpp:112-190
    import paper_0907_1788_b200 as F
    from paper_0907_1788_b200 import CodeParams, Symbol
    assert F.encode_systematic(CodeParams.make(2, 4), [5, 7]) == [5, 7, 65032, 65030]
    assert F.encode_systematic(CodeParams.make(4, 8), [100, 200, 300, 400]) == [
        100, 200, 300, 400, 33256, 17912, 53593, 3200]
    assert F.encode_systematic(CodeParams.make(1, 6), [9]) == [9] * 6
    p = CodeParams.make(4, 8)
    enc = F.encode_systematic(p, [100, 200, 300, 400])
    take = lambda keep: [Symbol(i, enc[i]) for i in keep]
    assert F.decode_systematic(p, take([0, 1, 2, 3, 6])) == [100, 200, 300, 400]
    assert F.decode_systematic(p, take([7, 2, 5, 3, 6, 4])) == [100, 200, 300, 400]
    with pytest.raises(F.NotEnoughSymbols):
        F.decode_systematic(p, take([1, 2, 3]))
    top = F.encode_systematic(CodeParams.make(3, 7), [65536] * 3)
    assert F.decode_systematic(CodeParams.make(3, 7), [Symbol(i, top[i]) for i in (2, 4, 6)]) == [65536] * 3
