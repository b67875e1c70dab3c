"""GPU parity: the CUDA path (through the C ABI) against the oracle / reference.

Bit-exact equality is the bar everywhere (integer arithmetic). Sizes are
chosen so the CPU checkers finish in seconds; full-size configs are covered
by size-independent properties (decode(encode(s)) == s, linearity).
"""
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = 65537
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0907_1788_b200 import Codec
    return Codec(0)


def dev_u16(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.int16)).cuda()


def host_u16(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16)


def dev_esc(e: np.ndarray):
    if e is None or len(e) == 0:
        return None
    return torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint64).view(np.int64)).cuda()


def source_with_escapes(S, k, L, seed, n_esc):
    from paper_0907_1788_b200 import workload as W
    src = W.symbols(seed, 0, S * k * L).reshape(S, k, L)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(S * k * L, size=min(n_esc, S * k * L), replace=False)).astype(np.uint64)
    flat = src.reshape(-1)
    flat[idx.astype(np.int64)] = 0
    return src, idx


# -------------------------------------------------------------- transform ----
@pytest.mark.parametrize("e", list(range(0, 13)))
def test_fnt_matches_oracle(codec, oracle, e):
    m = 1 << e
    rng = np.random.default_rng(e)
    for L in (1, 3, 40):
        x = rng.integers(0, P, (m, L)).astype(np.uint32)
        x[0, 0] = 65536
        t = torch.from_numpy(x.view(np.int32)).cuda()
        fw = codec.fnt(t).cpu().numpy().view(np.uint32)
        iv = codec.fnt(t, inverse=True).cpu().numpy().view(np.uint32)
        for c in range(L):
            assert np.array_equal(fw[:, c], oracle.fnt(x[:, c])), (m, L, c)
            assert np.array_equal(iv[:, c], oracle.fnt(x[:, c], True)), (m, L, c)


# -------------------------------------------------------------- per-codeword API ----
def test_reference_interface_golden(codec):  # proj/tests/test_codec.cpp:60-112
    import paper_0907_1788_b200 as F
    p = F.CodeParams.make(3, 6)
    assert (p.k, p.n, p.n_domain) == (3, 6, 8)
    for bad in [(0, 4), (5, 4), (1, 65537)]:
        with pytest.raises(F.SizeMismatch):
            F.CodeParams.make(*bad)
    assert F.encode_nonsystematic(F.CodeParams.make(1, 5, False), [77]) == [77] * 5
    p24 = F.CodeParams.make(2, 4, False)
    assert F.encode_nonsystematic(p24, [5, 7]) == [12, 63750, 65535, 1797]
    with pytest.raises(F.SizeMismatch):
        F.encode_nonsystematic(p24, [1])
    assert F.decode_nonsystematic(p24, [F.Symbol(0, 12), F.Symbol(2, 65535)]) == [5, 7]
    assert F.decode_nonsystematic(p24, [F.Symbol(0, 12), F.Symbol(2, 65535)], F.Path.Fast) == [5, 7]
    with pytest.raises(F.NotEnoughSymbols):
        F.decode_nonsystematic(p24, [F.Symbol(0, 1)])
    with pytest.raises(F.DuplicatePosition):
        F.decode_nonsystematic(p24, [F.Symbol(1, 5), F.Symbol(1, 6)])
    with pytest.raises(F.PositionOutOfRange):
        F.decode_nonsystematic(p24, [F.Symbol(0, 5), F.Symbol(4, 6)])
    p8 = F.CodeParams.make(8, 8, False)
    assert F.encode_nonsystematic(p8, list(range(1, 9))) == [36, 50109, 1020, 48061, 65533, 17468, 64509, 15420]
    src = [65536, 65536, 65536]
    p37 = F.CodeParams.make(3, 7, False)
    enc = F.encode_nonsystematic(p37, src)
    assert F.decode_nonsystematic(p37, [F.Symbol(z, enc[z]) for z in (2, 4, 6)]) == src


def test_reference_interface_mds(codec):  # test_codec.cpp:192-224
    import itertools
    import paper_0907_1788_b200 as F
    rng = np.random.default_rng(9)
    for n, k in [(4, 2), (8, 4), (8, 5)]:
        p = F.CodeParams.make(k, n, False)
        src = [int(x) for x in rng.integers(0, P, k)]
        enc = F.encode_nonsystematic(p, src)
        for s in range(k, n + 1):
            for keep in itertools.combinations(range(n), s):
                assert F.decode_nonsystematic(p, [F.Symbol(z, enc[z]) for z in keep]) == src, (n, k, keep)


def test_cpp_dropin_suite():
    exe = os.path.join(ROOT, "build", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "cpptest"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


# ---------------------------------------------------------------- batched ----
SHAPES = [  # (k, n, L, stripes)
    (1, 1, 8, 2), (1, 5, 3, 2), (2, 4, 16, 3), (3, 8, 5, 2), (5, 11, 7, 2), (12, 16, 32, 2),
    (64, 128, 64, 3), (128, 256, 64, 4), (100, 256, 24, 2), (200, 256, 16, 2),
    (512, 1024, 32, 2), (1024, 2048, 512, 1), (2048, 4096, 64, 1), (1000, 4000, 16, 1),
    # fused v2 kernels (n_domain 32..4096, L a multiple of the tile width), incl. k != n/2
    (16, 32, 64, 3), (100, 256, 64, 2), (50, 256, 64, 1), (300, 512, 64, 2), (1500, 4096, 16, 1),
    (700, 2048, 32, 1), (512, 1000, 64, 1),
    # four-step kernels (n_domain 8192..65536, L a multiple of 64)
    (4096, 8192, 64, 2), (8192, 16384, 64, 2), (16384, 32768, 64, 1), (32768, 65536, 64, 1),
    (5000, 12000, 64, 1), (3000, 8192, 128, 1),
    # general column path (codec_cols.cu): product size M != n_domain above 4096, any L
    (3000, 4096, 16, 1), (2000, 16384, 8, 1), (1000, 8192, 10, 2), (4096, 8192, 40, 1), (5000, 9000, 8, 1),
    (20000, 32768, 8, 1), (40, 10000, 16, 1),
    # fused M != n_domain decode (codec_gen.cu): k > N/2 and k <= N/4 at N <= 4096
    (200, 256, 64, 3), (20, 256, 32, 2), (12, 256, 32, 2), (600, 1024, 32, 1), (100, 1024, 32, 1),
    (700, 4096, 16, 1), (20, 32, 32, 2), (5, 32, 32, 2), (2, 32, 32, 2), (3000, 3500, 16, 1),
    # 2k > 65536: the product by halves (reference poly::mul_low)
    (33000, 65536, 8, 1), (40000, 50000, 4, 2),
]


@pytest.mark.parametrize("k,n,L,S", SHAPES)
def test_encode_matches_oracle(codec, oracle, k, n, L, S):
    src, esc = source_with_escapes(S, k, L, seed=k * 7 + n, n_esc=3)
    want, want_esc = oracle.encode_stripes(k, n, src, esc)
    out, oe, cnt = codec.encode(k, n, dev_u16(src), dev_esc(esc))
    from paper_0907_1788_b200 import escapes_to_numpy
    assert np.array_equal(host_u16(out), want)
    assert np.array_equal(escapes_to_numpy(oe, cnt), want_esc)


def _patterns(S, n, k, seed):
    rng = np.random.default_rng(seed)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(S)]).astype(np.uint32)
    return pats, np.arange(S, dtype=np.uint32)


@pytest.mark.parametrize("k,n,L,S", SHAPES)
def test_decode_matches_oracle(codec, oracle, k, n, L, S):
    from oracle_bind import gather_received
    from paper_0907_1788_b200 import escapes_to_numpy
    src, esc = source_with_escapes(S, k, L, seed=k + n, n_esc=2)
    enc, enc_esc = oracle.encode_stripes(k, n, src, esc)
    pats, sp = _patterns(S, n, k, seed=n)
    # arbitrary (non-codeword) received values too: tamper with one stripe's payload
    rx, rx_esc = gather_received(enc, enc_esc, pats, sp)
    rx = rx.copy()
    rx[-1, 0, 0] ^= 0x5A5A
    rx_esc = rx_esc[rx_esc != np.uint64(((S - 1) * k) * L)]
    want, want_esc = oracle.decode_stripes(k, n, pats, sp, rx, rx_esc)
    plans = codec.plans(k, n, pats)
    spd = torch.from_numpy(sp.view(np.int32)).cuda()
    out, oe, cnt = codec.decode(plans, spd, dev_u16(rx), dev_esc(rx_esc))
    assert np.array_equal(host_u16(out), want)
    assert np.array_equal(escapes_to_numpy(oe, cnt), want_esc)


@pytest.mark.parametrize("n,k", [(2, 2), (4, 2), (8, 3), (8, 5), (16, 12), (256, 128), (2048, 1024), (4096, 2048),
                                 (1000, 300), (200, 100), (64, 17), (16384, 8192), (12000, 5000),
                                 (65536, 33000), (16384, 2000), (8192, 5000)])
def test_plan_fields_match_oracle(codec, oracle, n, k):
    nd = 1 << (n - 1).bit_length()
    rng = np.random.default_rng(n + k)
    pos = np.sort(rng.choice(n, k, replace=False)).astype(np.uint32)
    st, a, ap, ps, af = oracle.build_plan(nd, pos)
    plans = codec.plans(k, n, pos[None, :])
    ga, gap, gps, gaf = plans.export(0)
    assert gps == ps
    assert np.array_equal(ga, a) and np.array_equal(gap, ap) and np.array_equal(gaf, af)


@pytest.mark.parametrize("m", [1 << e for e in range(13, 17)])
def test_fnt_large_matches_oracle(codec, oracle, m):
    rng = np.random.default_rng(m)
    L = 3
    x = rng.integers(0, P, (m, L)).astype(np.uint32)
    t = torch.from_numpy(x.view(np.int32)).cuda()
    fw = codec.fnt(t).cpu().numpy().view(np.uint32)
    iv = codec.fnt(t, inverse=True).cpu().numpy().view(np.uint32)
    for c in range(L):
        assert np.array_equal(fw[:, c], oracle.fnt(x[:, c]))
        assert np.array_equal(iv[:, c], oracle.fnt(x[:, c], True))


def test_frozen_plan_three_positions(codec):  # test_interp.cpp:52-63
    plans = codec.plans(3, 8, np.array([[0, 2, 5]], dtype=np.uint32))
    a, ap, ps, af = plans.export(0)
    inv = lambda x: pow(x, P - 2, P)
    assert list(a) == [16, 61169, 4351, 1]
    assert list(ap) == [inv(4337), inv(61712), inv(3600)]


def test_complete_reception_is_inverse_transform(codec, oracle):  # codec.cpp:137-144
    from paper_0907_1788_b200 import escapes_to_numpy
    n, k, L = 16, 5, 8
    rng = np.random.default_rng(11)
    vals = rng.integers(0, 65536, (1, n, L)).astype(np.uint16)  # not a codeword
    plans = codec.plans(k, n, np.arange(n, dtype=np.uint32)[None, :])
    out, oe, cnt = codec.decode(plans, torch.zeros(1, dtype=torch.int32, device="cuda"), dev_u16(vals))
    got = host_u16(out)
    want_esc = []
    for c in range(L):
        want = oracle.fnt(vals[0, :, c].astype(np.uint32), inverse=True)[:k]
        assert np.array_equal(got[0, :, c], np.where(want == 65536, 0, want))
        want_esc += [f * L + c for f in range(k) if want[f] == 65536]
    assert np.array_equal(escapes_to_numpy(oe, cnt), np.sort(np.array(want_esc, dtype=np.uint64)))


def test_complete_reception_large_domain(codec, oracle):  # codec.cpp:137-144 at n_domain 8192 (column path)
    from paper_0907_1788_b200 import escapes_to_numpy
    n, k, L = 8192, 100, 3
    rng = np.random.default_rng(12)
    vals = rng.integers(0, 65536, (1, n, L)).astype(np.uint16)  # not a codeword
    perm = rng.permutation(n).astype(np.uint32)  # positions in any order
    plans = codec.plans(k, n, perm[None, :])
    out, oe, cnt = codec.decode(plans, torch.zeros(1, dtype=torch.int32, device="cuda"), dev_u16(vals[:, perm, :]))
    got = host_u16(out)
    want_esc = []
    for c in range(L):
        want = oracle.fnt(vals[0, :, c].astype(np.uint32), inverse=True)[:k]
        assert np.array_equal(got[0, :, c], np.where(want == 65536, 0, want))
        want_esc += [f * L + c for f in range(k) if want[f] == 65536]
    assert np.array_equal(escapes_to_numpy(oe, cnt), np.sort(np.array(want_esc, dtype=np.uint64)))


@pytest.mark.parametrize("k,n,L,S", [(128, 256, 128, 3), (1024, 2048, 64, 1), (2048, 4096, 32, 1), (300, 512, 64, 1),
                                     (200, 256, 64, 2), (50, 256, 64, 2), (600, 1024, 32, 1),
                                     # many tiles per persistent CTA (counter-claimed tiles, TMA prefetch of
                                     # the next tile, mbarrier phases) in every fused family: n_domain 256
                                     # k = n/2 and k != n/2, M = 2N and M < N, n_domain 4096 at one CTA per SM
                                     (128, 256, 64, 1200), (100, 256, 64, 1600), (200, 256, 64, 1200),
                                     (50, 256, 64, 1200), (2048, 4096, 16, 200), (1500, 4096, 16, 200)])
def test_fast_kernels_match_general_kernels(codec, k, n, L, S):
    """A/B: the fused v2 kernels and the general tile kernels agree bit for bit."""
    from paper_0907_1788_b200 import _lib, escapes_to_numpy, workload as W
    lib = _lib.load()
    src, esc = source_with_escapes(S, k, L, seed=5 * k + n, n_esc=4)
    pats, sp = _patterns(S, n, k, seed=k)
    res = []
    for fast in (1, 0):
        assert lib.fntrs_gpu_set_fast_path(codec.ctx, fast) == 0
        out, oe, cnt = codec.encode(k, n, dev_u16(src), dev_esc(esc))
        enc_esc = escapes_to_numpy(oe, cnt)
        rx, rxe = W.received_packets(out, torch.from_numpy(enc_esc.view(np.int64)).cuda() if enc_esc.size else oe,
                                     cnt, pats, sp, n)
        plans = codec.plans(k, n, pats)
        dec, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), rx, rxe)
        res.append((host_u16(out), enc_esc, host_u16(dec), escapes_to_numpy(de, dc)))
    lib.fntrs_gpu_set_fast_path(codec.ctx, 1)
    for a, b in zip(res[0], res[1]):
        assert np.array_equal(a, b)
    assert np.array_equal(res[0][2], src)


def test_errors_map_to_reference_classes(codec):
    import paper_0907_1788_b200 as F
    with pytest.raises(F.PositionOutOfRange):
        codec.plans(2, 4, np.array([[0, 4]], dtype=np.uint32))
    with pytest.raises(F.DuplicatePosition):
        codec.plans(2, 4, np.array([[1, 1]], dtype=np.uint32))
    with pytest.raises(F.NotEnoughSymbols):
        codec.plans(3, 4, np.array([[1, 2]], dtype=np.uint32))
    with pytest.raises(F.SizeMismatch):
        codec.encode(0, 4, torch.zeros((1, 0, 8), dtype=torch.int16, device="cuda"))


# ---------------------------------------------------- configs, full size ----
def test_config_c1_bit_exact_vs_reference(codec, oracle):
    """C1 (n=2048, k=1024, L=512, 1 stripe) in full against the reference library."""
    from oracle_bind import RefLib, gather_received
    from paper_0907_1788_b200 import escapes_to_numpy, workload as W
    cfg = W.CONFIGS["C1"]
    src = W.symbols(W.SEED, 0, cfg.stripes * cfg.k * cfg.L).reshape(cfg.stripes, cfg.k, cfg.L)
    chk = RefLib() if RefLib.available() else oracle
    want, want_esc = chk.encode_stripes(cfg.k, cfg.n, src) if isinstance(chk, RefLib) else oracle.encode_stripes(cfg.k, cfg.n, src)
    out, oe, cnt = codec.encode(cfg.k, cfg.n, dev_u16(src))
    assert np.array_equal(host_u16(out), want)
    assert np.array_equal(escapes_to_numpy(oe, cnt), want_esc)
    pats, sp = W.patterns(cfg)
    rx, rxe = gather_received(want, want_esc, pats, sp)
    plans = codec.plans(cfg.k, cfg.n, pats)
    dec, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), dev_u16(rx), dev_esc(rxe))
    assert np.array_equal(host_u16(dec), src)
    assert escapes_to_numpy(de, dc).size == 0


@pytest.mark.parametrize("name,stripes", [("C2", 512), ("C5", 16), ("C3", 1), ("C4", 6)])
def test_config_roundtrip_sampled(codec, oracle, name, stripes):
    """decode(encode(s)) == s on device for a sample of the config's stripes, plus
    bit-exact encode against the oracle on the first two stripes."""
    from oracle_bind import gather_received
    from paper_0907_1788_b200 import escapes_to_numpy, workload as W
    cfg = W.CONFIGS[name]
    src = W.symbols(W.SEED, 0, stripes * cfg.k * cfg.L).reshape(stripes, cfg.k, cfg.L)
    out, oe, cnt = codec.encode(cfg.k, cfg.n, dev_u16(src))
    enc = host_u16(out)
    enc_esc = escapes_to_numpy(oe, cnt)
    # bit-exact against the oracle on the first stripe(s), a column sample for the long codes
    ns = min(2, stripes)
    cols = slice(0, cfg.L) if cfg.n <= 4096 else slice(0, 64)
    sub = np.ascontiguousarray(src[:ns, :, cols])
    want, want_esc = oracle.encode_stripes(cfg.k, cfg.n, sub)
    assert np.array_equal(enc[:ns, :, cols], want)
    Lc = sub.shape[2]
    got_esc = [e for e in enc_esc if e < ns * cfg.n * cfg.L and (e % cfg.L) < Lc]
    want_esc_full = [int(e // Lc) * cfg.L + int(e % Lc) for e in want_esc]
    assert [int(e) for e in got_esc] == want_esc_full
    pats, sp = W.patterns(cfg, stripes=stripes)
    rx, rxe = gather_received(enc, enc_esc, pats, sp)
    plans = codec.plans(cfg.k, cfg.n, pats)
    dec, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), dev_u16(rx), dev_esc(rxe))
    got = host_u16(dec)
    assert np.array_equal(got, src)
    # decode bit-exact against the oracle on a column sample of the first stripe, from the same input
    rx0 = np.ascontiguousarray(rx[:1, :, :16])
    e0 = [int(e // cfg.L) * 16 + int(e % cfg.L) for e in rxe if e < cfg.k * cfg.L and e % cfg.L < 16]
    want_dec, _ = oracle.decode_stripes(cfg.k, cfg.n, pats, sp[:1], rx0, np.array(e0, dtype=np.uint64))
    assert np.array_equal(got[:1, :, :16], want_dec)


def test_device_generator_matches_numpy(codec):
    import ctypes as C
    from paper_0907_1788_b200 import _lib, workload as W
    t = torch.empty(100003, dtype=torch.int16, device="cuda")
    st = _lib.load().fntrs_gpu_fill_symbols(W.SEED, 12345, t.numel(), C.c_void_p(t.data_ptr()),
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    assert np.array_equal(host_u16(t), W.symbols(W.SEED, 12345, t.numel()))


def test_host_pipeline_multistream_matches_single_stream(codec):
    """Concurrent calls on several streams (HostPipeline) give the same packets and
    escape lists as one call on one stream (no shared scratch between streams)."""
    from paper_0907_1788_b200 import escapes_to_numpy, workload as W
    from paper_0907_1788_b200.pipeline import HostPipeline, escape_ranges
    k, n, L, S, chunk = 128, 256, 256, 48, 8
    src = W.symbols(77, 0, S * k * L).reshape(S, k, L)
    # many escapes: 65536 sources produce many 65536 outputs
    src[:, 0, :] = 0
    esc = np.sort(np.array([(s * k) * L + c for s in range(S) for c in range(L)], dtype=np.uint64))
    whole, we, wc = codec.encode(k, n, dev_u16(src), dev_esc(esc))
    want = host_u16(whole)
    want_esc = escapes_to_numpy(we, wc)
    pipe = HostPipeline(codec, k, n, L, chunk)
    # the pipeline API takes no source escapes: use a clean source for it
    src2 = W.symbols(78, 0, S * k * L).reshape(S, k, L)
    w2, we2, wc2 = codec.encode(k, n, dev_u16(src2))
    src_h = torch.from_numpy(src2.view(np.int16)).pin_memory()
    nch = S // chunk
    enc_h = torch.empty((S, n, L), dtype=torch.int16).pin_memory()
    esc_h = torch.empty((nch, pipe.cap_e), dtype=torch.int64).pin_memory()
    cnt_h = torch.zeros(nch, dtype=torch.int64).pin_memory()
    pipe.encode_host(src_h, enc_h, esc_h, cnt_h)
    pipe.join()
    torch.cuda.synchronize()
    assert np.array_equal(enc_h.numpy().view(np.uint16), host_u16(w2))
    got = np.concatenate([esc_h[c, : int(cnt_h[c])].numpy().view(np.uint64) + np.uint64(c * chunk * n * L)
                          for c in range(nch)])
    assert np.array_equal(got, escapes_to_numpy(we2, wc2))
    # decode through the pipeline from received packets with escapes
    pats, sp = _patterns(S, n, k, seed=3)
    rx, rxe = W.received_packets(w2, we2, wc2, pats, sp, n)
    rx_h = rx.cpu().pin_memory()
    rxe_np = rxe.cpu().numpy().view(np.uint64) if rxe is not None else np.zeros(0, np.uint64)
    plans = codec.plans(k, n, pats)
    dec_h = torch.empty((S, k, L), dtype=torch.int16).pin_memory()
    desc_h = torch.empty((nch, pipe.cap_e), dtype=torch.int64).pin_memory()
    dcnt_h = torch.zeros(nch, dtype=torch.int64).pin_memory()
    pipe.decode_host(plans, torch.from_numpy(sp.view(np.int32)).cuda(), rx_h, rxe, dec_h, desc_h, dcnt_h,
                     escape_ranges(rxe_np, S, chunk, k, L))
    pipe.join()
    torch.cuda.synchronize()
    assert np.array_equal(dec_h.numpy().view(np.uint16), src2)
    assert int(dcnt_h.sum()) == 0
    assert want_esc.size > 0 and want.shape == (S, n, L)
    # encode and decode chunks interleaved on the streams (code_host): same results
    for nstreams in (2, 4):
        pipe2 = HostPipeline(codec, k, n, L, chunk, nstreams=nstreams)
        enc2 = torch.empty_like(enc_h).pin_memory()
        dec2 = torch.empty_like(dec_h).pin_memory()
        esc2 = torch.empty_like(esc_h).pin_memory()
        desc2 = torch.empty_like(desc_h).pin_memory()
        cnt2 = torch.zeros(nch, dtype=torch.int64).pin_memory()
        dcnt2 = torch.zeros(nch, dtype=torch.int64).pin_memory()
        pipe2.code_host(src_h, enc2, esc2, cnt2, plans, torch.from_numpy(sp.view(np.int32)).cuda(), rx_h, rxe,
                        dec2, desc2, dcnt2, escape_ranges(rxe_np, S, chunk, k, L))
        pipe2.join()
        torch.cuda.synchronize()
        assert np.array_equal(enc2.numpy().view(np.uint16), host_u16(w2))
        assert np.array_equal(dec2.numpy().view(np.uint16), src2) and int(dcnt2.sum()) == 0
        got2 = np.concatenate([esc2[c, : int(cnt2[c])].numpy().view(np.uint64) + np.uint64(c * chunk * n * L)
                               for c in range(nch)])
        assert np.array_equal(got2, escapes_to_numpy(we2, wc2))


# ------------------------------------------------------- randomized sweep ----
def _random_shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        e = int(rng.integers(1, 14))                       # n_domain up to 8192
        n = int(rng.integers((1 << (e - 1)) + 1, (1 << e) + 1)) if e > 1 else int(rng.integers(1, 3))
        k = int(rng.integers(1, n + 1))
        L = int(rng.choice([1, 3, 8, 16, 32, 40, 64]))
        S = int(rng.integers(1, 3))
        if n * L * S > 400_000 or (k > 2048 and L * S > 16):
            continue
        out.append((k, n, L, S))
    return out


@pytest.mark.parametrize("k,n,L,S", _random_shapes(20261019, 40))
def test_random_shapes_match_oracle(codec, oracle, k, n, L, S):
    """Seeded random (k, n, L, stripes) across every kernel family; each draw is
    encoded and decoded (from random k-subsets, including tampered values and
    input escapes) and compared bit for bit with the oracle."""
    from oracle_bind import gather_received
    from paper_0907_1788_b200 import escapes_to_numpy
    src, esc = source_with_escapes(S, k, L, seed=k * 31 + n * 7 + L, n_esc=2)
    want, want_esc = oracle.encode_stripes(k, n, src, esc)
    out, oe, cnt = codec.encode(k, n, dev_u16(src), dev_esc(esc))
    assert np.array_equal(host_u16(out), want) and np.array_equal(escapes_to_numpy(oe, cnt), want_esc)
    pats, sp = _patterns(S, n, k, seed=n + L)
    rx, rx_esc = gather_received(want, want_esc, pats, sp)
    rx = rx.copy()
    rx[0, -1, 0] ^= 0x1234  # not a codeword any more
    rx_esc = rx_esc[rx_esc != np.uint64((k - 1) * L)]
    dwant, dwant_esc = oracle.decode_stripes(k, n, pats, sp, rx, rx_esc)
    plans = codec.plans(k, n, pats)
    dout, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), dev_u16(rx), dev_esc(rx_esc))
    assert np.array_equal(host_u16(dout), dwant) and np.array_equal(escapes_to_numpy(de, dc), dwant_esc)


# ------------------------------------------------ committed golden fixtures ----
def test_gpu_matches_golden_fixtures(codec):
    """The CUDA path against tests/golden/reference_vectors.npz, generated from the
    reference library itself (tests/golden/make_golden.py): no oracle involved."""
    import paper_0907_1788_b200 as F
    path = os.path.join(ROOT, "tests", "golden", "reference_vectors.npz")
    g = np.load(path)
    for name in sorted({x.split("__")[0] for x in g.files}):
        kind, n, k = name.split("_")[0], int(name.split("_")[1]), int(name.split("_")[2])
        if kind in ("enc", "senc"):
            p = F.CodeParams.make(k, n, kind == "senc")
            fn = F.encode_systematic if kind == "senc" else F.encode_nonsystematic
            assert fn(p, [int(x) for x in g[name + "__src"]]) == [int(x) for x in g[name + "__out"]], name
        elif kind in ("dec", "sdec"):
            p = F.CodeParams.make(k, n, kind == "sdec")
            rx = [F.Symbol(int(z), int(v)) for z, v in zip(g[name + "__pos"], g[name + "__val"])]
            fn = F.decode_systematic if kind == "sdec" else F.decode_nonsystematic
            assert fn(p, rx) == [int(x) for x in g[name + "__out"]], name
        elif kind == "plan":
            a, ap, ps, af = codec.plans(k, n, g[name + "__pos"][None, :]).export(0)
            assert np.array_equal(a, g[name + "__a"]) and np.array_equal(ap, g[name + "__ap"]), name
            assert np.array_equal(af, g[name + "__afnt"]), name


# ------------------------------------------------------------ extreme sizes ----
@pytest.mark.parametrize("k,n,L", [(65536, 65536, 3), (65535, 65536, 2), (1, 65536, 5), (32768, 65536, 3)])
def test_maximum_sizes_match_oracle(codec, oracle, k, n, L):
    """Largest domain: rate 1 (complete reception), 2k > 65536 at its limit, k = 1."""
    from oracle_bind import gather_received
    from paper_0907_1788_b200 import escapes_to_numpy
    S = 1
    src, esc = source_with_escapes(S, k, L, seed=k + L, n_esc=2)
    want, want_esc = oracle.encode_stripes(k, n, src, esc)
    out, oe, cnt = codec.encode(k, n, dev_u16(src), dev_esc(esc), esc_cap=S * n * L)  # k = 1: 65536 everywhere
    assert np.array_equal(host_u16(out), want) and np.array_equal(escapes_to_numpy(oe, cnt), want_esc)
    if want_esc.size > 1000:  # the default (statistical) capacity reports the overflow instead of truncating
        import paper_0907_1788_b200 as F
        o2, e2, c2 = codec.encode(k, n, dev_u16(src), dev_esc(esc))
        with pytest.raises(F.TooManyEscapes):
            escapes_to_numpy(e2, c2)
    rng = np.random.default_rng(k)
    kp = n if k == n else k
    pats = np.sort(rng.choice(n, kp, replace=False)).astype(np.uint32)[None, :]
    sp = np.zeros(1, dtype=np.uint32)
    rx, rx_esc = gather_received(want, want_esc, pats, sp)
    plans = codec.plans(k, n, pats)
    dec, de, dc = codec.decode(plans, torch.zeros(1, dtype=torch.int32, device="cuda"), dev_u16(rx), dev_esc(rx_esc))
    assert np.array_equal(host_u16(dec), src)
    assert np.array_equal(escapes_to_numpy(de, dc), esc)


def test_empty_batches_are_no_ops(codec):
    from paper_0907_1788_b200 import escapes_to_numpy
    for k, n in [(128, 256), (8192, 16384), (3000, 4096)]:
        out, oe, cnt = codec.encode(k, n, torch.zeros((0, k, 64), dtype=torch.int16, device="cuda"))
        assert out.shape == (0, n, 64) and escapes_to_numpy(oe, cnt).size == 0
        plans = codec.plans(k, n, np.arange(k, dtype=np.uint32)[None, :])
        dec, de, dc = codec.decode(plans, torch.zeros(0, dtype=torch.int32, device="cuda"),
                                   torch.zeros((0, k, 64), dtype=torch.int16, device="cuda"))
        assert dec.shape == (0, k, 64) and escapes_to_numpy(de, dc).size == 0


@pytest.mark.parametrize("k,n,P", [(128, 256, 64), (1024, 2048, 3), (16, 32, 500), (2048, 4096, 2)])
def test_plan_methods_agree(codec, oracle, k, n, P, monkeypatch):
    """Direct products and the log-domain convolution (plans_create picks by
    cost; FNTRS_PLAN forces one) give identical plans and decodes."""
    from oracle_bind import gather_received
    rng = np.random.default_rng(k + P)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(P)]).astype(np.uint32)
    L, S = 32, P
    src, esc = source_with_escapes(S, k, L, seed=P, n_esc=2)
    want, want_esc = oracle.encode_stripes(k, n, src, esc)
    sp = np.arange(S, dtype=np.uint32)
    rx, rx_esc = gather_received(want, want_esc, pats, sp)
    outs = []
    for method in ("direct", "log"):
        monkeypatch.setenv("FNTRS_PLAN", method)
        plans = codec.plans(k, n, pats)
        fields = [plans.export(p) for p in (0, P - 1)]
        dec, _, _ = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), dev_u16(rx), dev_esc(rx_esc))
        outs.append((fields, host_u16(dec)))
    for (a, b) in zip(outs[0][0], outs[1][0]):
        assert all(np.array_equal(x, y) if isinstance(x, np.ndarray) else x == y for x, y in zip(a, b))
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][1], src)


@pytest.mark.parametrize("n,L,S,hot,cap", [
    (16, 64, 4, 0, None),          # no escapes
    (16, 64, 4, 1, None),          # one codeword: 16 escapes, single-CTA sort
    (64, 256, 2, 200, 16384),      # 12800 escapes, single-CTA sort at its 16K limit
    (64, 256, 2, 256, 16384),      # exactly 16384 = cap
    (256, 512, 2, 300, None),      # 76800 escapes > default cap: count reports the overflow
    (256, 512, 2, 300, 80000),     # 76800 escapes: tile sort + 5 merge passes
    (256, 512, 4, 5, 80000),       # few escapes in a large buffer (merge sort, mostly ~0 fill)
    (256, 512, 2, 40, 80000),      # 10240 live keys: tile sort + 2 merge passes (even: result in place)
    (256, 512, 2, 79, 80000),      # 20224 live keys: 3 merge passes (odd: copied back from scratch)
    (256, 1024, 4, 1000, 300000),  # 256000 live keys: 6 merge passes over 125 merge tiles
])
def test_escape_sort_paths(codec, n, L, S, hot, cap):
    """k = 1: every output of a codeword equals its source symbol, so `hot`
    codewords sourced with 65536 give exactly hot * n escapes, emitted in
    kernel order; both escape-sort paths must list them ascending."""
    from paper_0907_1788_b200 import escapes_to_numpy, TooManyEscapes
    rng = np.random.default_rng(n * L + hot)
    src = rng.integers(0, 65536, (S, 1, L)).astype(np.uint16)
    idx = np.sort(rng.choice(S * L, size=hot, replace=False)).astype(np.uint64)
    src.reshape(-1)[idx.astype(np.int64)] = 0
    s_i, c_i = idx // L, idx % L
    want_esc = np.sort(((s_i[:, None] * n + np.arange(n, dtype=np.uint64)[None, :]) * L + c_i[:, None]).reshape(-1))
    out, oe, cnt = codec.encode(1, n, dev_u16(src), dev_esc(idx), esc_cap=cap)
    want = np.repeat(src, n, axis=1)
    assert np.array_equal(host_u16(out), want)
    if cap is None and want_esc.size > oe.numel():
        assert int(cnt.item()) == want_esc.size
        with pytest.raises(TooManyEscapes):
            escapes_to_numpy(oe, cnt)
        return
    assert np.array_equal(escapes_to_numpy(oe, cnt), want_esc)
    assert np.all(oe[want_esc.size:].cpu().numpy() == -1)  # the ~0 fill stays after the real keys


def test_wide_stripe_offsets_beyond_32_bits(codec, oracle):
    """One stripe whose rows * L exceeds 2^32 symbols (a > 4 GiB file coded as
    one stripe, shards.encode_file): the fused kernels' 32-bit row offsets
    would wrap, so the C ABI routes it to the 64-bit tile kernels. The last
    columns (offsets above 2^32) are checked against the oracle, and
    decode(encode(s)) == s on the same columns."""
    from paper_0907_1788_b200 import escapes_to_numpy
    k, n, L = 16, 32, (1 << 27) + 64
    assert n * L >= 1 << 32
    src = torch.randint(-32768, 32767, (1, k, L), dtype=torch.int16, device="cuda")
    out, oe, cnt = codec.encode(k, n, src)
    tail = slice(L - 64, L)
    s_h = src[0, :, tail].cpu().numpy().view(np.uint16)[None].copy()
    want, want_esc = oracle.encode_stripes(k, n, s_h)
    got = out[0, :, tail].cpu().numpy().view(np.uint16)[None]
    assert np.array_equal(got, want)
    esc = escapes_to_numpy(oe, cnt)
    tail_esc = [int(e // L) * 64 + int(e % L) - (L - 64) for e in esc if e % L >= L - 64]
    assert tail_esc == [int(e) for e in want_esc]
    pats = np.array([np.arange(n - k, n)], dtype=np.uint32)  # parity rows only
    plans = codec.plans(k, n, pats)
    rx = out[:, n - k:, :].contiguous()
    rx_esc = [int(e) - (n - k) * L for e in esc if e >= (n - k) * L]
    rxe = torch.tensor(rx_esc, dtype=torch.int64, device="cuda") if rx_esc else None
    del out
    dec, de, dc = codec.decode(plans, torch.zeros(1, dtype=torch.int32, device="cuda"), rx, rxe)
    assert torch.equal(dec[0, :, tail], src[0, :, tail])
    assert torch.equal(dec[0, :, :4096], src[0, :, :4096])
    assert escapes_to_numpy(de, dc).size == 0


@pytest.mark.parametrize("k,n,L,S", [(4096, 8192, 64, 3), (8192, 16384, 128, 2), (5000, 16384, 64, 2),
                                     (5000, 10000, 64, 2), (16384, 32768, 64, 1), (32768, 65536, 64, 1)])
def test_streamed_four_step_matches_batched(codec, monkeypatch, k, n, L, S):
    """The streamed four-step kernels (one persistent launch, L2 rings,
    FNTRS_STREAM=1) give the batched kernels' payloads and escape lists."""
    from paper_0907_1788_b200 import escapes_to_numpy, workload as W
    src = torch.from_numpy(W.symbols(k * 7 + n, 0, S * k * L).view(np.int16).reshape(S, k, L)).cuda()
    rng = np.random.default_rng(k + n)
    pats = np.stack([np.sort(rng.choice(n, k, replace=False)) for _ in range(S)]).astype(np.uint32)
    sp = np.arange(S, dtype=np.uint32)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("FNTRS_STREAM", mode)
        out, oe, cnt = codec.encode(k, n, src)
        rx, rxe = W.received_packets(out, oe, cnt, pats, sp, n)
        rx[:, 0, :7] = 0  # a few zero words; some become escapes below
        rxe = rxe if rxe is not None else torch.zeros(0, dtype=torch.int64, device="cuda")
        rxe = torch.unique(torch.cat([rxe, torch.arange(3, device="cuda", dtype=torch.int64)]))
        plans = codec.plans(k, n, pats)
        dec, de, dc = codec.decode(plans, torch.from_numpy(sp.view(np.int32)).cuda(), rx, rxe)
        res[mode] = (out.cpu(), escapes_to_numpy(oe, cnt), dec.cpu(), escapes_to_numpy(de, dc))
        plans.close()
    for a, b in zip(res["0"], res["1"]):
        assert (torch.equal(a, b) if isinstance(a, torch.Tensor) else np.array_equal(a, b))
