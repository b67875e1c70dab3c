"""Config-scale bit-exactness: the CUDA path against the UNMODIFIED reference
library (oracle/_ref, all host cores) on the five BASELINE.json configs.

Model: the reference's own acceptance test (proj/tests/acceptance.cpp:134-191)
and SURVEY.md 8(d)'s bit-exact plan:
  * encode payloads AND escape lists compared in full: C1, C3, C4, C5 (every
    stripe, streamed in stripe chunks -- stripes are independent, so a chunked
    comparison covers exactly the same codewords), C2 on a stratified 1/32
    sample (32 blocks of 64 consecutive stripes spread over all 65536, both
    pattern classes);
  * decode compared in full on C1, C3, C4 (every stripe of the three erasure
    classes: uniform, parity-only, bursts) and C5, and on the same 1/32 sample
    of C2 (shared and distinct patterns); from the codewords, and on a subset
    of stripes of every config from tampered received rows (non-codewords:
    the decoder must return the same unique interpolant as the reference,
    escapes included).
Source symbols are generated on the device by the product's generator
(fntrs_gpu_fill_symbols, itself checked against numpy in
test_gpu_parity.py::test_device_generator_matches_numpy) at the global symbol
index of each stripe, so every chunk is the config's own data.
"""
import ctypes as C
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0907_1788_b200 import Codec
    return Codec(0)


@pytest.fixture(scope="module")
def reflib():
    from oracle_bind import RefLib
    if not RefLib.available():
        pytest.skip("reference library (oracle/_ref) not built")
    return RefLib()


def device_source(cfg, s0, count, seed=None):
    """Stripes [s0, s0+count) of the config's source, generated on the device."""
    from paper_0907_1788_b200 import _lib, workload as W
    t = torch.empty((count, cfg.k, cfg.L), dtype=torch.int16, device="cuda")
    st = _lib.load().fntrs_gpu_fill_symbols(W.SEED if seed is None else seed, s0 * cfg.k * cfg.L, t.numel(),
                                            C.c_void_p(t.data_ptr()),
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    return t


def host(t):
    return t.cpu().numpy().view(np.uint16)


def esc_np(e, cnt):
    from paper_0907_1788_b200 import escapes_to_numpy
    return escapes_to_numpy(e, cnt)


def dev_esc(e):
    if e is None or len(e) == 0:
        return None
    return torch.from_numpy(np.ascontiguousarray(e, dtype=np.uint64).view(np.int64)).cuda()


def check_encode_chunk(codec, reflib, cfg, s0, count):
    src = device_source(cfg, s0, count)
    out, oe, cnt = codec.encode(cfg.k, cfg.n, src)
    got, got_esc = host(out), esc_np(oe, cnt)
    want, want_esc = reflib.encode_stripes(cfg.k, cfg.n, host(src), threads=THREADS)
    assert np.array_equal(got, want), f"{cfg.name} encode payload differs in stripes [{s0}, {s0 + count})"
    assert np.array_equal(got_esc, want_esc), f"{cfg.name} encode escape list differs in [{s0}, {s0 + count})"
    return host(src), got, got_esc


def tamper(rx, rxe, seed, rows_per_stripe=3):
    """Overwrite a few received rows per stripe with random words (some 0 words
    become 65536 through the escape list): the input is no longer a codeword."""
    rng = np.random.default_rng(seed)
    S, kp, L = rx.shape
    rx = rx.copy()
    for s in range(S):
        for r in rng.choice(kp, size=min(rows_per_stripe, kp), replace=False):
            rx[s, r] = rng.integers(0, 65536, L, dtype=np.uint16)
    # keep the escapes that still sit on zero words; add fresh ones on some zero words
    flat = rx.reshape(-1)
    keep = [int(e) for e in rxe if flat[int(e)] == 0]
    zeros = np.flatnonzero(flat == 0)
    extra = rng.choice(zeros, size=min(len(zeros), 4 * S), replace=False) if zeros.size else []
    esc = np.unique(np.array(keep + [int(z) for z in extra], dtype=np.uint64))
    return rx, esc


def check_decode(codec, reflib, cfg, pats, sp, rx, rxe, label):
    """GPU decode of [S, k, L] received rows vs the reference library (Path::Fast:
    Auto/Fast/Direct give the same values, tests/test_oracle.py)."""
    plans = codec.plans(cfg.k, cfg.n, pats)
    dec, de, dc = codec.decode(plans, torch.from_numpy(sp.astype(np.int32)).cuda(),
                               torch.from_numpy(np.ascontiguousarray(rx).view(np.int16)).cuda(), dev_esc(rxe))
    got, got_esc = host(dec), esc_np(de, dc)
    want, want_esc = reflib.decode_stripes(cfg.k, cfg.n, pats, sp, rx, rxe, path=1, threads=THREADS)
    assert np.array_equal(got, want), f"{cfg.name} decode payload differs ({label})"
    assert np.array_equal(got_esc, want_esc), f"{cfg.name} decode escape list differs ({label})"
    plans.close()
    return got, got_esc


def sub_patterns(pats_all, sp_all, stripes):
    used, sp = np.unique(sp_all[stripes], return_inverse=True)
    return pats_all[used], sp.astype(np.uint32)


def decode_sample(codec, reflib, cfg, stripes, src_h, enc_h, esc_h, pats_all, sp_all, tamper_seed, tampered=None):
    """Decode the listed stripes (their encoded rows given) from codewords and,
    for the first `tampered` of them (all by default), from tampered rows; both
    against the reference."""
    from oracle_bind import gather_received
    pats, sp = sub_patterns(pats_all, sp_all, stripes)
    rx, rxe = gather_received(enc_h, esc_h, pats, sp)
    got, got_esc = check_decode(codec, reflib, cfg, pats, sp, rx, rxe, "codewords")
    assert np.array_equal(got, src_h) and got_esc.size == 0
    t = len(stripes) if tampered is None else min(tampered, len(stripes))
    if t:
        pats_t, sp_t = sub_patterns(pats_all, sp_all, np.asarray(stripes)[:t])
        esc_t = rxe[rxe < np.uint64(t * cfg.k * cfg.L)]
        trx, trxe = tamper(rx[:t], esc_t, tamper_seed)
        check_decode(codec, reflib, cfg, pats_t, sp_t, trx, trxe, "tampered rows")


# --------------------------------------------------------------------- C1 ----
def test_c1_full(codec, reflib):
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS["C1"]
    src, enc, esc = check_encode_chunk(codec, reflib, cfg, 0, 1)
    pats, sp = W.patterns(cfg)
    decode_sample(codec, reflib, cfg, np.arange(1), src, enc, esc, pats, sp, 11)


# --------------------------------------------------------------------- C3 ----
def test_c3_full(codec, reflib):
    """n = 65536: encode of all 2048 codewords and decode of all 2048 (16384
    source + 16384 parity rows received), then the same decode from tampered rows."""
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS["C3"]
    src, enc, esc = check_encode_chunk(codec, reflib, cfg, 0, 1)
    pats, sp = W.patterns(cfg)
    assert (pats[0] < 32768).sum() == 16384
    decode_sample(codec, reflib, cfg, np.arange(1), src, enc, esc, pats, sp, 33)


# --------------------------------------------------------------------- C4 ----
def test_c4_full(codec, reflib):
    """All 256 stripes encoded AND decoded (chunks of 32) against the
    reference: every stripe of the three erasure classes (uniform, parity
    only, 1024-bursts); tampered rows on 6 stripes (two per class) per chunk."""
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS["C4"]
    pats_all, sp_all = W.patterns(cfg)
    chunk = 32
    for c, s0 in enumerate(range(0, cfg.stripes, chunk)):
        src, enc, esc = check_encode_chunk(codec, reflib, cfg, s0, chunk)
        idx = np.arange(chunk)
        decode_sample(codec, reflib, cfg, s0 + idx, src, enc, esc, pats_all, sp_all, 44 + c, tampered=6)
    assert {int(s) % 3 for s in range(6)} == {0, 1, 2}


# --------------------------------------------------------------------- C5 ----
def test_c5_full(codec, reflib):
    """All 2048 stripes (8 GiB of source) encoded AND decoded in chunks of 128
    against the reference; tampered rows on 8 stripes of every fourth chunk."""
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS["C5"]
    pats_all, sp_all = W.patterns(cfg)
    chunk = 128
    for c, s0 in enumerate(range(0, cfg.stripes, chunk)):
        src, enc, esc = check_encode_chunk(codec, reflib, cfg, s0, chunk)
        idx = np.arange(chunk)
        decode_sample(codec, reflib, cfg, s0 + idx, src, enc, esc, pats_all, sp_all, 55 + c,
                      tampered=8 if c % 4 == 1 else 0)


# --------------------------------------------------------------------- C2 ----
def test_c2_stratified_sample(codec, reflib):
    """1/32 of C2 (32 blocks of 64 consecutive stripes, one block every 2048
    stripes): encode payload + escapes and decode of every sampled stripe
    (even stripes on the shared pattern P0, odd on distinct patterns); tampered
    rows on 16 stripes per block."""
    from paper_0907_1788_b200 import workload as W
    cfg = W.CONFIGS["C2"]
    pats_all, sp_all = W.patterns(cfg)
    block = 64
    for b, s0 in enumerate(range(0, cfg.stripes, 2048)):
        src, enc, esc = check_encode_chunk(codec, reflib, cfg, s0, block)
        idx = np.arange(block)
        assert (sp_all[s0 + idx][0::2] == 0).all() and (sp_all[s0 + idx][1::2] != 0).all()
        decode_sample(codec, reflib, cfg, s0 + idx, src, enc, esc, pats_all, sp_all, 200 + b, tampered=16)
