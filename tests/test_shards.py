"""Shard / manifest wire format (host formatting, paper_0907_1788_b200/shards.py)
against the reference's frozen bytes (proj/tests/test_shardio.cpp) and the
reference library itself (oracle/_ref: shardio::write_shard / read_shard)."""
import numpy as np
import pytest

import paper_0907_1788_b200 as F
from paper_0907_1788_b200 import shards as SH


def test_shard_bytes_match_the_frozen_layout():  # test_shardio.cpp:70-87
    info = SH.ShardInfo(0x0102030405060708, 2, 4, 1, True)
    b = SH.write_shard(info, [5, 65536, 7])
    want = bytes([0x46, 0x4e, 0x54, 0x43, 0x01,
                  0x01, 0x02, 0x03, 0x04, 0x05, 0x06, 0x07, 0x08,
                  0x00, 0x02, 0x00, 0x04, 0x00, 0x01, 0x01,
                  0x00, 0x00, 0x00, 0x03,
                  0x00, 0x01, 0x00, 0x00, 0x00, 0x01,
                  0x00, 0x05, 0x00, 0x00, 0x00, 0x07])
    assert b == want
    back, payload = SH.read_shard(b)
    assert back == info and payload == [5, 65536, 7]


def test_payload_without_escapes():  # test_shardio.cpp:89-100
    b = SH.write_shard(SH.ShardInfo(1, 1, 2, 0, False), [1, 2, 3])
    assert len(b) == 26 + 6 and b[24] == 0 and b[25] == 0
    info, payload = SH.read_shard(b)
    assert info.systematic is False and payload == [1, 2, 3]


def test_manifest_roundtrip_and_n_65536():
    m = SH.ChunkManifest(7, 1000, 300, 65536, 2, True)
    b = SH.write_manifest(m)
    assert len(b) == 30 and SH.read_manifest(b) == m
    assert SH.manifest_filename(7) == "0000000000000007.manifest.fnt"
    assert SH.shard_filename(0xABC, 12) == "0000000000000abc.12.fnt"
    with pytest.raises(F.LengthMismatch):
        SH.write_manifest(SH.ChunkManifest(7, 1201, 300, 400, 2, True))


def test_write_shard_matches_reference_library(ref):
    rng = np.random.default_rng(3)
    for trial in range(40):
        k = int(rng.integers(1, 2000))
        n = int(rng.integers(k, 65537))
        idx = int(rng.integers(0, n))
        cnt = int(rng.integers(0, 300))
        payload = rng.integers(0, 65537, cnt)
        if cnt:
            payload[rng.integers(0, cnt, 3)] = 65536
        info = SH.ShardInfo(int(rng.integers(0, 2**63)), k, n, idx, bool(trial & 1))
        want, st = ref.write_shard(info.chunk_id, k, n, idx, info.systematic, payload)
        assert st == 0 and SH.write_shard(info, payload) == want


CODE = {"Error": 1, "TooManyEscapes": 11, "BadMagic": 12, "BadVersion": 13, "TruncatedShard": 14,
        "MalformedEscapes": 15, "MalformedHeader": 16, "LengthMismatch": 17, "SizeMismatch": 4}


def _status(b):
    try:
        SH.read_shard(b)
        return 0
    except F.Error as e:
        return CODE[type(e).__name__]


def test_read_shard_validation_matches_reference_library(ref):  # shardio.cpp:157-209
    good = SH.write_shard(SH.ShardInfo(9, 3, 8, 5, True), [1, 65536, 3, 0, 65536])
    cases = [good, good[:3], b"XNTC" + good[4:], good[:4] + b"\x02" + good[5:], good[:20], good[:-1],
             good + b"\x00", good[:19] + b"\x02" + good[20:],       # unknown flag
             good[:13] + b"\x00\x00" + good[15:],                   # k = 0
             good[:13] + b"\x00\x09" + good[15:],                   # n < k
             good[:17] + b"\x00\x08" + good[19:],                   # index >= n
             good[:26] + b"\x00\x00\x00\x04" + good[30:],           # escapes not increasing
             good[:30] + b"\x00\x00\x00\x09" + good[34:],           # escape out of range
             good[:36] + b"\x00\x07" + good[38:]]                   # escape at a nonzero word
    for b in cases:
        assert _status(b) == ref.read_shard_status(b), b.hex()
