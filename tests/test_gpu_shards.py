"""GPU file codec (paper_0907_1788_b200.shards.encode_file / decode_file):
byte-identical shards and manifest versus the reference CLI's encode loop run
through the reference library (oracle/_ref: symbolize, per-stripe encode,
write_shard, write_manifest), and recovery under shard loss and corruption
(acceptance.cpp:423-494, criterion 8, without the CLI binary)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def codec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_0907_1788_b200 import Codec
    return Codec(0)


def _bytes(size, seed):
    return np.random.default_rng(seed).integers(0, 256, size, dtype=np.uint8).tobytes()


CASES = [  # (bytes, k, n, systematic)
    (1001, 3, 7, True), (1000, 3, 7, False), (100001, 16, 32, False), (300000, 1024, 2048, True),
    (40000, 100, 256, True), (50000, 5000, 9000, True), (20000, 100, 65536, False), (0, 4, 8, True), (1, 1, 2, False),
]


@pytest.mark.parametrize("size,k,n,sys_", CASES)
def test_encode_file_matches_reference(codec, ref, size, k, n, sys_):
    from paper_0907_1788_b200 import shards as SH
    data = _bytes(size, size + k)
    got = SH.encode_file(data, k, n, systematic=sys_, chunk_id=0x1234 + size, codec=codec)
    man, shards = ref.encode_file(data, k, n, systematic=sys_, chunk_id=0x1234 + size)
    assert got[SH.manifest_filename(0x1234 + size)] == man
    for j in range(n):
        assert got[SH.shard_filename(0x1234 + size, j)] == shards[j], j


@pytest.mark.parametrize("size,k,n,sys_", CASES[:6])
def test_decode_file_recovers_from_any_k_shards(codec, size, k, n, sys_):
    import paper_0907_1788_b200 as F
    from paper_0907_1788_b200 import shards as SH
    data = _bytes(size, 7 * size + n)
    files = SH.encode_file(data, k, n, systematic=sys_, chunk_id=5, codec=codec)
    rng = np.random.default_rng(size)
    man = SH.manifest_filename(5)
    for trial in range(3):
        keep = rng.choice(n, k + (trial == 2), replace=False)
        sub = {man: files[man]}
        sub.update({SH.shard_filename(5, int(j)): files[SH.shard_filename(5, int(j))] for j in keep})
        assert SH.decode_file(sub, codec=codec) == data
    # a corrupt shard and a foreign shard are skipped; with them only, too few remain
    keep = list(rng.choice(n, k, replace=False))
    sub = {man: files[man]}
    sub.update({SH.shard_filename(5, int(j)): files[SH.shard_filename(5, int(j))] for j in keep})
    bad = SH.shard_filename(5, int(keep[0]))
    sub[bad] = b"XXXX" + sub[bad][4:]
    warned = []
    with pytest.raises(F.NotEnoughShards):
        SH.decode_file(sub, codec=codec, warn=warned.append)
    assert warned and "unreadable" in warned[0]
    spare = next(j for j in range(n) if j not in keep)
    sub[SH.shard_filename(5, spare)] = files[SH.shard_filename(5, spare)]
    assert SH.decode_file(sub, codec=codec) == data


def test_ten_megabytes_survive_deletion_patterns(codec):  # criterion 8 shape: 10 MB, (1024, 2048)
    from paper_0907_1788_b200 import shards as SH
    data = _bytes(10 * 1024 * 1024, 808)
    files = SH.encode_file(data, 1024, 2048, chunk_id=424242, codec=codec)
    man = SH.manifest_filename(424242)
    rng = np.random.default_rng(808)
    for _ in range(5):
        ids = rng.permutation(2048)[1024:]
        sub = {man: files[man]}
        sub.update({SH.shard_filename(424242, int(j)): files[SH.shard_filename(424242, int(j))] for j in ids})
        assert SH.decode_file(sub, codec=codec) == data
