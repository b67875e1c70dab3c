"""Shard and manifest wire format, and whole-file encode / decode
(reference: proj/src/shardio.cpp, proj/include/fntrs/shardio.hpp, and the
CLI's encode/decode loops proj/tools/fntrs_main.cpp:117-238).

The payload bytes move on the GPU (fntrs_gpu_symbolize / words_to_be /
be_to_words / desymbolize) and the codec runs in the batched kernels; this
module formats the small per-shard headers, escape lists and the manifest on
the host, with the reference's validation and error classes.

    files = encode_file(data, k=1024, n=2048, chunk_id=7)      # {name: bytes}
    data2 = decode_file({name: b for name, b in files.items() if keep(name)})
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .codec import (BadMagic, BadVersion, Codec, LengthMismatch, MalformedEscapes, MalformedHeader,
                    NotEnoughShards, SizeMismatch, TooManyEscapes, TruncatedShard, escapes_to_numpy)

SHARD_MAGIC = b"FNTC"      # shardio.cpp:11
MANIFEST_MAGIC = b"FNTM"   # shardio.cpp:12
VERSION = 1                # shardio.cpp:13
FLAG_SYSTEMATIC = 0x01     # shardio.cpp:14
HEADER_BYTES = 26          # magic 4, version 1, chunk 8, k 2, n 2, index 2, flags 1, symbols 4, escapes 2
MAX_ESCAPES = 65535


@dataclass(frozen=True)
class ShardInfo:  # shardio.hpp:36-44
    chunk_id: int
    k: int
    n: int
    shard_index: int
    systematic: bool = True


@dataclass(frozen=True)
class ChunkManifest:  # shardio.hpp:62-71
    chunk_id: int
    original_length: int
    k: int
    n: int
    stripes: int
    systematic: bool = True


def shard_filename(chunk_id: int, shard_index: int) -> str:  # shardio.cpp:261-266
    return f"{chunk_id:016x}.{shard_index}.fnt"


def manifest_filename(chunk_id: int) -> str:  # shardio.cpp:268-273
    return f"{chunk_id:016x}.manifest.fnt"


def _n_to_wire(n: int) -> int:  # 65536 travels as 0 (shardio.cpp:74-77)
    return 0 if n == 65536 else n


def _n_from_wire(w: int) -> int:
    return 65536 if w == 0 else w


def _check_info(info: ShardInfo):  # write_shard validation (shardio.cpp:118-128)
    if not 1 <= info.k <= 65535:
        raise SizeMismatch(f"shard header k must be in [1, 65535], got {info.k}")
    if not info.k <= info.n <= 65536:
        raise SizeMismatch(f"shard header n must be in [k, 65536], got {info.n}")
    if info.shard_index >= info.n:
        raise SizeMismatch(f"shard index {info.shard_index} not below n = {info.n}")


def shard_header(info: ShardInfo, payload_symbols: int, escapes) -> bytes:
    """Header + escape list of write_shard (shardio.cpp:141-152)."""
    _check_info(info)
    if payload_symbols > 0xFFFFFFFF:
        raise SizeMismatch("payload too long for a shard")
    esc = np.asarray(escapes, dtype=np.uint32)
    if esc.size > MAX_ESCAPES:
        raise TooManyEscapes(f"{esc.size} escaped symbols in one shard, limit is {MAX_ESCAPES}")
    head = SHARD_MAGIC + struct.pack(">BQHHHBIH", VERSION, info.chunk_id, info.k, _n_to_wire(info.n),
                                     info.shard_index, FLAG_SYSTEMATIC if info.systematic else 0,
                                     payload_symbols, esc.size)
    return head + esc.astype(">u4").tobytes()


def write_shard(info: ShardInfo, payload) -> bytes:
    """shardio::write_shard (shardio.cpp:118-155) for a host list of field values."""
    v = np.asarray(payload, dtype=np.int64)
    if v.size and (v.min() < 0 or v.max() > 65536):
        raise SizeMismatch("payload value outside the field")
    esc = np.nonzero(v == 65536)[0]
    words = np.where(v == 65536, 0, v).astype(">u2")
    return shard_header(info, v.size, esc) + words.tobytes()


def _parse_shard(b: bytes):
    """read_shard (shardio.cpp:157-209) without materialising the payload:
    returns (info, payload_symbols, escapes uint32, payload byte offset)."""
    if len(b) < 4:
        raise TruncatedShard(f"need 4 more bytes at offset 0, have {len(b)}")
    if b[:4] != SHARD_MAGIC:
        raise BadMagic("unrecognized file magic")
    if len(b) < 5:
        raise TruncatedShard("need 1 more bytes at offset 4, have 0")
    if b[4] != VERSION:
        raise BadVersion(f"shard version {b[4]}, expected {VERSION}")
    if len(b) < HEADER_BYTES:
        raise TruncatedShard(f"need {HEADER_BYTES - 5} more bytes at offset 5, have {len(b) - 5}")
    chunk, k, nw, idx, flags, symbols, ne = struct.unpack(">QHHHBIH", b[5:HEADER_BYTES])
    if flags & ~FLAG_SYSTEMATIC:
        raise MalformedHeader(f"unknown flag bits set: {flags}")
    info = ShardInfo(chunk, k, _n_from_wire(nw), idx, bool(flags & FLAG_SYSTEMATIC))
    if info.k == 0:
        raise MalformedHeader("shard header has k = 0")
    if info.n < info.k:
        raise MalformedHeader(f"shard header has n = {info.n} below k = {info.k}")
    if info.shard_index >= info.n:
        raise MalformedHeader(f"shard index {info.shard_index} not below n = {info.n}")
    off = HEADER_BYTES + 4 * ne
    if len(b) < off:
        raise TruncatedShard(f"need {4 * ne} more bytes at offset {HEADER_BYTES}, have {len(b) - HEADER_BYTES}")
    esc = np.frombuffer(b, dtype=">u4", count=ne, offset=HEADER_BYTES).astype(np.uint32)
    if ne and int(esc.max()) >= symbols:
        bad = int(esc[np.argmax(esc >= symbols)])
        raise MalformedEscapes(f"escape position {bad} not below payload size {symbols}")
    if ne > 1 and np.any(esc[1:] <= esc[:-1]):
        raise MalformedEscapes("escape positions not strictly increasing")
    if len(b) < off + 2 * symbols:
        raise TruncatedShard(f"need {2 * symbols} more bytes at offset {off}, have {len(b) - off}")
    if len(b) != off + 2 * symbols:
        raise MalformedHeader(f"{len(b) - off - 2 * symbols} trailing bytes after the payload")
    words = np.frombuffer(b, dtype=">u2", count=symbols, offset=off)
    if ne and np.any(words[esc.astype(np.int64)] != 0):
        bad = int(esc[np.argmax(words[esc.astype(np.int64)] != 0)])
        raise MalformedEscapes(f"escape at position {bad} points at a nonzero word")
    return info, symbols, esc, off


def read_shard(b: bytes):
    """shardio::read_shard: (ShardInfo, payload as a list of field values)."""
    info, symbols, esc, off = _parse_shard(b)
    v = np.frombuffer(b, dtype=">u2", count=symbols, offset=off).astype(np.int64)
    v[esc.astype(np.int64)] = 65536
    return info, [int(x) for x in v]


def write_manifest(m: ChunkManifest) -> bytes:  # shardio.cpp:211-231
    if not 1 <= m.k <= 65535:
        raise SizeMismatch(f"manifest k must be in [1, 65535], got {m.k}")
    if not m.k <= m.n <= 65536:
        raise SizeMismatch(f"manifest n must be in [k, 65536], got {m.n}")
    if m.original_length > m.stripes * m.k * 2:
        raise LengthMismatch(f"manifest length {m.original_length} exceeds stripe capacity")
    return MANIFEST_MAGIC + struct.pack(">BQQHHIB", VERSION, m.chunk_id, m.original_length, m.k, _n_to_wire(m.n),
                                        m.stripes, FLAG_SYSTEMATIC if m.systematic else 0)


def read_manifest(b: bytes) -> ChunkManifest:  # shardio.cpp:233-259
    if len(b) < 4:
        raise TruncatedShard("manifest too short")
    if b[:4] != MANIFEST_MAGIC:
        raise BadMagic("unrecognized file magic")
    if len(b) < 5:
        raise TruncatedShard("manifest too short")
    if b[4] != VERSION:
        raise BadVersion(f"manifest version {b[4]}, expected {VERSION}")
    if len(b) < 30:
        raise TruncatedShard(f"need {30 - len(b)} more bytes")
    chunk, length, k, nw, stripes, flags = struct.unpack(">QQHHIB", b[5:30])
    if flags & ~FLAG_SYSTEMATIC:
        raise MalformedHeader(f"unknown flag bits set: {flags}")
    if len(b) != 30:
        raise MalformedHeader(f"{len(b) - 30} trailing bytes after the manifest")
    m = ChunkManifest(chunk, length, k, _n_from_wire(nw), stripes, bool(flags & FLAG_SYSTEMATIC))
    if m.k == 0:
        raise MalformedHeader("manifest has k = 0")
    if m.n < m.k:
        raise MalformedHeader("manifest has n below k")
    if m.original_length > m.stripes * m.k * 2:
        raise MalformedHeader("manifest length exceeds stripe capacity")
    return m


# ------------------------------------------------------------ file codec ----
def _width(S: int, n_domain: int) -> int:
    """Symbols per packet: the CLI stripe count rounded up to a multiple of every
    fused kernel's tile width (64)."""
    w = 64
    return max(w, (S + w - 1) // w * w)


def _check(codec: Codec, st: int):
    codec._check(st)


def encode_file(data: bytes, k: int, n: int, systematic: bool = True, chunk_id: int = 0,
                codec: Codec | None = None) -> dict:
    """The reference CLI's `encode` (fntrs_main.cpp:117-160) without the file
    system: returns {file name: bytes} for the manifest and the n shards,
    byte-identical to the reference's output."""
    import torch
    from .codec import CodeParams
    params = CodeParams.make(k, n, systematic)
    if k > 65535:
        raise SizeMismatch(f"shard header k must be in [1, 65535], got {k}")
    codec = codec or Codec(0)
    lib = _lib.load()
    dev = torch.device(f"cuda:{codec.device}")
    nbytes = len(data)
    words = (nbytes + 1) // 2
    S = (words + k - 1) // k                     # CLI stripes = symbols per shard
    L = _width(S, params.n_domain)
    d_data = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev) if nbytes else \
        torch.zeros(1, dtype=torch.uint8, device=dev)
    src = torch.empty((1, k, L), dtype=torch.int16, device=dev)
    _check(codec, lib.fntrs_gpu_symbolize(codec.ctx, C.c_void_p(d_data.data_ptr()), nbytes, k, L,
                                          C.c_void_p(src.data_ptr()), None))
    enc, oe, cnt = codec.encode(k, n, src, systematic=systematic)
    esc = escapes_to_numpy(oe, cnt)              # ascending row*L + col
    pay = torch.empty((n, max(2 * S, 1)), dtype=torch.uint8, device=dev)
    _check(codec, lib.fntrs_gpu_words_to_be(codec.ctx, C.c_void_p(enc.data_ptr()), n, L, S,
                                            C.c_void_p(pay.data_ptr()), pay.shape[1], None))
    pay_h = pay.cpu().numpy()
    rows = (esc // L).astype(np.int64)
    cols = (esc % L).astype(np.uint32)
    cuts = np.searchsorted(rows, np.arange(n + 1))
    out = {manifest_filename(chunk_id): write_manifest(ChunkManifest(chunk_id, nbytes, k, n, S, systematic))}
    for j in range(n):
        head = shard_header(ShardInfo(chunk_id, k, n, j, systematic), S, cols[cuts[j]:cuts[j + 1]])
        out[shard_filename(chunk_id, j)] = head + pay_h[j, :2 * S].tobytes()
    return out


def decode_file(files: dict, manifest_name: str | None = None, codec: Codec | None = None,
                warn=None) -> bytes:
    """The reference CLI's `decode` (fntrs_main.cpp:186-238) over {file name:
    bytes}: shards that fail to parse or disagree with the manifest are
    skipped (reported through `warn`), the k lowest surviving positions are
    decoded, and the original bytes returned. NotEnoughShards below k."""
    import torch
    from .codec import CodeParams
    if manifest_name is None:
        names = [nm for nm in files if nm.endswith(".manifest.fnt")]
        if len(names) != 1:
            raise ValueError("no manifest" if not names else "multiple manifests; pass one explicitly")
        manifest_name = names[0]
    m = read_manifest(files[manifest_name])
    params = CodeParams.make(m.k, m.n, m.systematic)
    codec = codec or Codec(0)
    lib = _lib.load()
    dev = torch.device(f"cuda:{codec.device}")
    positions, parsed = [], []
    for j in range(m.n):
        b = files.get(shard_filename(m.chunk_id, j))
        if b is None:
            continue
        try:
            info, symbols, esc, off = _parse_shard(b)
        except Exception as e:  # the reference's Error classes: unreadable shard, skipped
            if warn:
                warn(f"{shard_filename(m.chunk_id, j)} unreadable ({e}), skipping")
            continue
        if (info.chunk_id != m.chunk_id or info.k != m.k or info.n != m.n or info.systematic != m.systematic
                or info.shard_index != j or symbols != m.stripes):
            if warn:
                warn(f"{shard_filename(m.chunk_id, j)} does not match the manifest, skipping")
            continue
        positions.append(j)
        parsed.append((b, esc, off))
    if len(positions) < m.k:
        raise NotEnoughShards(f"not enough shards: found {len(positions)}, required {m.k}")
    S = m.stripes
    if (m.original_length + 1) // 2 > S * m.k or S * m.k > 0 and (m.original_length + 1) // 2 <= (S - 1) * m.k:
        raise LengthMismatch(f"length {m.original_length} implies a different stripe count than {S}")
    L = _width(S, params.n_domain)
    full = params.n == params.n_domain and len(positions) == params.n and not m.systematic
    kp = m.n if full else m.k                     # codec.cpp:137-144, else the k lowest positions
    use = list(range(kp))
    pitch = 2 * S
    host = np.empty((kp, max(pitch, 1)), dtype=np.uint8)
    keys = []
    for r, i in enumerate(use):
        b, esc, off = parsed[i]
        host[r, :pitch] = np.frombuffer(b, dtype=np.uint8, count=pitch, offset=off)
        if esc.size:
            keys.append(np.uint64(r) * np.uint64(L) + esc.astype(np.uint64))
    d_pay = torch.from_numpy(host).to(dev)
    rx = torch.empty((1, kp, L), dtype=torch.int16, device=dev)
    _check(codec, lib.fntrs_gpu_be_to_words(codec.ctx, C.c_void_p(d_pay.data_ptr()), host.shape[1], kp, S, L,
                                            C.c_void_p(rx.data_ptr()), None))
    rx_esc = None
    if keys:
        k_all = np.concatenate(keys)
        rx_esc = torch.from_numpy(k_all.view(np.int64)).to(dev)
    pos = np.array([positions[i] for i in use], dtype=np.uint32)
    plans = codec.plans(m.k, m.n, pos[None, :])
    sp = torch.zeros(1, dtype=torch.int32, device=dev)
    dec, _, _ = codec.decode(plans, sp, rx, rx_esc, systematic=m.systematic)
    out = torch.empty(max(m.original_length, 1), dtype=torch.uint8, device=dev)
    _check(codec, lib.fntrs_gpu_desymbolize(codec.ctx, C.c_void_p(dec.data_ptr()), m.k, L, m.original_length,
                                            C.c_void_p(out.data_ptr()), None))
    result = bytes(out[: m.original_length].cpu().numpy().tobytes())
    plans.close()
    return result
