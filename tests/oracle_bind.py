"""ctypes bindings of the TEST-ONLY checkers (oracle/).

* ``Oracle``: oracle/liboracle.so, the C restatement (oracle/fntrs_oracle.c).
* ``RefLib``: oracle/_ref/libfntrs_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src (oracle/Makefile) plus ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libfntrs_ref.so")

u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def _ensure(path: str, target: str):
    if not os.path.exists(path):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), target], check=True,
                       stdout=subprocess.DEVNULL)


def _a32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


class Oracle:
    def __init__(self):
        _ensure(ORACLE_SO, "oracle")
        L = self.lib = C.CDLL(ORACLE_SO)
        u32, i32, i64, u64 = C.c_uint32, C.c_int, C.c_int64, C.c_uint64
        for n in ("orc_add", "orc_sub", "orc_mul"):
            getattr(L, n).restype = u32
            getattr(L, n).argtypes = [u32, u32]
        L.orc_neg.restype = u32
        L.orc_neg.argtypes = [u32]
        L.orc_pow.restype = u32
        L.orc_pow.argtypes = [u32, u64]
        L.orc_inv.restype = u32
        L.orc_inv.argtypes = [u32]
        L.orc_root_of_unity.restype = i32
        L.orc_root_of_unity.argtypes = [u32, i32, C.POINTER(u32)]
        L.orc_fnt_forward.argtypes = [u32, u32p, u32p]
        L.orc_fnt_inverse.argtypes = [u32, u32p, u32p]
        L.orc_dif_forward.argtypes = [u32, u32p]
        L.orc_naive_dft.argtypes = [u32, u32, u32p, i32, u32p]
        L.orc_naive_dft.restype = None
        L.orc_poly_mul.argtypes = [u32p, u32, u32p, u32, u32p]
        L.orc_subproduct_root.argtypes = [u32p, u32, u32p]
        L.orc_eval_horner.restype = u32
        L.orc_eval_horner.argtypes = [u32p, u32, u32]
        L.orc_build_plan.argtypes = [u32, u32, u32p, u32p, u32p, C.POINTER(u32), C.c_void_p]
        L.orc_interpolate.argtypes = [u32, u32, u32p, u32p, u32, u32p, u32p, u32p]
        L.orc_lagrange.argtypes = [u32, u32p, u32p, u32p]
        L.orc_code_params.argtypes = [u32, u32, C.POINTER(u32)]
        L.orc_encode.argtypes = [u32, u32, u32p, u32p]
        L.orc_decode.argtypes = [u32, u32, u32, u32p, u32p, u32p]
        L.orc_encode_systematic.argtypes = [u32, u32, u32p, u32p]
        L.orc_decode_systematic.argtypes = [u32, u32, u32, u32p, u32p, u32p]
        L.orc_escape_split.restype = i64
        L.orc_escape_split.argtypes = [u32p, u64, u16p, u32p]
        L.orc_encode_stripes.restype = i64
        L.orc_encode_stripes.argtypes = [u32, u32, u32, u32, u16p, C.c_void_p, u64, u16p, u64p, u64]
        L.orc_decode_stripes.restype = i64
        L.orc_decode_stripes.argtypes = [u32, u32, u32, u32, u32, u32p, u32p, u16p, C.c_void_p, u64, u16p,
                                         u64p, u64]

    # field
    def add(self, a, b): return self.lib.orc_add(a, b)
    def sub(self, a, b): return self.lib.orc_sub(a, b)
    def mul(self, a, b): return self.lib.orc_mul(a, b)
    def neg(self, a): return self.lib.orc_neg(a)
    def pow(self, a, e): return self.lib.orc_pow(a, e)
    def inv(self, a): return self.lib.orc_inv(a)

    def root(self, n, inverse=False):
        r = C.c_uint32()
        st = self.lib.orc_root_of_unity(n, int(inverse), C.byref(r))
        return st, r.value

    def fnt(self, a, inverse=False):
        a = _a32(a)
        out = np.empty_like(a)
        st = (self.lib.orc_fnt_inverse if inverse else self.lib.orc_fnt_forward)(a.size, a, out)
        assert st == 0, st
        return out

    def naive_dft(self, root, a, inverse=False):
        a = _a32(a)
        out = np.empty_like(a)
        self.lib.orc_naive_dft(root, a.size, a, int(inverse), out)
        return out

    def build_plan(self, n, positions):
        pos = _a32(positions)
        k = pos.size
        a = np.zeros(k + 1, dtype=np.uint32)
        ap = np.zeros(k, dtype=np.uint32)
        ps = C.c_uint32()
        m = 1
        while m < 2 * k:
            m <<= 1
        af = np.zeros(m, dtype=np.uint32)
        st = self.lib.orc_build_plan(n, k, pos, a, ap, C.byref(ps), af.ctypes.data)
        return st, a, ap, ps.value, af[: ps.value]

    def interpolate(self, n, positions, values):
        st, a, ap, ps, af = self.build_plan(n, positions)
        assert st == 0
        out = np.zeros(len(positions), dtype=np.uint32)
        st = self.lib.orc_interpolate(n, len(positions), _a32(positions), ap, ps, _a32(af), _a32(values), out)
        return st, out

    def lagrange(self, xs, vs):
        xs, vs = _a32(xs), _a32(vs)
        out = np.zeros(xs.size, dtype=np.uint32)
        st = self.lib.orc_lagrange(xs.size, xs, vs, out)
        return st, out

    def encode(self, k, n, src):
        out = np.zeros(n, dtype=np.uint32)
        st = self.lib.orc_encode(k, n, _a32(src), out)
        return st, out

    def decode(self, k, n, pos, val):
        pos, val = _a32(pos), _a32(val)
        out = np.zeros(k, dtype=np.uint32)
        st = self.lib.orc_decode(k, n, pos.size, pos, val, out)
        return st, out

    def encode_systematic(self, k, n, src):
        out = np.zeros(n, dtype=np.uint32)
        st = self.lib.orc_encode_systematic(k, n, _a32(src), out)
        return st, out

    def decode_systematic(self, k, n, pos, val):
        pos, val = _a32(pos), _a32(val)
        out = np.zeros(k, dtype=np.uint32)
        st = self.lib.orc_decode_systematic(k, n, pos.size, pos, val, out)
        return st, out

    def encode_stripes(self, k, n, src, src_esc=None):
        S, kk, L = src.shape
        src = np.ascontiguousarray(src, dtype=np.uint16)
        out = np.zeros((S, n, L), dtype=np.uint16)
        cap = S * n * L + 1024  # worst case: every symbol escaped
        esc = np.zeros(cap, dtype=np.uint64)
        e = None if src_esc is None or len(src_esc) == 0 else np.ascontiguousarray(src_esc, dtype=np.uint64)
        ne = self.lib.orc_encode_stripes(k, n, S, L, src, None if e is None else e.ctypes.data,
                                         0 if e is None else e.size, out, esc, cap)
        assert ne >= 0, ne
        return out, esc[:ne]

    def decode_stripes(self, k, n, pats, sp, rx, rx_esc=None):
        S, kp, L = rx.shape
        rx = np.ascontiguousarray(rx, dtype=np.uint16)
        out = np.zeros((S, k, L), dtype=np.uint16)
        cap = S * k * L + 1024
        esc = np.zeros(cap, dtype=np.uint64)
        e = None if rx_esc is None or len(rx_esc) == 0 else np.ascontiguousarray(rx_esc, dtype=np.uint64)
        ne = self.lib.orc_decode_stripes(k, n, S, L, pats.shape[0], _a32(pats), _a32(sp), rx,
                                         None if e is None else e.ctypes.data, 0 if e is None else e.size,
                                         out, esc, cap)
        assert ne >= 0, ne
        return out, esc[:ne]


class RefLib:
    """The reference library itself (oracle/_ref)."""

    @staticmethod
    def available() -> bool:
        if not os.path.exists(REF_SO) and os.path.isdir("/root/reference/proj/src"):
            try:
                _ensure(REF_SO, "ref")
            except Exception:
                return False
        return os.path.exists(REF_SO)

    def __init__(self):
        L = self.lib = C.CDLL(REF_SO)
        u32, i32, i64, u64, uns = C.c_uint32, C.c_int, C.c_int64, C.c_uint64, C.c_uint
        L.ref_fnt_forward.argtypes = [u32, u32p, u32p]
        L.ref_fnt_inverse.argtypes = [u32, u32p, u32p]
        L.ref_encode.argtypes = [u32, u32, u32, u32p, u32p]
        L.ref_decode.argtypes = [u32, u32, u32, u32p, u32p, i32, u32p]
        L.ref_encode_systematic.argtypes = [u32, u32, u32, u32p, i32, u32p]
        L.ref_decode_systematic.argtypes = [u32, u32, u32, u32p, u32p, i32, u32p]
        L.ref_build_plan.argtypes = [u32, u32, u32p, u32p, C.POINTER(u32), u32p, C.POINTER(u32), C.c_void_p]
        L.ref_encode_stripes.restype = i64
        L.ref_encode_stripes.argtypes = [u32, u32, u32, u32, u16p, C.c_void_p, u64, u16p, u64p, u64, uns]
        L.ref_decode_stripes.restype = i64
        L.ref_decode_stripes.argtypes = [u32, u32, u32, u32, u32, u32p, u32p, u16p, C.c_void_p, u64, u16p,
                                         u64p, u64, i32, uns]
        L.ref_has_avx2.restype = i32
        L.ref_set_systematic.argtypes = [i32]
        L.ref_set_systematic.restype = None
        u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
        L.ref_encode_file.restype = i64
        L.ref_encode_file.argtypes = [u8p, u64, u32, u32, i32, u64, u8p, u64, u64p]
        L.ref_write_shard.restype = i64
        L.ref_write_shard.argtypes = [u64, u32, u32, u32, i32, u32p, u64, u8p, u64]
        L.ref_read_shard_status.restype = i32
        L.ref_read_shard_status.argtypes = [u8p, u64]

    def encode_file(self, data: bytes, k, n, systematic=True, chunk_id=0):
        """The reference CLI's encode over the library: (manifest bytes, [shard bytes])."""
        d = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
        words = (len(data) + 1) // 2
        S = (words + k - 1) // k
        cap = 64 + n * (64 + 2 * S) + 4 * (S * n // 1000 + 1024)
        out = np.zeros(cap, dtype=np.uint8)
        sizes = np.zeros(n + 1, dtype=np.uint64)
        tot = self.lib.ref_encode_file(np.ascontiguousarray(d), len(data), k, n, int(systematic), chunk_id, out, cap,
                                       sizes)
        assert tot >= 0, tot
        parts, pos = [], 0
        for sz in sizes:
            parts.append(out[pos:pos + int(sz)].tobytes())
            pos += int(sz)
        return parts[0], parts[1:]

    def write_shard(self, chunk_id, k, n, index, systematic, payload):
        p = _a32(payload)
        out = np.zeros(64 + 6 * max(p.size, 1), dtype=np.uint8)
        sz = self.lib.ref_write_shard(chunk_id, k, n, index, int(systematic), p, p.size, out, out.size)
        return (out[:sz].tobytes(), 0) if sz >= 0 else (b"", -sz)

    def read_shard_status(self, b: bytes) -> int:
        a = np.frombuffer(b, dtype=np.uint8) if b else np.zeros(1, np.uint8)
        return self.lib.ref_read_shard_status(np.ascontiguousarray(a), len(b))

    def set_systematic(self, on: bool):
        """Batched stripe loops run encode/decode_systematic instead of the non-systematic pair."""
        self.lib.ref_set_systematic(int(bool(on)))

    def fnt(self, a, inverse=False):
        a = _a32(a)
        out = np.empty_like(a)
        st = (self.lib.ref_fnt_inverse if inverse else self.lib.ref_fnt_forward)(a.size, a, out)
        return st, out

    def encode(self, k, n, src):
        src = _a32(src)
        out = np.zeros(max(n, 1), dtype=np.uint32)
        st = self.lib.ref_encode(k, n, src.size, src, out)
        return st, out

    def decode(self, k, n, pos, val, path=0):
        pos, val = _a32(pos), _a32(val)
        out = np.zeros(max(k, 1), dtype=np.uint32)
        st = self.lib.ref_decode(k, n, pos.size, pos, val, path, out)
        return st, out

    def encode_systematic(self, k, n, src, path=0):
        src = _a32(src)
        out = np.zeros(max(n, 1), dtype=np.uint32)
        st = self.lib.ref_encode_systematic(k, n, src.size, src, path, out)
        return st, out

    def decode_systematic(self, k, n, pos, val, path=0):
        pos, val = _a32(pos), _a32(val)
        out = np.zeros(max(k, 1), dtype=np.uint32)
        st = self.lib.ref_decode_systematic(k, n, pos.size, pos, val, path, out)
        return st, out

    def build_plan(self, n, positions):
        pos = _a32(positions)
        k = pos.size
        a = np.zeros(k + 1, dtype=np.uint32)
        alen = C.c_uint32()
        ap = np.zeros(k, dtype=np.uint32)
        ps = C.c_uint32()
        m = 1
        while m < 2 * k:
            m <<= 1
        af = np.zeros(m, dtype=np.uint32)
        st = self.lib.ref_build_plan(n, k, pos, a, C.byref(alen), ap, C.byref(ps), af.ctypes.data)
        return st, a[: alen.value], ap, ps.value, af[: ps.value]

    def encode_stripes(self, k, n, src, threads=1, src_esc=None):
        S, kk, L = src.shape
        src = np.ascontiguousarray(src, dtype=np.uint16)
        out = np.zeros((S, n, L), dtype=np.uint16)
        e = None if src_esc is None or len(src_esc) == 0 else np.ascontiguousarray(src_esc, dtype=np.uint64)
        # escapes are rare (~1 per 65537 symbols); grow to the worst case only on overflow (-11)
        for cap in (S * n * L // 4096 + 4096, S * n * L + 1024):
            esc = np.zeros(cap, dtype=np.uint64)
            ne = self.lib.ref_encode_stripes(k, n, S, L, src, None if e is None else e.ctypes.data,
                                             0 if e is None else e.size, out, esc, cap, threads)
            if ne != -11:
                break
        assert ne >= 0, ne
        return out, esc[:ne]

    def decode_stripes(self, k, n, pats, sp, rx, rx_esc=None, path=0, threads=1):
        S, kp, L = rx.shape
        rx = np.ascontiguousarray(rx, dtype=np.uint16)
        out = np.zeros((S, k, L), dtype=np.uint16)
        e = None if rx_esc is None or len(rx_esc) == 0 else np.ascontiguousarray(rx_esc, dtype=np.uint64)
        for cap in (S * k * L // 4096 + 4096, S * k * L + 1024):
            esc = np.zeros(cap, dtype=np.uint64)
            ne = self.lib.ref_decode_stripes(k, n, S, L, pats.shape[0], _a32(pats), _a32(sp), rx,
                                             None if e is None else e.ctypes.data, 0 if e is None else e.size,
                                             out, esc, cap, path, threads)
            if ne != -11:
                break
        assert ne >= 0, ne
        return out, esc[:ne]


def gather_received(enc: np.ndarray, enc_esc: np.ndarray, pats: np.ndarray, sp: np.ndarray):
    """Received packets rx[s, i] = enc[s, pats[sp[s], i]] and their escapes (host, numpy)."""
    S, n, L = enc.shape
    k = pats.shape[1]
    rows = pats[sp]                                   # [S, k]
    rx = enc[np.arange(S)[:, None], rows]             # [S, k, L]
    if enc_esc.size == 0:
        return rx, np.zeros(0, dtype=np.uint64)
    # map escape keys (s*n + pos)*L + col -> (s*k + i)*L + col
    e = enc_esc.astype(np.int64)
    row, col = e // L, e % L
    s, pos = row // n, row % n
    inv = np.full((S, n), -1, dtype=np.int64)
    inv[np.arange(S)[:, None], rows] = np.arange(k)[None, :]
    i = inv[s, pos]
    keep = i >= 0
    out = ((s[keep] * k + i[keep]) * L + col[keep]).astype(np.uint64)
    return rx, np.sort(out)
