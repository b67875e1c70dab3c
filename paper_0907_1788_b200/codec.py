"""Python host API mirroring the reference codec interface, executed on a B200.

Two layers, both calling the C ABI (include/fntrs_gpu.h) through ctypes:

* The reference's per-codeword interface (proj/include/fntrs/codec.hpp:15-51)
  -- ``CodeParams.make``, ``Symbol``, ``Path``, ``encode_nonsystematic``,
  ``decode_nonsystematic`` and the exception classes of
  proj/include/fntrs/errors.hpp:9-38 -- with the same argument meaning, results
  and error behaviour. Each call is one codeword (batch of 1).
* ``Codec``: the batched interface the throughput path uses -- packet-major
  uint16 stripes resident in device memory, escape lists, per-pattern plans.

torch supplies device memory and streams only (plumbing); all codec
arithmetic runs in libfntrs_b200.so. No CPU fallback exists: without a CUDA
device every call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib

# ---------------------------------------------------------------- errors ----


class Error(RuntimeError):
    """fntrs::Error"""


def _mk(name):
    return type(name, (Error,), {"__doc__": f"fntrs::{name}"})


ZeroInverse = _mk("ZeroInverse")
InvalidTransformSize = _mk("InvalidTransformSize")
SizeMismatch = _mk("SizeMismatch")
ProductTooLarge = _mk("ProductTooLarge")
DuplicatePoint = _mk("DuplicatePoint")
DuplicatePosition = _mk("DuplicatePosition")
PositionOutOfRange = _mk("PositionOutOfRange")
TooFewPositions = _mk("TooFewPositions")
NotEnoughSymbols = _mk("NotEnoughSymbols")
TooManyEscapes = _mk("TooManyEscapes")
BadMagic = _mk("BadMagic")
BadVersion = _mk("BadVersion")
TruncatedShard = _mk("TruncatedShard")
MalformedEscapes = _mk("MalformedEscapes")
MalformedHeader = _mk("MalformedHeader")
LengthMismatch = _mk("LengthMismatch")
NotEnoughShards = _mk("NotEnoughShards")

STATUS_CLASSES = {
    1: Error, 2: ZeroInverse, 3: InvalidTransformSize, 4: SizeMismatch, 5: ProductTooLarge,
    6: DuplicatePoint, 7: DuplicatePosition, 8: PositionOutOfRange, 9: TooFewPositions,
    10: NotEnoughSymbols, 11: TooManyEscapes, 12: BadMagic, 13: BadVersion, 14: TruncatedShard,
    15: MalformedEscapes, 16: MalformedHeader, 17: LengthMismatch, 18: NotEnoughShards,
}


class UnsupportedShape(Error):
    """Shape outside this build (FNTRS_E_UNSUPPORTED)."""


def raise_status(status: int, detail: str = "") -> None:
    if status == 0:
        return
    lib = _lib.load()
    name = lib.fntrs_gpu_status_string(status).decode()
    if status == 101:
        raise UnsupportedShape(f"{name}: {detail}")
    raise STATUS_CLASSES.get(status, Error)(f"{name}: {detail}")


# ------------------------------------------------------------ batched API ----

def _torch():
    import torch  # plumbing: device memory and streams
    return torch


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream) -> int | None:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Plans:
    """Device-resident decode plans for a batch of erasure patterns."""

    def __init__(self, codec: "Codec", handle: C.c_void_p, k: int, n: int, kp: int, npatterns: int):
        self._codec, self.handle, self.k, self.n, self.kp, self.npatterns = codec, handle, k, n, kp, npatterns

    def export(self, pattern: int):
        """DecodePlan fields (interp.hpp:18-32): (a, aprime_inv, product_size, a_fnt)."""
        lib = _lib.load()
        a = np.zeros(self.kp + 1, dtype=np.uint32)
        ap = np.zeros(self.kp, dtype=np.uint32)
        ps = C.c_uint32(0)
        m = 1
        while m < 2 * self.k:
            m <<= 1
        af = np.zeros(max(m, 1), dtype=np.uint32)
        st = lib.fntrs_gpu_plans_export(self._codec.ctx, self.handle, pattern, a.ctypes.data, ap.ctypes.data,
                                        C.byref(ps), af.ctypes.data)
        self._codec._check(st)
        return a, ap, int(ps.value), af[: ps.value]

    def close(self):
        if self.handle:
            _lib.load().fntrs_gpu_plans_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Codec:
    """Batched non-systematic FNT codec on one CUDA device (one fntrs_ctx)."""

    def __init__(self, device: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise Error("fntrs: no CUDA device (the codec has no CPU fallback)")
        lib = _lib.load()
        self.device = device
        self.ctx = C.c_void_p()
        torch.cuda.init()
        with torch.cuda.device(device):
            st = lib.fntrs_gpu_create(device, C.byref(self.ctx))
        if st:
            raise_status(st, "fntrs_gpu_create failed")
        self._counts = torch.zeros(4, dtype=torch.int64, device=f"cuda:{device}")

    def _check(self, st: int):
        if st:
            raise_status(st, _lib.load().fntrs_gpu_last_error(self.ctx).decode())

    @property
    def launches(self) -> int:
        return int(_lib.load().fntrs_gpu_launch_count(self.ctx))

    def close(self):
        if self.ctx:
            _lib.load().fntrs_gpu_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- encode -----------------------------------------------------------
    def encode(self, k: int, n: int, src, src_esc=None, out=None, esc_out=None, esc_cap: int | None = None,
               count=None, stream=None, systematic: bool = False):
        """src: int16 CUDA tensor [S, k, L] (uint16 bits). Returns (out [S, n, L], esc, count)."""
        torch = _torch()
        S, kk, L = src.shape
        if kk != k:
            raise SizeMismatch(f"encode: got {kk} source packets for k = {k}")
        dev = src.device
        if out is None:
            out = torch.empty((S, n, L), dtype=torch.int16, device=dev)
        if esc_cap is None:
            esc_cap = default_escape_capacity(S * n * L)
        if esc_out is None:
            esc_out = torch.empty(max(esc_cap, 1), dtype=torch.int64, device=dev)
        if count is None:
            count = self._counts[0:1]
        ne = 0 if src_esc is None else src_esc.numel()
        fn = _lib.load().fntrs_gpu_encode_systematic if systematic else _lib.load().fntrs_gpu_encode
        st = fn(self.ctx, k, n, S, L, _ptr(src), _ptr(src_esc) if ne else None, ne,
                _ptr(out), _ptr(esc_out), esc_cap, _ptr(count), _stream_ptr(stream))
        self._check(st)
        return out, esc_out, count

    def encode_systematic(self, k: int, n: int, src, src_esc=None, out=None, esc_out=None,
                          esc_cap: int | None = None, count=None, stream=None):
        """codec::encode_systematic batched (codec.cpp:151-161): rows 0..k-1 of every
        output stripe are the source; rows k..n-1 the parity. Synchronises `stream` once."""
        return self.encode(k, n, src, src_esc, out, esc_out, esc_cap, count, stream, systematic=True)

    # -- plans ------------------------------------------------------------
    def plans(self, k: int, n: int, positions, stream=None) -> Plans:
        """positions: host [P, kp] uint32 received positions per pattern (a numpy
        array, or a pinned CPU torch tensor for a fully asynchronous upload)."""
        if hasattr(positions, "data_ptr"):
            pos_t = positions if positions.dim() == 2 else positions[None, :]
            P, kp = pos_t.shape
            ptr, keep = pos_t.data_ptr(), pos_t
        else:
            pos = np.ascontiguousarray(positions, dtype=np.uint32)
            if pos.ndim == 1:
                pos = pos[None, :]
            P, kp = pos.shape
            ptr, keep = pos.ctypes.data, pos
        h = C.c_void_p()
        st = _lib.load().fntrs_gpu_plans_create(self.ctx, k, n, kp, P, ptr, C.byref(h), _stream_ptr(stream))
        del keep
        self._check(st)
        return Plans(self, h, k, n, kp, P)

    # -- decode -----------------------------------------------------------
    def decode(self, plans: Plans, stripe_pattern, rx, rx_esc=None, out=None, esc_out=None,
               esc_cap: int | None = None, count=None, stream=None, systematic: bool = False):
        """rx: int16 CUDA tensor [S, kp, L]; stripe_pattern: int32 CUDA tensor [S]."""
        torch = _torch()
        S, kp, L = rx.shape
        if kp != plans.kp:
            raise SizeMismatch(f"decode: got {kp} received packets per stripe, plan has {plans.kp}")
        if out is None:
            out = torch.empty((S, plans.k, L), dtype=torch.int16, device=rx.device)
        if esc_cap is None:
            esc_cap = default_escape_capacity(S * plans.k * L)
        if esc_out is None:
            esc_out = torch.empty(max(esc_cap, 1), dtype=torch.int64, device=rx.device)
        if count is None:
            count = self._counts[1:2]
        ne = 0 if rx_esc is None else rx_esc.numel()
        fn = _lib.load().fntrs_gpu_decode_systematic if systematic else _lib.load().fntrs_gpu_decode
        st = fn(self.ctx, plans.handle, S, L, _ptr(stripe_pattern), _ptr(rx), _ptr(rx_esc) if ne else None, ne,
                _ptr(out), _ptr(esc_out), esc_cap, _ptr(count), _stream_ptr(stream))
        self._check(st)
        return out, esc_out, count

    def decode_systematic(self, plans: Plans, stripe_pattern, rx, rx_esc=None, out=None, esc_out=None,
                          esc_cap: int | None = None, count=None, stream=None):
        """codec::decode_systematic batched (codec.cpp:163-196): the source rows
        0..k-1 of every stripe, rebuilt from the packets the plan names.
        Synchronises `stream` once."""
        return self.decode(plans, stripe_pattern, rx, rx_esc, out, esc_out, esc_cap, count, stream,
                           systematic=True)

    # -- transform --------------------------------------------------------
    def fnt(self, x, inverse: bool = False, stream=None):
        """Columns of an int32 CUDA tensor [m, L] (canonical values); natural order."""
        torch = _torch()
        m, L = x.shape
        out = torch.empty_like(x)
        st = _lib.load().fntrs_gpu_fnt(self.ctx, m, int(inverse), L, _ptr(x), _ptr(out), _stream_ptr(stream))
        self._check(st)
        return out


def default_escape_capacity(symbols: int) -> int:
    """Escapes occur at rate 1/65537 per symbol; keep a wide margin."""
    expected = symbols / 65537.0
    return int(4 * expected + 64 * np.sqrt(expected + 1) + 256)


def escapes_to_numpy(esc, count) -> np.ndarray:
    n = int(count.item()) if hasattr(count, "item") else int(count)
    if n > esc.numel():
        raise TooManyEscapes(f"{n} escapes exceed the capacity {esc.numel()}")
    return esc[:n].cpu().numpy().view(np.uint64)


# ------------------------------------------- reference per-codeword API ----

@dataclass(frozen=True)
class CodeParams:
    """codec::CodeParams (codec.hpp:15-23)."""
    k: int
    n: int
    n_domain: int
    systematic: bool = True

    @staticmethod
    def make(k: int, n: int, systematic: bool = True) -> "CodeParams":
        nd = C.c_uint32(0)
        if not (0 <= k < 2**32 and 0 <= n < 2**32) or _lib.load().fntrs_gpu_code_params(k, n, C.byref(nd)):
            raise SizeMismatch(f"code parameters need 1 <= k <= n <= 65536, got k = {k}, n = {n}")
        return CodeParams(k, n, int(nd.value), systematic)


@dataclass(frozen=True)
class Symbol:
    position: int
    value: int


class Path(enum.Enum):
    Auto = 0
    Fast = 1
    Direct = 2


DIRECT_PATH_MAX_K = 256

_shared_lock = threading.Lock()
_shared: dict = {}


def _shared_codec(device: int = 0) -> Codec:
    with _shared_lock:
        c = _shared.get(device)
        if c is None:
            c = _shared[device] = Codec(device)
            c._plan_lru = OrderedDict()
        return c


def _split(values) -> tuple[np.ndarray, np.ndarray]:
    v = np.asarray(values, dtype=np.int64)
    if v.size and (v.min() < 0 or v.max() > 65536):
        raise SizeMismatch("value outside the field")
    esc = np.nonzero(v == 65536)[0].astype(np.int64)
    return np.where(v == 65536, 0, v).astype(np.uint16), esc


def _join(words: np.ndarray, esc: np.ndarray) -> list[int]:
    out = words.astype(np.int64)
    out[esc.astype(np.int64)] = 65536
    return [int(x) for x in out]


def encode_nonsystematic(params: CodeParams, source) -> list[int]:
    """codec::encode_nonsystematic (codec.cpp:124-131): output j is s(r^j), j < n."""
    return _encode_one(params, source, systematic=False)


def _encode_one(params: CodeParams, source, systematic: bool) -> list[int]:
    torch = _torch()
    src = list(source)
    if len(src) != params.k:
        raise SizeMismatch(f"encode: got {len(src)} source symbols for k = {params.k}")
    c = _shared_codec()
    words, esc = _split(src)
    with _shared_lock:
        dev = f"cuda:{c.device}"
        t = torch.from_numpy(words.view(np.int16).reshape(1, params.k, 1)).to(dev)
        te = torch.from_numpy(esc).to(dev) if esc.size else None
        out, oe, cnt = c.encode(params.k, params.n, t, te, esc_cap=params.n, systematic=systematic)
        return _join(out.cpu().numpy().reshape(-1).view(np.uint16), escapes_to_numpy(oe, cnt))


def _sorted_received(params: CodeParams, received) -> list[tuple[int, int]]:
    """sorted_received (codec.cpp:32-48): range check, sort, duplicates, count."""
    rx = [(int(s.position), int(s.value)) for s in received]
    for p, _ in rx:
        if p >= params.n:
            raise PositionOutOfRange(f"received position {p} not below n = {params.n}")
    rx.sort(key=lambda t: t[0])
    for i in range(1, len(rx)):
        if rx[i][0] == rx[i - 1][0]:
            raise DuplicatePosition(f"received position {rx[i][0]} repeats")
    if len(rx) < params.k:
        raise NotEnoughSymbols(f"have {len(rx)} symbols, need {params.k}")
    return rx


def decode_nonsystematic(params: CodeParams, received, path: Path = Path.Auto) -> list[int]:
    """codec::decode_nonsystematic (codec.cpp:133-149) with sorted_received (:32-48)."""
    rx = _sorted_received(params, received)
    full = params.n == params.n_domain and len(rx) == params.n
    return _decode_one(params, rx, params.n if full else params.k, systematic=False)


def decode_systematic(params: CodeParams, received, path: Path = Path.Auto) -> list[int]:
    """codec::decode_systematic (codec.cpp:163-196): interpolate the k lowest
    received symbols and evaluate at positions 0..k-1. When those k lowest are
    0..k-1 the kernels reproduce them exactly (the reference's verbatim copy)."""
    return _decode_one(params, _sorted_received(params, received), params.k, systematic=True)


def encode_systematic(params: CodeParams, source, path: Path = Path.Auto) -> list[int]:
    """codec::encode_systematic (codec.cpp:151-161): outputs 0..k-1 are the source."""
    return _encode_one(params, source, systematic=True)


def _decode_one(params: CodeParams, rx, kp: int, systematic: bool) -> list[int]:
    torch = _torch()
    pos = np.array([p for p, _ in rx[:kp]], dtype=np.uint32)
    vals = [v for _, v in rx[:kp]]
    c = _shared_codec()
    with _shared_lock:
        key = (params.k, params.n, pos.tobytes())
        plan = c._plan_lru.get(key)
        if plan is None:
            plan = c.plans(params.k, params.n, pos[None, :])
            c._plan_lru[key] = plan
            if len(c._plan_lru) > 16:  # interp::plan_for LRU capacity (interp.cpp:75)
                torch.cuda.synchronize(c.device)
                c._plan_lru.popitem(last=False)[1].close()
        else:
            c._plan_lru.move_to_end(key)
        dev = f"cuda:{c.device}"
        words, esc = _split(vals)
        t = torch.from_numpy(words.view(np.int16).reshape(1, kp, 1)).to(dev)
        te = torch.from_numpy(esc).to(dev) if esc.size else None
        sp = torch.zeros(1, dtype=torch.int32, device=dev)
        out, oe, cnt = c.decode(plan, sp, t, te, esc_cap=params.k, systematic=systematic)
        return _join(out.cpu().numpy().reshape(-1).view(np.uint16), escapes_to_numpy(oe, cnt))
