"""ctypes binding of libfntrs_b200.so (the C ABI declared in include/fntrs_gpu.h).

This is the reference-side FFI stub a Python caller would write against the
C ABI. Loading fails loudly when the library has not
been built: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfntrs_b200.so")

_u32 = C.c_uint32
_u64 = C.c_uint64
_int = C.c_int
_vp = C.c_void_p
_pu32 = C.POINTER(C.c_uint32)

# (name, restype, argtypes) for every symbol include/fntrs_gpu.h declares
SIGNATURES = [
    ("fntrs_gpu_create", _int, [_int, C.POINTER(_vp)]),
    ("fntrs_gpu_destroy", _int, [_vp]),
    ("fntrs_gpu_status_string", C.c_char_p, [_int]),
    ("fntrs_gpu_last_error", C.c_char_p, [_vp]),
    ("fntrs_gpu_device", _int, [_vp]),
    ("fntrs_gpu_version", C.c_char_p, []),
    ("fntrs_gpu_code_params", _int, [_u32, _u32, _pu32]),
    ("fntrs_gpu_encode", _int, [_vp, _u32, _u32, _u32, _u32, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    ("fntrs_gpu_plans_create", _int, [_vp, _u32, _u32, _u32, _u32, _vp, C.POINTER(_vp), _vp]),
    ("fntrs_gpu_plans_destroy", _int, [_vp]),
    ("fntrs_gpu_plans_count", _u32, [_vp]),
    ("fntrs_gpu_plans_export", _int, [_vp, _vp, _u32, _vp, _vp, _pu32, _vp]),
    ("fntrs_gpu_decode", _int, [_vp, _vp, _u32, _u32, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    ("fntrs_gpu_encode_systematic", _int, [_vp, _u32, _u32, _u32, _u32, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    ("fntrs_gpu_decode_systematic", _int, [_vp, _vp, _u32, _u32, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp]),
    ("fntrs_gpu_symbolize", _int, [_vp, _vp, _u64, _u32, _u32, _vp, _vp]),
    ("fntrs_gpu_desymbolize", _int, [_vp, _vp, _u32, _u32, _u64, _vp, _vp]),
    ("fntrs_gpu_words_to_be", _int, [_vp, _vp, _u32, _u32, _u32, _vp, _u64, _vp]),
    ("fntrs_gpu_be_to_words", _int, [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp]),
    ("fntrs_gpu_fnt", _int, [_vp, _u32, _int, _u32, _vp, _vp, _vp]),
    ("fntrs_gpu_launch_count", _u64, [_vp]),
    ("fntrs_gpu_set_fast_path", _int, [_vp, _int]),
    ("fntrs_gpu_fill_symbols", _int, [_u64, _u64, _u64, _vp, _vp]),
    ("fntrs_gpu_transform_counts", _int, [_vp, C.POINTER(_u64)]),
    ("fntrs_gpu_naive_dft", _int, [_vp, _u32, _int, _u32, _vp, _vp, _vp]),
    ("fntrs_gpu_transform_tables", _int, [_vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_poly_products", _int, [_vp, _u32, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_subproduct_tree_layout", _int, [_u32, _pu32, _pu32, _u32, _pu32, C.POINTER(_u64), C.POINTER(_u64)]),
    ("fntrs_gpu_subproduct_tree", _int, [_vp, _u32, _vp, _vp, _vp]),
    ("fntrs_gpu_lagrange", _int, [_vp, _u32, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_chirp_table", _int, [_vp, _u32, _u32, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_geom_eval", _int, [_vp, _u32, _u32, _vp, _u32, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_geom_eval_negative", _int, [_vp, _u32, _u32, _vp, _u32, _vp, _vp, _vp, _vp]),
    ("fntrs_gpu_poly_derivative", _int, [_vp, _u32, _vp, _vp, _vp]),
    ("fntrs_gpu_poly_eval", _int, [_vp, _u32, _vp, _u32, _vp, _vp]),
]

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} not found: build it with `make lib` (or __graft_entry__.build()); "
            "the codec has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return [s[0] for s in SIGNATURES]
