"""fntrs_b200 -- B200-native batched FNT Reed-Solomon codec over GF(65537).

Drop-in for the non-systematic encode/decode path of the reference `fntrs`
(arXiv 0907.1788; /root/reference/proj/include/fntrs/codec.hpp). The compute
lives in libfntrs_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/fntrs_gpu.h); this package is the Python host mirror of the
reference interface plus the batched API. See DESIGN.md.
"""
from .codec import (  # noqa: F401
    Codec, CodeParams, Path, Plans, Symbol, decode_nonsystematic, decode_systematic, encode_nonsystematic,
    encode_systematic,
    Error, ZeroInverse, InvalidTransformSize, SizeMismatch, ProductTooLarge, DuplicatePoint,
    DuplicatePosition, PositionOutOfRange, TooFewPositions, NotEnoughSymbols, TooManyEscapes,
    BadMagic, BadVersion, TruncatedShard, MalformedEscapes, MalformedHeader, LengthMismatch, NotEnoughShards,
    UnsupportedShape, default_escape_capacity, escapes_to_numpy,
)
from . import workload  # noqa: F401
from . import shards  # noqa: F401
from .shards import decode_file, encode_file  # noqa: F401

__version__ = "0.1.0"
