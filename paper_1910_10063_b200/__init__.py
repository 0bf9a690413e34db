"""B200-native skew-aware repositioning index (arXiv 1910.10063) and the
operators it accelerates: FK-join gather, group-by, selection.

The compute path is libskx.so (hand-written sm_100a CUDA behind the C-ABI in
include/skx.h); ``paper_1910_10063_b200.skewdx`` mirrors the reference's
operator API over it and ``paper_1910_10063_b200.dist`` shards it across GPUs.
"""
from .errors import DomainViolation, Error, FormatError, InvalidArgument, IoError, NativeUnavailable

__version__ = "0.1.0"

__all__ = ["DomainViolation", "Error", "FormatError", "InvalidArgument", "IoError",
           "NativeUnavailable"]
