"""B200-native lip-sync hot path of the lipstream reference (arXiv 2512.18318).

The compute lives in liblsg.so (hand-written sm_100a CUDA behind the C ABI
in include/lsg.h); this package is the Python mirror of the reference's
operator API over that ABI.  There is no CPU fallback.
"""
from ._lib import InvalidArgument, LogicError, LsgError, header_symbols, lib  # noqa: F401

__all__ = ["InvalidArgument", "LogicError", "LsgError", "header_symbols", "lib"]
