"""B200-native (sm_100a) Lie-closure hot path of arXiv 2506.01120 (liecl).

The product is libliecl_b200.so (C-ABI: include/liecl_b200.h); `liecl` is the
Python mirror of the reference's closure interface over it.
"""
from . import liecl, native, workloads  # noqa: F401

__all__ = ["liecl", "native", "workloads"]
