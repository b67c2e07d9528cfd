"""B200-native hot path of Adaptive SGD (arXiv 2110.07029).

The product is libadasgd.so (C-ABI in include/adasgd.h: CUDA kernels for
sm_100a, NCCL, the host scheduler).  This package is its thin Python binding:
``api`` (Replica, group_merge), ``sched`` (routing, Alg. 1/2), ``driver``
(the mega-batch loop).  It never imports ``oracle``.
"""
from . import _lib  # noqa: F401

__all__ = ["api", "sched", "driver"]
