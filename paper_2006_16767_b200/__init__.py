"""B200-native adaptive SpMV/SpMSpV (arXiv 2006.16767 hot path).

The product is ``libadaspmv_cuda.so`` (hand-written sm_100a kernels behind the
C-ABI in ``include/adaspmv_cuda.h``); :mod:`.adaspmv` mirrors the reference's
``namespace adaspmv`` API over it for Python callers, tests and the bench.
"""
from . import adaspmv  # noqa: F401

__all__ = ["adaspmv"]
