"""B200-native MASK hot path: multilevel Lloyd k-means index build + batched k-NN query.

MASK = "Multilevel Approximate Similarity search with k-means" (arXiv 2208.02734).  The
compute lives in ``libmask.so`` (hand-written sm_100a CUDA behind the C-ABI of
``include/mask.h``); this package is the argument-marshalling binding plus host-side
sharding helpers.  Importing it does not require a GPU; calling it does (no CPU fallback).
"""
from . import _lib
from .api import (Comm, Csr, Index, assign, build, build_grouped, collective_count, device_ok, grouped_depth,
                  kernel_launches, matrix, merge, route, seeded_init, update)
from ._lib import (
    MASK_BORROW_DATA,
    MASK_FORCE_SIMT,
    MASK_NO_FIXUP,
    MASK_NO_FUSED,
    MASK_NO_SORT,
    MASK_TIME_ASSIGN,
    MASK_TIME_KERNELS,
    MASK_TRACE_PASSES,
    MASK_CSR_TC,
    MASK_TC_TF32,
    MASK_VALIDATE_FINITE,
    MaskError,
)
from .shard import query_range, row_range

__all__ = [
    "Comm", "Csr", "Index", "assign", "build", "build_grouped", "grouped_depth", "device_ok", "kernel_launches", "matrix",
    "update", "route", "merge", "collective_count", "seeded_init", "row_range",
    "query_range", "MaskError", "MASK_BORROW_DATA", "MASK_FORCE_SIMT", "MASK_NO_FIXUP",
    "MASK_VALIDATE_FINITE", "MASK_TIME_KERNELS", "MASK_TIME_ASSIGN", "MASK_NO_SORT", "MASK_NO_FUSED",
    "MASK_TRACE_PASSES",
    "MASK_CSR_TC",
    "MASK_TC_TF32",
]
