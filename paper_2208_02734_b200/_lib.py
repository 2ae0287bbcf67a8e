"""ctypes declarations of include/mask.h (argument marshalling only).

The CUDA library ``libmask.so`` is built in-tree by ``paper_2208_02734_b200.build``.  If it
is missing this module raises — there is no CPU fallback anywhere in the package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmask.so")

MASK_OK = 0
STATUS = {
    0: "MASK_OK",
    -1: "MASK_ERR_ARG",
    -2: "MASK_ERR_NONFINITE",
    -3: "MASK_ERR_OOM",
    -4: "MASK_ERR_CUDA",
    -5: "MASK_ERR_NCCL",
    -6: "MASK_ERR_UNSUPPORTED",
}
MASK_DENSE_F32, MASK_CSR_F32 = 0, 1
MASK_MEM_DEVICE, MASK_MEM_HOST = 0, 1
MASK_EMPTY_KEEP = 0
MASK_EMPTY_FARTHEST = 1
MASK_VALIDATE_FINITE = 1 << 0
MASK_BORROW_DATA = 1 << 1
MASK_FORCE_SIMT = 1 << 2
MASK_NO_FIXUP = 1 << 3
MASK_TIME_KERNELS = 1 << 5
MASK_NO_SORT = 1 << 6
MASK_NO_FUSED = 1 << 7
MASK_TIME_ASSIGN = 1 << 8
MASK_NO_PARTITION_COPY = 1 << 9
MASK_TRACE_PASSES = 1 << 10
MASK_CSR_TC = 1 << 11
MASK_TC_TF32 = 1 << 12
MASK_RANGE_PAPER, MASK_RANGE_COVER = 0, 1
T_ASSIGN, T_FIXUP, T_UPDATE, T_FINALIZE = 0, 1, 2, 3

# every symbol include/mask.h declares (checked by tests/test_boundary.py)
EXPORTS = [
    "mask_abi_version", "mask_last_error", "mask_device_ok", "mask_comm_unique_id", "mask_comm_init",
    "mask_comm_free", "mask_build", "mask_query", "mask_free", "mask_assign", "mask_update",
    "mask_num_levels", "mask_level_info", "mask_get_prototypes", "mask_get_labels",
    "mask_get_children", "mask_get_trace", "mask_kernel_launches", "mask_get_timing",
    "mask_grouped_depth", "mask_build_grouped", "mask_range_query", "mask_insert",
    "mask_top_prototypes", "mask_route", "mask_query_routed", "mask_merge", "mask_collective_count",
    "mask_seeded_init", "mask_debug_fail_alloc", "mask_get_displacement", "mask_get_pass",
    "mask_comm_init_host", "mask_split", "mask_relocate",
]


class MaskMatrix(C.Structure):
    _fields_ = [
        ("format", C.c_int32),
        ("memory", C.c_int32),
        ("dim", C.c_int32),
        ("_pad", C.c_int32),
        ("rows", C.c_int64),
        ("n_global", C.c_int64),
        ("row_offset", C.c_int64),
        ("values", C.c_void_p),
        ("row_ptr", C.c_void_p),
        ("col_idx", C.c_void_p),
        ("nnz", C.c_int64),
    ]


HOST_COLL = C.CFUNCTYPE(C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p)
MASK_COLL_ALLREDUCE, MASK_COLL_BROADCAST, MASK_COLL_ALLGATHER = 0, 1, 2
MASK_COLL_SUM, MASK_COLL_MAX = 0, 1

ITER_CB = C.CFUNCTYPE(None, C.c_int32, C.c_int32, C.POINTER(C.c_float), C.c_int64, C.c_int32,
                      C.POINTER(C.c_int32), C.c_int64, C.c_void_p)


class MaskBuildParams(C.Structure):
    _fields_ = [
        ("num_levels", C.c_int32),
        ("max_iters", C.c_int32),
        ("k", C.POINTER(C.c_int64)),
        ("tol", C.c_double),
        ("seed", C.c_uint64),
        ("init_idx", C.POINTER(C.POINTER(C.c_int64))),
        ("empty_policy", C.c_int32),
        ("flags", C.c_int32),
        ("iter_cb", ITER_CB),
        ("iter_cb_user", C.c_void_p),
    ]


class MaskSplitParams(C.Structure):
    _fields_ = [
        ("threshold", C.c_int64),
        ("max_iters", C.c_int32),
        ("flags", C.c_int32),
        ("seed", C.c_uint64),
    ]


class MaskGroupedParams(C.Structure):
    _fields_ = [
        ("length_group", C.c_int32),
        ("n_centroids", C.c_int32),
        ("max_iters", C.c_int32),
        ("flags", C.c_int32),
        ("perm", C.POINTER(C.c_int64)),
    ]


class MaskError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lock = threading.Lock()
_lib = None


def load():
    """Load libmask.so (raises if it was not built: no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2208_02734_b200.buildlib` "
                "(the package has no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        sig = {
            "mask_abi_version": (i32, []),
            "mask_last_error": (C.c_char_p, []),
            "mask_device_ok": (i32, []),
            "mask_comm_unique_id": (i32, [P]),
            "mask_comm_init": (i32, [P, i32, i32, C.POINTER(P)]),
            "mask_comm_free": (None, [P]),
            "mask_build": (i32, [C.POINTER(MaskMatrix), C.POINTER(MaskBuildParams), P, P, C.POINTER(P)]),
            "mask_query": (i32, [P, C.POINTER(MaskMatrix), i32, i32, P, P, P]),
            "mask_free": (None, [P]),
            "mask_assign": (i32, [C.POINTER(MaskMatrix), P, i64, i32, P, P, C.POINTER(i64), P]),
            "mask_update": (i32, [C.POINTER(MaskMatrix), P, i64, P, P, P, C.POINTER(C.c_double), P]),
            "mask_num_levels": (i32, [P]),
            "mask_level_info": (i32, [P, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32),
                                      C.POINTER(i32), C.POINTER(i32)]),
            "mask_get_prototypes": (i32, [P, i32, P]),
            "mask_get_labels": (i32, [P, i32, P]),
            "mask_get_children": (i32, [P, i32, P, P]),
            "mask_get_trace": (i32, [P, i32, P, P, P, i32]),
            "mask_kernel_launches": (i64, []),
            "mask_get_timing": (i32, [P, i32, P, i32]),
            "mask_grouped_depth": (i32, [i64, i32, i32, P, i32]),
            "mask_build_grouped": (i32, [C.POINTER(MaskMatrix), C.POINTER(MaskGroupedParams), P, C.POINTER(P)]),
            "mask_relocate": (i32, [P, P, P, P, i32, P, P, C.POINTER(i64), P]),
            "mask_range_query": (i32, [P, C.POINTER(MaskMatrix), P, i32, i64, P, P, P, C.POINTER(i64), P]),
            "mask_insert": (i32, [P, C.POINTER(MaskMatrix), P, P]),
            "mask_top_prototypes": (i32, [P, P, C.POINTER(i64)]),
            "mask_route": (i32, [P, P, i64, i32, C.POINTER(MaskMatrix), C.c_double, P, P]),
            "mask_query_routed": (i32, [P, C.POINTER(MaskMatrix), P, i64, i64, i32, i32, P, P, P]),
            "mask_merge": (i32, [P, P, i32, i64, i32, P, P, P]),
            "mask_collective_count": (i64, []),
            "mask_seeded_init": (i32, [C.c_uint64, i32, i64, i64, P]),
            "mask_debug_fail_alloc": (None, [i64]),
            "mask_get_displacement": (i32, [P, i32, P, i32]),
            "mask_get_pass": (i32, [P, i32, i32, P, P]),
            "mask_comm_init_host": (i32, [i32, i32, HOST_COLL, P, C.POINTER(P)]),
            "mask_split": (i32, [P, C.POINTER(MaskSplitParams), C.POINTER(i64), P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.mask_abi_version() != 1:
            raise ImportError("libmask ABI version mismatch")
        _lib = L
        return _lib


def check(rc: int) -> None:
    if rc != MASK_OK:
        msg = load().mask_last_error()
        raise MaskError(rc, msg.decode(errors="replace") if msg else "")
