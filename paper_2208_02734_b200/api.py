"""Thin Python binding over the libmask C-ABI (include/mask.h): argument marshalling only.

Every step of the hot path runs in libmask.so's CUDA kernels; this module turns torch
tensors / numpy arrays into pointers and sizes, calls the C entry point of the same name,
and wraps the returned handle.  PyTorch is used for device memory and streams only.

Dense data: a 2-D float32 tensor (CUDA -> device memory, CPU/numpy -> host memory).
Sparse data: a ``Csr(row_ptr int64, col int32, val float32, dim)`` of tensors/arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Any, Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import MaskBuildParams, MaskMatrix, check, load

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


@dataclass
class Csr:
    row_ptr: Any
    col: Any
    val: Any
    dim: int

    @property
    def rows(self) -> int:
        return int(self.row_ptr.shape[0]) - 1


def _is_cuda(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def _ptr(a) -> int:
    if a is None:
        return 0
    if torch is not None and isinstance(a, torch.Tensor):
        return a.data_ptr()
    return a.ctypes.data


def _prep(a, dtype):
    """Contiguous array of the requested dtype, keeping device placement."""
    if torch is not None and isinstance(a, torch.Tensor):
        tdt = {np.float32: torch.float32, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        if a.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {a.dtype}")
        return a.contiguous()
    a = np.ascontiguousarray(a)
    if a.dtype != dtype:
        raise TypeError(f"expected {np.dtype(dtype)}, got {a.dtype}")
    return a


def matrix(data, n_global: Optional[int] = None, row_offset: int = 0) -> Tuple[MaskMatrix, tuple]:
    """mask_matrix for dense (2-D float32) or Csr data; returns (struct, keepalive)."""
    m = MaskMatrix()
    if isinstance(data, Csr):
        rp = _prep(data.row_ptr, np.int64)
        col = _prep(data.col, np.int32)
        val = _prep(data.val, np.float32)
        dev = _is_cuda(rp)
        if dev != _is_cuda(col) or dev != _is_cuda(val):
            raise ValueError("CSR arrays must all live on the same side")
        m.format = _lib.MASK_CSR_F32
        m.memory = _lib.MASK_MEM_DEVICE if dev else _lib.MASK_MEM_HOST
        m.dim = int(data.dim)
        m.rows = int(rp.shape[0]) - 1
        m.values, m.row_ptr, m.col_idx = _ptr(val), _ptr(rp), _ptr(col)
        m.nnz = int(col.shape[0])
        keep = (rp, col, val)
    else:
        x = _prep(data, np.float32)
        if x.ndim != 2:
            raise ValueError("dense data must be 2-D (rows x dim)")
        m.format = _lib.MASK_DENSE_F32
        m.memory = _lib.MASK_MEM_DEVICE if _is_cuda(x) else _lib.MASK_MEM_HOST
        m.dim = int(x.shape[1])
        m.rows = int(x.shape[0])
        m.values = _ptr(x)
        keep = (x,)
    m.n_global = m.rows if n_global is None else int(n_global)
    m.row_offset = int(row_offset)
    return m, keep


def _stream(stream) -> int:
    if stream is not None:
        return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)
    if torch is not None and torch.cuda.is_available():
        return int(torch.cuda.current_stream().cuda_stream)
    return 0


class Comm:
    """NCCL communicator (one process per GPU); id exchanged over the caller's process group."""

    def __init__(self, handle: int, world: int, rank: int):
        self.handle = handle
        self.world = world
        self.rank = rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(load().mask_comm_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    @classmethod
    def init(cls, uid: bytes, world: int, rank: int) -> "Comm":
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        out = C.c_void_p()
        check(load().mask_comm_init(C.cast(buf, C.c_void_p), world, rank, C.byref(out)))
        return cls(out.value, world, rank)

    @classmethod
    def from_process_group(cls) -> "Comm":
        """Create from an initialised torch.distributed default group (broadcasts the id)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.init(obj[0], world, rank)

    @classmethod
    def host(cls, group=None) -> "Comm":
        """Host-transport communicator (mask_comm_init_host): libmask's collectives are carried
        out by torch.distributed on host buffers of ``group`` (e.g. gloo), so several ranks can
        share one GPU in tests.  Performance runs use ``from_process_group`` (NCCL)."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        fn = _lib.HOST_COLL(lambda *a: host_collective(*a, group=group))
        out = C.c_void_p()
        check(load().mask_comm_init_host(world, rank, fn, None, C.byref(out)))
        c = cls(out.value, world, rank)
        c._fn = fn  # the C function pointer must outlive the communicator
        return c

    def free(self) -> None:
        if self.handle:
            load().mask_comm_free(self.handle)
            self.handle = None


_COLL_NP = {0: np.float32, 1: np.float64, 2: np.int32, 3: np.int64, 4: np.int64}  # u64 sums as int64 bits


def host_collective(kind, buf, send, count, dtype, arg, user=None, group=None) -> int:
    """The host transport of mask_comm_init_host over torch.distributed (argument marshalling:
    the buffers are wrapped, not copied; the reduction is the process group's)."""
    try:
        import torch.distributed as dist

        count = int(count)
        if count == 0:
            return 0
        npdt = np.dtype(_COLL_NP[int(dtype)])
        world = dist.get_world_size(group)

        def view(addr, n):
            return torch.from_numpy(np.frombuffer((C.c_char * (n * npdt.itemsize)).from_address(addr), dtype=npdt))

        if kind == _lib.MASK_COLL_ALLREDUCE:
            op = dist.ReduceOp.MAX if arg == _lib.MASK_COLL_MAX else dist.ReduceOp.SUM
            dist.all_reduce(view(buf, count), op=op, group=group)
        elif kind == _lib.MASK_COLL_BROADCAST:
            src = int(arg) if group is None else dist.get_global_rank(group, int(arg))
            dist.broadcast(view(buf, count), src=src, group=group)
        elif kind == _lib.MASK_COLL_ALLGATHER:
            out = view(buf, count * world)
            dist.all_gather(list(out.split(count)), view(send, count).clone(), group=group)
        else:
            return 2
        return 0
    except Exception:  # reported to the library as a failed collective (MASK_ERR_NCCL)
        import traceback

        traceback.print_exc()
        return 1


class Index:
    """A built multilevel index (owns its device memory until ``free``)."""

    def __init__(self, handle: int, keep: tuple, dim: int, csr: bool):
        self.handle = handle
        self._keep = keep  # borrowed data must outlive the index (MASK_BORROW_DATA)
        self.dim = dim
        self.csr = csr

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def free(self) -> None:
        if getattr(self, "handle", None):
            load().mask_free(self.handle)
            self.handle = None

    # ---------------------------------------------------------------- query
    def query(self, queries, knn: int = 10, beam: int = 1, stream=None, out=None):
        """Batched k-NN (Algorithm 2).  Device queries -> device (ids int64, d2 float32)
        tensors; host queries -> numpy arrays."""
        m, keep = matrix(queries)
        nq = m.rows
        if m.memory == _lib.MASK_MEM_DEVICE:
            dev = (keep[0]).device
            ids = out[0] if out is not None else torch.empty((nq, knn), dtype=torch.int64, device=dev)
            d2 = out[1] if out is not None else torch.empty((nq, knn), dtype=torch.float32, device=dev)
        else:
            ids = out[0] if out is not None else np.empty((nq, knn), np.int64)
            d2 = out[1] if out is not None else np.empty((nq, knn), np.float32)
        check(load().mask_query(self.handle, C.byref(m), knn, beam, _ptr(ids), _ptr(d2), _stream(stream)))
        del keep
        return ids, d2

    def range_query(self, queries, radius, mode: str = "cover", stream=None):
        """mask_range_query: rows within ``radius`` (scalar or one per query) of each query.

        mode "cover" is lossless (cover-radius pruning), "paper" is Algorithm 3's rule.
        Returns (offsets int64[nq+1], ids int64[total], d2 float32[total]) on the queries' side."""
        m, keep = matrix(queries)
        nq = m.rows
        md = {"paper": _lib.MASK_RANGE_PAPER, "cover": _lib.MASK_RANGE_COVER}[mode]
        dev = m.memory == _lib.MASK_MEM_DEVICE
        if dev:
            d = keep[0].device
            r = torch.full((nq,), float(radius), dtype=torch.float32, device=d) if np.isscalar(radius) else \
                _prep(radius, np.float32)
            alloc_i = lambda n: torch.empty(n, dtype=torch.int64, device=d)  # noqa: E731
            alloc_f = lambda n: torch.empty(n, dtype=torch.float32, device=d)  # noqa: E731
        else:
            r = np.full(nq, radius, np.float32) if np.isscalar(radius) else _prep(radius, np.float32)
            alloc_i = lambda n: np.empty(n, np.int64)  # noqa: E731
            alloc_f = lambda n: np.empty(n, np.float32)  # noqa: E731
        off = alloc_i(nq + 1)
        total = C.c_int64(0)
        rc = load().mask_range_query(self.handle, C.byref(m), _ptr(r), md, 0, _ptr(off), None, None,
                                     C.byref(total), _stream(stream))
        if rc != 0 and total.value == 0:
            check(rc)
        ids, d2 = alloc_i(max(total.value, 1)), alloc_f(max(total.value, 1))
        if total.value:
            check(load().mask_range_query(self.handle, C.byref(m), _ptr(r), md, total.value, _ptr(off), _ptr(ids),
                                          _ptr(d2), C.byref(total), _stream(stream)))
        del keep
        return off, ids[:total.value], d2[:total.value]

    def insert(self, points, stream=None):
        """mask_insert: add ``points`` (dense) to the partitions their descent reaches; returns the
        level-1 prototype of each (int64, on the points' side).  New row ids continue the index."""
        m, keep = matrix(points)
        if m.memory == _lib.MASK_MEM_DEVICE:
            part = torch.empty(m.rows, dtype=torch.int64, device=keep[0].device)
        else:
            part = np.empty(m.rows, np.int64)
        check(load().mask_insert(self.handle, C.byref(m), _ptr(part), _stream(stream)))
        del keep
        return part

    def split(self, threshold: int, iters: int, seed: int = 0, flags: int = 0, stream=None) -> int:
        """mask_split: split every level-1 partition with more than ``threshold`` rows
        by a local Lloyd k-means and rebuild the local part of the index; returns the number of
        partitions split."""
        p = _lib.MaskSplitParams()
        p.threshold = int(threshold)
        p.max_iters = int(iters)
        p.flags = int(flags)
        p.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        out = C.c_int64(0)
        check(load().mask_split(self.handle, C.byref(p), C.byref(out), _stream(stream)))
        return int(out.value)

    def query_routed(self, queries, routed, node: int, id_base: int, knn: int = 10, beam: int = 1, stream=None):
        """mask_query_routed (§3.4): answer only the queries with routed[q, node] != 0 (the rest
        are padded), reporting global ids id_base + local id.  Device tensors only."""
        m, keep = matrix(queries)
        nq = m.rows
        dev = keep[0].device
        ids = torch.empty((nq, knn), dtype=torch.int64, device=dev)
        d2 = torch.empty((nq, knn), dtype=torch.float32, device=dev)
        W = int(routed.shape[1]) if nq else 1
        check(load().mask_query_routed(self.handle, C.byref(m), _ptr(routed) + int(node), W, int(id_base), knn, beam,
                                       _ptr(ids), _ptr(d2), _stream(stream)))
        del keep
        return ids, d2

    def top_prototypes(self) -> np.ndarray:
        """mask_top_prototypes: the top-level prototypes with children (what a node registers)."""
        cnt = C.c_int64(0)
        check(load().mask_top_prototypes(self.handle, None, C.byref(cnt)))
        out = np.empty((max(cnt.value, 1), self.dim), np.float32)
        check(load().mask_top_prototypes(self.handle, out.ctypes.data, C.byref(cnt)))
        return out[:cnt.value]

    # ---------------------------------------------------------------- introspection
    @property
    def num_levels(self) -> int:
        return int(load().mask_num_levels(self.handle))

    def level_info(self, level: int) -> dict:
        n, k = C.c_int64(), C.c_int64()
        d, passes, upd = C.c_int32(), C.c_int32(), C.c_int32()
        check(load().mask_level_info(self.handle, level, C.byref(n), C.byref(k), C.byref(d), C.byref(passes),
                                     C.byref(upd)))
        return dict(n_items=n.value, k=k.value, dim=d.value, passes=passes.value, updates=upd.value)

    def prototypes(self, level: int) -> np.ndarray:
        info = self.level_info(level)
        out = np.empty((info["k"], info["dim"]), np.float32)
        check(load().mask_get_prototypes(self.handle, level, out.ctypes.data))
        return out

    def labels(self, level: int) -> np.ndarray:
        info = self.level_info(level)
        out = np.empty(info["n_items"], np.int32)
        check(load().mask_get_labels(self.handle, level, out.ctypes.data))
        return out

    def children(self, level: int) -> Tuple[np.ndarray, np.ndarray]:
        info = self.level_info(level)
        off = np.empty(info["k"] + 1, np.int64)
        mem = np.empty(max(info["n_items"], 1), np.int64)
        check(load().mask_get_children(self.handle, level, off.ctypes.data, mem.ctypes.data))
        return off, mem[: info["n_items"]]

    def trace(self, level: int) -> dict:
        cap = self.level_info(level)["passes"]
        J = np.zeros(cap, np.float64)
        ch = np.zeros(cap, np.int64)
        em = np.zeros(cap, np.int64)
        n = load().mask_get_trace(self.handle, level, J.ctypes.data, ch.ctypes.data, em.ctypes.data, cap)
        if n < 0:
            check(n)
        dm = np.zeros(cap, np.float64)
        m = load().mask_get_displacement(self.handle, level, dm.ctypes.data, cap)
        if m < 0:
            check(m)
        return dict(J=J[:n], changed=ch[:n], empties=em[:n], dmax=dm[:m])

    def pass_trace(self, level: int, pass_: int) -> Tuple[np.ndarray, np.ndarray]:
        """mask_get_pass (build with MASK_TRACE_PASSES): (P used by the pass, labels it produced)."""
        info = self.level_info(level)
        P = np.empty((info["k"], info["dim"]), np.float32)
        lab = np.empty(max(info["n_items"], 1), np.int32)
        n = load().mask_get_pass(self.handle, level, int(pass_), P.ctypes.data, lab.ctypes.data)
        if n < 0:
            check(n)
        return P, lab[:n]

    def passes(self, level: int) -> List[Tuple[np.ndarray, np.ndarray]]:
        """Every assignment pass of a level (MASK_TRACE_PASSES builds): [(P_t, labels_t), ...]."""
        return [self.pass_trace(level, t) for t in range(self.level_info(level)["passes"])]

    def timing(self, level: int) -> dict:
        """CUDA-event device times of the step kernels (build with MASK_TIME_KERNELS)."""
        out = np.zeros(9, np.float64)
        n = load().mask_get_timing(self.handle, level, out.ctypes.data, 9)
        if n < 0:
            check(n)
        names = ["assign", "fixup", "update", "finalize"]
        res = {nm: dict(ms=float(out[2 * i]), launches=int(out[2 * i + 1])) for i, nm in enumerate(names)}
        res["assign_kernel"] = {0: "K2-simt", 1: "K1-tcgen05-3xtf32", 2: "K3-csr", 3: "K11-fused-small-level", 4: "K12-grouped", 5: "K3T-csr-tcgen05", 6: "K1-tcgen05-3xfp16"}.get(int(out[8]), "none")
        return res


def kernel_launches() -> int:
    """Cumulative kernel launches issued by libmask in this process."""
    return int(load().mask_kernel_launches())


def build(data, levels: Sequence[int], iters: int, init_idx: Optional[Sequence[np.ndarray]] = None,
          tol: float = 0.0, flags: int = 0, comm: Optional[Comm] = None, iter_cb: Optional[Callable] = None,
          stream=None, n_global: Optional[int] = None, row_offset: int = 0, seed: int = 0,
          empty: str = "keep") -> Index:
    """mask_build: multilevel index over ``data`` (this rank's shard when ``comm`` is given).

    init_idx: one array of distinct indices per level, or None to let the library draw them
    from ``seed`` (mask_seeded_init).  iter_cb(level, pass, P (k x dim float32 numpy), labels
    (int32 numpy)) is the test-only step-parity hook.  empty: "keep" (D5) or "farthest" (D5b,
    SPEC S:128: emptied prototypes re-seeded at the pass's farthest rows)."""
    m, keep = matrix(data, n_global=n_global, row_offset=row_offset)
    L = len(levels)
    ks = (C.c_int64 * L)(*[int(k) for k in levels])
    ptrs = None
    if init_idx is not None:
        idx_arrays = [np.ascontiguousarray(a, dtype=np.int64) for a in init_idx]
        if len(idx_arrays) != L:
            raise ValueError("one init index array per level")
        ptrs = (C.POINTER(C.c_int64) * L)(*[a.ctypes.data_as(C.POINTER(C.c_int64)) for a in idx_arrays])
    p = MaskBuildParams()
    p.num_levels = L
    p.max_iters = int(iters)
    p.k = ks
    p.tol = float(tol)
    p.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    if ptrs is not None:
        p.init_idx = ptrs
    p.empty_policy = {"keep": _lib.MASK_EMPTY_KEEP, "farthest": _lib.MASK_EMPTY_FARTHEST}[empty]
    p.flags = int(flags)
    cb_ref = None
    if iter_cb is not None:
        def _cb(level, pass_, P, k, dim, labels, n_items, user):
            Pa = np.ctypeslib.as_array(P, shape=(k, dim)).copy()
            la = np.ctypeslib.as_array(labels, shape=(n_items,)).copy() if n_items else np.zeros(0, np.int32)
            iter_cb(int(level), int(pass_), Pa, la)

        cb_ref = _lib.ITER_CB(_cb)
        p.iter_cb = cb_ref
    out = C.c_void_p()
    rc = load().mask_build(C.byref(m), C.byref(p), comm.handle if comm else None, _stream(stream), C.byref(out))
    check(rc)
    keep_all = keep if (flags & _lib.MASK_BORROW_DATA) else ()
    return Index(out.value, keep_all, m.dim, m.format == _lib.MASK_CSR_F32)


def seeded_init(seed: int, level: int, n: int, k: int) -> np.ndarray:
    """mask_seeded_init: the k distinct init indices mask_build draws from ``seed`` for a level."""
    out = np.empty(max(int(k), 1), np.int64)
    check(load().mask_seeded_init(int(seed) & 0xFFFFFFFFFFFFFFFF, int(level), int(n), int(k), out.ctypes.data))
    return out[:int(k)]


def grouped_depth(n: int, length_group: int, n_centroids: int) -> Tuple[int, List[int]]:
    """Depth and prototypes per layer of the grouped construction (floor recurrence)."""
    cap = 64
    out = (C.c_int64 * cap)()
    depth = load().mask_grouped_depth(int(n), int(length_group), int(n_centroids), out, cap)
    if depth < 0:
        check(depth)
    return depth, [int(out[i]) for i in range(min(depth, cap))]


def relocate(index: "Index", got, order, keys, n_centroids: int, stream=None):
    """mask_relocate (§5.1, reading G8): the next data-layer order of a grouped index from the
    point-search results ``got`` (device int64, one per point), the current order and the
    iteration's keys (device int64).  Returns (order_out, reached, misses): device int64
    tensors and the number of points the search did not return."""
    n = int(got.shape[0])
    for a in (got, order, keys):
        if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.int64 and a.is_contiguous()):
            raise TypeError("got / order / keys must be contiguous int64 CUDA tensors")
    out = torch.empty(n, dtype=torch.int64, device=got.device)
    reached = torch.empty(n, dtype=torch.int64, device=got.device)
    misses = C.c_int64(0)
    check(load().mask_relocate(index.handle, _ptr(got), _ptr(order), _ptr(keys), int(n_centroids), _ptr(out),
                               _ptr(reached), C.byref(misses), _stream(stream)))
    return out, reached, int(misses.value)


def build_grouped(data, length_group: int, n_centroids: int, iters: int, perm: Optional[np.ndarray] = None,
                  flags: int = 0, stream=None) -> Index:
    """mask_build_grouped: the paper's Algorithm 1 (groups of ``length_group`` items, each
    clustered into ``n_centroids`` prototypes; ``perm`` = the seeded data-layer split order)."""
    m, keep = matrix(data)
    p = _lib.MaskGroupedParams()
    p.length_group = int(length_group)
    p.n_centroids = int(n_centroids)
    p.max_iters = int(iters)
    p.flags = int(flags)
    perm_arr = None
    if perm is not None:
        perm_arr = np.ascontiguousarray(perm, dtype=np.int64)
        p.perm = perm_arr.ctypes.data_as(C.POINTER(C.c_int64))
    out = C.c_void_p()
    check(load().mask_build_grouped(C.byref(m), C.byref(p), _stream(stream), C.byref(out)))
    keep_all = keep if (flags & _lib.MASK_BORROW_DATA) else ()
    return Index(out.value, keep_all, m.dim, False)


def assign(data, P, flags: int = 0, stream=None):
    """mask_assign: one assignment pass on the device. Returns (labels int32, d2 float32, n_flagged)."""
    m, keep = matrix(data)
    P = _prep(P, np.float32)
    n = m.rows
    dev = P.device
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev)
    nf = C.c_int64(0)
    check(load().mask_assign(C.byref(m), _ptr(P), int(P.shape[0]), int(flags), _ptr(labels), _ptr(d2),
                             C.byref(nf), _stream(stream)))
    del keep
    return labels, d2, int(nf.value)


def update(data, labels, P_in, stream=None):
    """mask_update: member means (empty clusters keep P_in). Returns (P_out, counts, max_disp)."""
    m, keep = matrix(data)
    P_in = _prep(P_in, np.float32)
    labels = _prep(labels, np.int32)
    P_out = torch.empty_like(P_in)
    counts = torch.empty(P_in.shape[0], dtype=torch.int32, device=P_in.device)
    md = C.c_double(0.0)
    check(load().mask_update(C.byref(m), _ptr(labels), int(P_in.shape[0]), _ptr(P_in), _ptr(P_out),
                             _ptr(counts), C.byref(md), _stream(stream)))
    del keep
    return P_out, counts, float(md.value)


def route(registry, node_of, n_nodes: int, queries, epsilon: float, stream=None):
    """mask_route (§3.4): uint8 (nq x n_nodes) device tensor, 1 where some registered centroid
    of the node is closer than epsilon (strict); epsilon = inf routes everywhere."""
    registry = _prep(registry, np.float32)
    node_of = _prep(node_of, np.int32)
    m, keep = matrix(queries)
    routed = torch.empty((m.rows, int(n_nodes)), dtype=torch.uint8, device=registry.device)
    check(load().mask_route(_ptr(registry), _ptr(node_of), int(registry.shape[0]), int(n_nodes), C.byref(m),
                            float(epsilon), _ptr(routed), _stream(stream)))
    del keep
    return routed


def merge(ids, d2, stream=None):
    """mask_merge (§3.4): ids / d2 of shape (n_nodes, nq, k) -> the k best per query by
    (d^2, node, id), shapes (nq, k)."""
    ids = _prep(ids, np.int64)
    d2 = _prep(d2, np.float32)
    W, nq, k = ids.shape
    oi = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    od = torch.empty((nq, k), dtype=torch.float32, device=ids.device)
    check(load().mask_merge(_ptr(ids), _ptr(d2), int(W), int(nq), int(k), _ptr(oi), _ptr(od), _stream(stream)))
    return oi, od


def collective_count() -> int:
    """NCCL calls libmask has issued in this process (the §3.4 zero-communication counter)."""
    return int(load().mask_collective_count())


def device_ok() -> bool:
    return bool(load().mask_device_ok())
