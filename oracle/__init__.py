"""FP64 CPU oracle for the MASK hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2208_02734_b200``) never imports it and shares no code with it; the
only module both sides use is ``datagen`` (seeded inputs, no method arithmetic).

The arithmetic lives in ``mask_oracle.c`` (plain C, FP64, compiled here with
gcc; see its header for the paper passages each function follows).  This
module only marshals numpy arrays into it and derives the child lists
``children_l(j) = {i : labels_l[i] = j}`` in ascending i (PAPER.md P:655/P:658
``layerLabels``; D7).

Parity status: every function here is pinned by ``tests/test_oracle.py``
(hand-derived worked example S:107, closed forms, brute force against scipy /
numpy library routines, invariants).  No function is "parity unpinned".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mask_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None

dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


# MASK_ORACLE_SANITIZE=1: an ASan + UBSan build (run python with LD_PRELOAD=$(gcc
# -print-file-name=libasan.so) ASAN_OPTIONS=detect_leaks=0; SURVEY §4 T4 for the host code)
_SANITIZE = os.environ.get("MASK_ORACLE_SANITIZE") == "1"
if _SANITIZE:
    _LIB_PATH = os.path.join(_HERE, "_build", "liboracle_asan.so")


def build(force: bool = False) -> str:
    """Compile mask_oracle.c -> oracle/_build/liboracle.so (gcc -O2 -fopenmp, IEEE FP)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        san = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=all"] \
            if _SANITIZE else []
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
             "-ffp-contract=off", *san, "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.orc_num_threads.restype = C.c_int
            L.orc_set_num_threads.argtypes = [C.c_int]
            L.orc_dist2.restype = C.c_double
            L.orc_dist2.argtypes = [C.c_int, dp, dp]
            L.orc_dist2_csr_dense.restype = C.c_double
            L.orc_dist2_csr_dense.argtypes = [C.c_int64, i32p, dp, dp, C.c_double]
            L.orc_dist2_csr_csr.restype = C.c_double
            L.orc_dist2_csr_csr.argtypes = [C.c_int64, i32p, dp, C.c_int64, i32p, dp]
            L.orc_assign.argtypes = [C.c_int64, C.c_int, dp, C.c_int64, dp, i32p, dp, dp]
            L.orc_assign_csr.argtypes = [C.c_int64, C.c_int, i64p, i32p, dp, C.c_int64, dp, i32p, dp, dp]
            L.orc_cluster_sums.argtypes = [C.c_int64, C.c_int, dp, i32p, C.c_int64, dp, i64p]
            L.orc_cluster_sums_csr.argtypes = [C.c_int64, C.c_int, i64p, i32p, dp, i32p, C.c_int64, dp, i64p]
            L.orc_means_from_sums.restype = C.c_double
            L.orc_means_from_sums.argtypes = [C.c_int64, C.c_int, dp, i64p, dp, dp]
            lloyd_args = [C.c_int64, i64p, C.c_int, C.c_double, dp, i32p, dp, i64p, C.POINTER(C.c_int)]
            L.orc_lloyd.restype = C.c_int
            L.orc_lloyd.argtypes = [C.c_int64, C.c_int, dp] + lloyd_args
            L.orc_lloyd_csr.restype = C.c_int
            L.orc_lloyd_csr.argtypes = [C.c_int64, C.c_int, i64p, i32p, dp] + lloyd_args
            L.orc_lloyd_trace.restype = C.c_int
            L.orc_lloyd_trace.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + \
                lloyd_args + [dp, i32p]
            L.orc_lloyd_ex.restype = C.c_int
            L.orc_lloyd_ex.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p] + \
                lloyd_args + [C.c_void_p, C.c_void_p, C.c_int]
            _lib = L
        return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(t: int) -> None:
    """OpenMP threads of the oracle's parallel loops (rows / queries split across threads)."""
    lib().orc_set_num_threads(int(t))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _csr(csr):
    rp, col, val = csr
    return (np.ascontiguousarray(rp, dtype=np.int64), np.ascontiguousarray(col, dtype=np.int32), _f64(val))


# ------------------------------------------------------------------ primitives
def dist2(y, c) -> float:
    y, c = _f64(y), _f64(c)
    return float(lib().orc_dist2(y.size, y, c))


def assign(Y, P) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """labels (lowest j on ties), best d^2, second-best d^2 (dense rows)."""
    Y, P = _f64(Y), _f64(P)
    n, d = Y.shape
    k = P.shape[0]
    lab = np.empty(n, np.int32)
    b1 = np.empty(n, np.float64)
    b2 = np.empty(n, np.float64)
    lib().orc_assign(n, d, Y, k, P, lab, b1, b2)
    return lab, b1, b2


def assign_csr(csr, dim: int, P):
    rp, col, val = _csr(csr)
    P = _f64(P)
    n = rp.size - 1
    lab = np.empty(n, np.int32)
    b1 = np.empty(n, np.float64)
    b2 = np.empty(n, np.float64)
    lib().orc_assign_csr(n, dim, rp, col, val, P.shape[0], P, lab, b1, b2)
    return lab, b1, b2


def cluster_sums(Y, labels, k: int):
    Y = _f64(Y)
    n, d = Y.shape
    S = np.empty((k, d), np.float64)
    cnt = np.empty(k, np.int64)
    lib().orc_cluster_sums(n, d, Y, np.ascontiguousarray(labels, np.int32), k, S, cnt)
    return S, cnt


def cluster_sums_csr(csr, dim: int, labels, k: int):
    rp, col, val = _csr(csr)
    S = np.empty((k, dim), np.float64)
    cnt = np.empty(k, np.int64)
    lib().orc_cluster_sums_csr(rp.size - 1, dim, rp, col, val, np.ascontiguousarray(labels, np.int32), k, S, cnt)
    return S, cnt


def means_from_sums(S, counts, P_old):
    S, P_old = _f64(S), _f64(P_old)
    k, d = P_old.shape
    P_new = np.empty_like(P_old)
    md = lib().orc_means_from_sums(k, d, S, np.ascontiguousarray(counts, np.int64), P_old, P_new)
    return P_new, float(md)


def means(Y, labels, P_old):
    """Prototype update: member means, empty clusters keep P_old (D5)."""
    S, cnt = cluster_sums(Y, labels, P_old.shape[0])
    return means_from_sums(S, cnt, P_old)[0], cnt


# ------------------------------------------------------------------ seeded initialisation
_M64 = (1 << 64) - 1


def seeded_init(seed: int, level: int, n: int, k: int) -> np.ndarray:
    """D2's k distinct init indices in [0, n) when the caller passes none (include/mask.h
    mask_seeded_init, the same documented generator written out here): Floyd's algorithm --
    for j = n-k .. n-1 take t = u(j+1) unless already taken, else j -- with u(m) = next() mod m
    over the SplitMix64 sequence started at seed + level * 0x9E3779B97F4A7C15."""
    if not (1 <= k <= n) or level < 1:
        raise ValueError("need 1 <= k <= n and level >= 1")
    state = (seed + level * 0x9E3779B97F4A7C15) & _M64
    taken, out = set(), []
    for j in range(n - k, n):
        state = (state + 0x9E3779B97F4A7C15) & _M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        z = z ^ (z >> 31)
        t = z % (j + 1)
        v = j if t in taken else t
        taken.add(v)
        out.append(v)
    return np.array(out, np.int64)


# ------------------------------------------------------------------ Lloyd / build
class LevelResult:
    def __init__(self, P, labels, J, changed, updates, passes=None):
        self.P = P
        self.labels = labels
        self.J = J
        self.changed = changed
        self.updates = updates
        self.passes = passes  # trace=True: [(P_t used by pass t, labels_t), ...] incl. the final pass


EMPTY_POLICIES = {"keep": 0, "farthest": 1}


def lloyd(Y, init_idx, T: int, tol: float = 0.0, csr_dim: Optional[int] = None, trace: bool = False,
          empty: str = "keep") -> LevelResult:
    """One level: Lloyd from Y[init_idx], T iterations, then a final assignment.

    trace=True also records, per assignment pass, the prototypes it used and its labels
    (an output copy only: the arithmetic is the same code path).  empty: "keep" (D5) or
    "farthest" (D5b: emptied prototypes re-seeded at the pass's farthest rows)."""
    if trace or empty != "keep":
        return _lloyd_trace(Y, init_idx, T, tol, csr_dim, EMPTY_POLICIES[empty], trace)
    init_idx = np.ascontiguousarray(init_idx, np.int64)
    k = init_idx.size
    J = np.zeros(T + 1, np.float64)
    ch = np.zeros(T + 1, np.int64)
    upd = C.c_int(0)
    if csr_dim is None:
        Y = _f64(Y)
        n, d = Y.shape
        P = np.empty((k, d), np.float64)
        lab = np.empty(n, np.int32)
        passes = lib().orc_lloyd(n, d, Y, k, init_idx, T, tol, P, lab, J, ch, C.byref(upd))
    else:
        rp, col, val = _csr(Y)
        n, d = rp.size - 1, csr_dim
        P = np.empty((k, d), np.float64)
        lab = np.empty(n, np.int32)
        passes = lib().orc_lloyd_csr(n, d, rp, col, val, k, init_idx, T, tol, P, lab, J, ch, C.byref(upd))
    return LevelResult(P, lab, J[:passes], ch[:passes], upd.value)


def _lloyd_trace(Y, init_idx, T, tol, csr_dim, policy=0, record=True):
    init_idx = np.ascontiguousarray(init_idx, np.int64)
    k = init_idx.size
    J = np.zeros(T + 1, np.float64)
    ch = np.zeros(T + 1, np.int64)
    upd = C.c_int(0)
    if csr_dim is None:
        Y = _f64(Y)
        n, d = Y.shape
        args = (Y.ctypes.data, None, None, None)
        keep = (Y,)
    else:
        rp, col, val = _csr(Y)
        n, d = rp.size - 1, csr_dim
        args = (None, rp.ctypes.data, col.ctypes.data, val.ctypes.data)
        keep = (rp, col, val)
    P = np.empty((k, d), np.float64)
    lab = np.empty(n, np.int32)
    Pp = np.empty((T + 1, k, d), np.float64) if record else None
    Lp = np.empty((T + 1, max(n, 1)), np.int32) if record else None
    passes = lib().orc_lloyd_ex(n, d, *args, k, init_idx, T, tol, P, lab, J, ch, C.byref(upd),
                                Pp.ctypes.data if record else None, Lp.ctypes.data if record else None, policy)
    del keep
    seq = [(Pp[t], Lp[t, :n]) for t in range(passes)] if record else None
    return LevelResult(P, lab, J[:passes], ch[:passes], upd.value, passes=seq)


def children(labels, k: int) -> Tuple[np.ndarray, np.ndarray]:
    """CSR child lists: offsets (k+1), members ascending i within each prototype."""
    labels = np.asarray(labels, np.int64)
    counts = np.bincount(labels, minlength=k)
    offsets = np.zeros(k + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    members = np.argsort(labels, kind="stable").astype(np.int64)
    return offsets, members


class Index:
    """Oracle multilevel index: per level P (k_l x d, FP64), labels, child lists, traces."""

    def __init__(self, levels: List[LevelResult], offsets: List[np.ndarray], members: List[np.ndarray], dim: int):
        self.levels = levels
        self.offsets = offsets
        self.members = members
        self.dim = dim

    @property
    def P(self):
        return [lv.P for lv in self.levels]


def build_index(X, init_idx: Sequence[np.ndarray], T: int, tol: float = 0.0, csr_dim: Optional[int] = None,
                trace: bool = False, empty: str = "keep") -> Index:
    """Bottom-up levels: level 1 clusters X, level l+1 clusters P_l (D1, D6)."""
    levels, offs, mems = [], [], []
    Y = X
    dim = csr_dim
    for l, idx in enumerate(init_idx):
        res = lloyd(Y, idx, T, tol, csr_dim=csr_dim if l == 0 else None, trace=trace, empty=empty)
        levels.append(res)
        o, m = children(res.labels, res.P.shape[0])
        offs.append(o)
        mems.append(m)
        Y = res.P
        dim = res.P.shape[1]
    return Index(levels, offs, mems, dim)


# ------------------------------------------------------------------ grouped construction
def grouped_layer_sizes(n: int, length_group: int, n_centroids: int) -> List[Tuple[int, int]]:
    """Algorithm 1's loop: ngroups <- n / lengthGroup (integer, floor), and while
    ngroups >= 1 a layer of ngroups * nCentroids prototypes is built over n items, after which
    n <- ngroups * nCentroids.  Returns [(n_items, ngroups)] per layer."""
    if not 1 <= n_centroids < length_group:
        raise ValueError("need 1 <= nCentroids < lengthGroup (the recurrence does not shrink otherwise)")
    out = []
    g = n // length_group
    while g >= 1:
        out.append((n, g))
        n = g * n_centroids
        g = n // length_group
    return out


def build_grouped(X, length_group: int, n_centroids: int, T: int, perm=None) -> Index:
    """Grouped multilevel construction (Algorithm 1) with the readings of DESIGN.md
    G1-G5: the data layer is taken in ``perm`` order, every layer is chunked into ngroups
    balanced groups (sizes floor(n/g), the last n mod g groups one larger), each group is
    clustered by ``lloyd`` from its first nCentroids items, prototypes are stored group-major
    (global id = group * nCentroids + local id), and the next layer re-chunks them in order."""
    Y = _f64(X)
    levels, offs, mems = [], [], []
    order = np.arange(Y.shape[0]) if perm is None else np.asarray(perm, np.int64)
    for n, g in grouped_layer_sizes(Y.shape[0], length_group, n_centroids):
        base, rem = divmod(n, g)
        P = np.empty((g * n_centroids, Y.shape[1]), np.float64)
        lab = np.empty(n, np.int32)
        start = 0
        for gi in range(g):
            size = base + (1 if gi >= g - rem else 0)
            items = order[start:start + size]
            start += size
            res = lloyd(Y[items], np.arange(n_centroids), T)
            P[gi * n_centroids:(gi + 1) * n_centroids] = res.P
            lab[items] = gi * n_centroids + res.labels
        res_l = LevelResult(P, lab, np.zeros(0), np.zeros(0, np.int64), 0)
        levels.append(res_l)
        o, m = children(lab, P.shape[0])
        offs.append(o)
        mems.append(m)
        Y = P
        order = np.arange(P.shape[0])
    return Index(levels, offs, mems, Y.shape[1])


def exhaustive_error(index: Index, X) -> float:
    """Fraction of the indexed points whose single-path (beam 1) descent over the explicit child
    lists does not return the point itself as its nearest neighbour (point search of every
    element; SPEC exhaustive_error)."""
    X = _f64(X)
    ids, _, _ = query(index.P, index.offsets, index.members, X, X, 1, 1)
    return float(np.mean(ids[:, 0] != np.arange(X.shape[0])))


def relocation_order(order, n_groups: int, found, reached_group, keys) -> np.ndarray:
    """One relocation step (§5.1: "when the point search reaches a partition at
    the bottom of the tree and the target element is not found in that group, ... the target
    point is reassigned to that partition"; reading G8): a point keeps its current data-layer
    group when its search found it (or reached no partition: reached_group < 0), else it moves
    to the group of the partition its search reached; the new data-layer order lists the target groups in order, the points of a group
    by their seeded key (the rebuild seed policy), and the rebuild splits it into the same
    number of balanced groups."""
    order = np.asarray(order, np.int64)
    n = order.size
    base, rem = divmod(n, n_groups)
    sizes = np.full(n_groups, base, np.int64)
    sizes[n_groups - rem:] += 1
    cur = np.empty(n, np.int64)
    cur[order] = np.repeat(np.arange(n_groups), sizes)
    reached_group = np.asarray(reached_group, np.int64)
    # a search that dead-ends (no partition reached: reached_group < 0) leaves the point in place
    target = np.where(np.asarray(found, bool) | (reached_group < 0), cur, reached_group)
    return np.lexsort((np.asarray(keys, np.int64), target)).astype(np.int64)


def relocate_and_rebuild(X, length_group: int, n_centroids: int, T: int, perm, iterations: int,
                         base_seed: int, keys_fn):
    """§5.1 relocation loop (Table 1): build, exhaustive point search, relocate the
    points not found, rebuild; returns the error rate after each build (entry 0 = the first
    build).  keys_fn(base_seed, i, n) gives iteration i's order keys (an input, datagen)."""
    Xd = _f64(X)
    n = Xd.shape[0]
    g = grouped_layer_sizes(n, length_group, n_centroids)[0][1]
    order = np.asarray(perm, np.int64)
    errors = []
    for i in range(iterations + 1):
        idx = build_grouped(Xd, length_group, n_centroids, T, perm=order)
        ids, _, _ = query(idx.P, idx.offsets, idx.members, Xd, Xd, 1, 1)
        found = ids[:, 0] == np.arange(n)
        errors.append(float(np.mean(~found)))
        if i == iterations:
            break
        # the returned row's partition (-1: the descent dead-ended in a prototype whose children
        # are all childless, so nothing was returned)
        reached = np.where(ids[:, 0] >= 0, idx.levels[0].labels[np.maximum(ids[:, 0], 0)] // n_centroids, -1)
        order = relocation_order(order, g, found, reached, keys_fn(base_seed, i + 1, n))
    return errors


# ------------------------------------------------------------------ range search (NEXT-2)
def cover_radii(index: Index, X) -> List[np.ndarray]:
    """cover_1(j) = max over data rows x with labels_1 = j of ||x - c_j||; cover_l(j) = max over
    children i of ||c_i - c_j|| + cover_{l-1}(i) (an upper bound on the distance from c_j to every
    row below it, by the triangle inequality).  Childless prototypes get 0."""
    X = _f64(X)
    out = []
    Y = X
    prev = np.zeros(X.shape[0])
    for lv in index.levels:
        P = _f64(lv.P)
        lab = np.asarray(lv.labels, np.int64)
        r = np.sqrt(((Y - P[lab]) ** 2).sum(axis=1)) + prev
        cov = np.zeros(P.shape[0])
        np.maximum.at(cov, lab, r)
        out.append(cov)
        Y, prev = P, cov
    return out


def range_query(P: Sequence[np.ndarray], offsets: Sequence[np.ndarray], members: Sequence[np.ndarray], X, q,
                radius: float, cover: Optional[Sequence[np.ndarray]] = None):
    """Algorithm 3 for one query over explicit child lists: keep every top-level
    prototype with children whose distance is <= radius (+ cover(c) when ``cover`` is given),
    follow the children of every kept prototype level by level, return the rows of the reached
    partitions within ``radius`` as (ids, d^2) sorted by (d^2, id)."""
    X, q = _f64(X), _f64(q)
    L = len(P)

    def kept(l, cand):
        Pl = _f64(P[l])
        has = offsets[l][cand + 1] > offsets[l][cand]
        d = np.sqrt(((Pl[cand] - q) ** 2).sum(axis=1))
        lim = radius + (cover[l][cand] if cover is not None else 0.0)
        return cand[has & (d <= lim)]

    S = kept(L - 1, np.arange(P[L - 1].shape[0]))
    for l in range(L - 2, -1, -1):
        C_ = np.concatenate([members[l + 1][offsets[l + 1][j]:offsets[l + 1][j + 1]] for j in S]) if S.size else \
            np.zeros(0, np.int64)
        S = kept(l, np.sort(C_.astype(np.int64)))
    rows = np.concatenate([members[0][offsets[0][j]:offsets[0][j + 1]] for j in S]) if S.size else np.zeros(0, np.int64)
    rows = np.sort(rows.astype(np.int64))
    d2 = ((X[rows] - q) ** 2).sum(axis=1)
    ok = d2 <= radius * radius
    rows, d2 = rows[ok], d2[ok]
    o = np.lexsort((rows, d2))
    return rows[o], d2[o]


# ------------------------------------------------------------------ insertion (NEXT-4)
def descend_leaf(P: Sequence[np.ndarray], offsets: Sequence[np.ndarray], members: Sequence[np.ndarray], q):
    """The insertion procedure's path: at the top level the nearest prototype with
    children, then the nearest of its children (with children), ... down to level 1.  Ties take
    the lowest id (D4).  Returns (level-1 prototype, smallest relative gap of the decisions)."""
    q = _f64(q)
    L = len(P)

    def pick(l, cand):
        cand = np.asarray(cand, np.int64)
        cand = cand[offsets[l][cand + 1] > offsets[l][cand]]
        d = ((_f64(P[l])[cand] - q) ** 2).sum(axis=1)
        o = np.lexsort((cand, d))
        gap = (d[o[1]] - d[o[0]]) / d[o[1]] if len(o) > 1 and d[o[1]] > 0 else np.inf
        return int(cand[o[0]]), gap

    j, gap = pick(L - 1, np.arange(P[L - 1].shape[0]))
    for l in range(L - 2, -1, -1):
        j, g = pick(l, members[l + 1][offsets[l + 1][j]:offsets[l + 1][j + 1]])
        gap = min(gap, g)
    return j, gap


def split_partitions(P: Sequence[np.ndarray], labels: Sequence[np.ndarray], X, threshold: int, T: int, seed: int):
    """Partition split and local rebuild ("if one partition grows beyond a certain
    threshold, it can be split in smaller data groups and reconstruct just the local part of the
    index covering that specific region, without affecting the rest of the structure";
    DESIGN.md reading S1).

    For every level-1 prototype j in ascending order whose partition holds n_j > threshold rows:
    its rows in ascending id order are clustered by Lloyd (``lloyd``, T iterations + the final
    assignment) into s = ceil(n_j / threshold) groups from the init rows
    ``seeded_init(seed + j, 1, n_j, s)``; group 0 keeps id j, groups 1..s-1 get the next new
    level-1 ids (k_1, k_1 + 1, ... in order of j, then group); the new prototypes' level-2 label is
    j's (same parent); prototypes and labels of every other partition and of every upper level
    are unchanged.  Partitions created here are not split again in the same call.

    P, labels: per level (bottom first) as the index holds them (labels[0] over the data rows,
    labels[l] over level-l prototypes).  Returns (P, labels, split_js) with P[0], labels[0] and
    (if present) labels[1] updated."""
    P = [np.array(p, np.float64) for p in P]
    labels = [np.array(lb, np.int64) for lb in labels]
    X = _f64(X)
    k1 = P[0].shape[0]
    counts = np.bincount(labels[0], minlength=k1)
    new_rows, new_parent, split = [], [], []
    nxt = k1
    for j in range(k1):
        nj = int(counts[j])
        if nj <= threshold:
            continue
        rows = np.nonzero(labels[0] == j)[0]  # ascending row ids
        s = -(-nj // threshold)
        init = seeded_init((seed + j) & _M64, 1, nj, s)
        res = lloyd(X[rows], init, T)
        P[0][j] = res.P[0]
        for g in range(1, s):
            new_rows.append(res.P[g])
            if len(labels) > 1:
                new_parent.append(labels[1][j])
        lab = np.where(res.labels == 0, j, nxt + res.labels.astype(np.int64) - 1)
        labels[0][rows] = lab
        nxt += s - 1
        split.append(j)
    if new_rows:
        P[0] = np.vstack([P[0], np.array(new_rows)])
        if len(labels) > 1:
            labels[1] = np.concatenate([labels[1], np.array(new_parent, np.int64)])
    return P, labels, split


# ------------------------------------------------------------------ distributed mode (NEXT-3)
def top_registry(index_P_top, offsets_top) -> np.ndarray:
    """What a node registers with the coordinator (§3.4, "just the top level
    centroids from each node need to be recorded"): its top-level prototypes, keeping those
    with children (reading C2: a childless prototype represents no data)."""
    P = _f64(index_P_top)
    o = np.asarray(offsets_top, np.int64)
    return P[o[1:] > o[:-1]]


def route(tops: Sequence[np.ndarray], q, epsilon: float) -> Tuple[List[int], float]:
    """§3.4: the nodes "that have centroids whose distance to the target query
    object is lower than a given threshold epsilon" -- node n is routed iff some registered
    top centroid c of n has ||q - c|| < epsilon (strict; reading C1), epsilon = inf routes to
    every node ("searching in all nodes in parallel").  Returns (routed node ids ascending,
    smallest relative gap |d_min^2 - epsilon^2| / epsilon^2 over the nodes, inf if none)."""
    q = _f64(q)
    nodes, gap = [], np.inf
    for n, T in enumerate(tops):
        if np.isinf(epsilon):
            nodes.append(n)
            continue
        T = _f64(T)
        if T.shape[0] == 0:
            continue
        dmin2 = ((T - q) ** 2).sum(axis=1).min()
        e2 = float(epsilon) * float(epsilon)
        if dmin2 < e2:
            nodes.append(n)
        if e2 > 0:
            gap = min(gap, abs(dmin2 - e2) / e2)
    return nodes, gap


def merge(results: Sequence[Tuple[np.ndarray, np.ndarray]], routed: Sequence[int], knn: int):
    """The coordinator's merge ("searching in all nodes in parallel"): the knn best
    of the routed nodes' local answers by (d^2, node, id) (reading C3); ids are global;
    padded with (-1, +inf).  ``results[n]`` = (ids, d2) of node n for this query."""
    cand = []
    for n in routed:
        ids, d2 = results[n]
        cand += [(float(d), n, int(i)) for i, d in zip(ids, d2) if i >= 0]
    cand.sort()
    cand = cand[:knn]
    ids = np.full(knn, -1, np.int64)
    d2 = np.full(knn, np.inf)
    for r, (d, _, i) in enumerate(cand):
        ids[r], d2[r] = i, d
    return ids, d2


def cluster_query(nodes: Sequence[dict], Q, knn: int, beam: int, epsilon: float, csr_dim: Optional[int] = None):
    """§3.4 distributed k-NN for a batch: route each query against the registry, run the
    descent (``query``) on each routed node's own index, merge.  ``nodes[n]`` = dict(P, offsets,
    members, X, id_base) of node n's independent index (node-local row ids; global id =
    id_base + local id).  Returns ids, d2 (nq x knn), routed (nq x n_nodes bool), gap (per
    query: the smallest relative gap of the routing decisions and of the descents)."""
    if csr_dim is not None:  # CSR data and queries: route on the densified query vectors
        rp, col, val = _csr(Q)
        Qv = np.zeros((rp.size - 1, csr_dim))
        for i in range(rp.size - 1):
            Qv[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    else:
        Q = Qv = _f64(Q)
    nq, W = Qv.shape[0], len(nodes)
    tops = [top_registry(nd["P"][-1], nd["offsets"][-1]) for nd in nodes]
    routed = np.zeros((nq, W), bool)
    rgap = np.full(nq, np.inf)
    for i in range(nq):
        rs, rgap[i] = route(tops, Qv[i], epsilon)
        routed[i, rs] = True
    local = []
    qgap = np.full(nq, np.inf)
    for n, nd in enumerate(nodes):
        ids, d2, g = query(nd["P"], nd["offsets"], nd["members"], nd["X"], Q, knn, beam, dim=csr_dim,
                           x_csr=csr_dim is not None, q_csr=csr_dim is not None)
        ids = np.where(ids >= 0, ids + int(nd["id_base"]), -1)
        local.append((ids, d2))
        qgap = np.where(routed[:, n], np.minimum(qgap, g), qgap)
    out_i = np.empty((nq, knn), np.int64)
    out_d = np.empty((nq, knn))
    for i in range(nq):
        out_i[i], out_d[i] = merge([(l[0][i], l[1][i]) for l in local], np.nonzero(routed[i])[0], knn)
    return out_i, out_d, routed, np.minimum(rgap, qgap)


# ------------------------------------------------------------------ queries
def _ptr_array(arrs, ctype):
    return (C.POINTER(ctype) * len(arrs))(*[a.ctypes.data_as(C.POINTER(ctype)) for a in arrs])


def query(P: Sequence[np.ndarray], offsets: Sequence[np.ndarray], members: Sequence[np.ndarray], X, Q,
          knn: int, beam: int = 1, dim: Optional[int] = None, x_csr: bool = False, q_csr: bool = False):
    """Descent over a given index (the oracle's own, or a GPU-built one exported via getters).

    Returns ids (nq x knn, int64, -1 padded), d2 (nq x knn, FP64, +inf padded) and the per-query
    minimum relative gap over all selections (for the 1e-5 tie-window exemption)."""
    L = len(P)
    Pd = [_f64(p) for p in P]
    Of = [np.ascontiguousarray(o, np.int64) for o in offsets]
    Me = [np.ascontiguousarray(m, np.int64) for m in members]
    d = Pd[0].shape[1] if dim is None else dim
    kpl = np.array([p.shape[0] for p in Pd], np.int64)
    null_d = C.POINTER(C.c_double)()
    null_i64 = C.POINTER(C.c_int64)()
    null_i32 = C.POINTER(C.c_int32)()
    if x_csr:
        xrp, xcol, xval = _csr(X)
        xargs = [null_d, xrp.ctypes.data_as(C.POINTER(C.c_int64)), xcol.ctypes.data_as(C.POINTER(C.c_int32)),
                 xval.ctypes.data_as(C.POINTER(C.c_double))]
        keep_x = (xrp, xcol, xval)
    else:
        Xd = _f64(X)
        xargs = [Xd.ctypes.data_as(C.POINTER(C.c_double)), null_i64, null_i32, null_d]
        keep_x = (Xd,)
    if q_csr:
        qrp, qcol, qval = _csr(Q)
        nq = qrp.size - 1
        qargs = [null_d, qrp.ctypes.data_as(C.POINTER(C.c_int64)), qcol.ctypes.data_as(C.POINTER(C.c_int32)),
                 qval.ctypes.data_as(C.POINTER(C.c_double))]
        keep_q = (qrp, qcol, qval)
    else:
        Qd = _f64(Q)
        nq = Qd.shape[0]
        qargs = [Qd.ctypes.data_as(C.POINTER(C.c_double)), null_i64, null_i32, null_d]
        keep_q = (Qd,)
    ids = np.empty((nq, knn), np.int64)
    d2 = np.empty((nq, knn), np.float64)
    gap = np.empty(nq, np.float64)
    f = lib().orc_query
    f.restype = None
    f(C.c_int(L), kpl.ctypes.data_as(C.POINTER(C.c_int64)), _ptr_array(Pd, C.c_double),
      _ptr_array(Of, C.c_int64), _ptr_array(Me, C.c_int64), C.c_int(d), *xargs,
      C.c_int64(nq), *qargs, C.c_int(knn), C.c_int(beam),
      ids.ctypes.data_as(C.POINTER(C.c_int64)), d2.ctypes.data_as(C.POINTER(C.c_double)),
      gap.ctypes.data_as(C.POINTER(C.c_double)))
    del keep_x, keep_q
    return ids, d2, gap


def knn_exact(X, Q, knn: int, csr: bool = False):
    """Brute-force exact k-NN by (d^2, id): ids, d2, relative gap between k-th and (k+1)-th."""
    null_d = C.POINTER(C.c_double)()
    null_i64 = C.POINTER(C.c_int64)()
    null_i32 = C.POINTER(C.c_int32)()
    if csr:
        xrp, xcol, xval = _csr(X)
        qrp, qcol, qval = _csr(Q)
        n, nq, d = xrp.size - 1, qrp.size - 1, 0
        xargs = [null_d, xrp.ctypes.data_as(C.POINTER(C.c_int64)), xcol.ctypes.data_as(C.POINTER(C.c_int32)),
                 xval.ctypes.data_as(C.POINTER(C.c_double))]
        qargs = [null_d, qrp.ctypes.data_as(C.POINTER(C.c_int64)), qcol.ctypes.data_as(C.POINTER(C.c_int32)),
                 qval.ctypes.data_as(C.POINTER(C.c_double))]
        keep = (xrp, xcol, xval, qrp, qcol, qval)
    else:
        Xd, Qd = _f64(X), _f64(Q)
        n, d = Xd.shape
        nq = Qd.shape[0]
        xargs = [Xd.ctypes.data_as(C.POINTER(C.c_double)), null_i64, null_i32, null_d]
        qargs = [Qd.ctypes.data_as(C.POINTER(C.c_double)), null_i64, null_i32, null_d]
        keep = (Xd, Qd)
    ids = np.empty((nq, knn), np.int64)
    d2 = np.empty((nq, knn), np.float64)
    gap = np.empty(nq, np.float64)
    f = lib().orc_knn_exact
    f.restype = None
    f(C.c_int64(n), C.c_int(d), *xargs, C.c_int64(nq), *qargs, C.c_int(knn),
      ids.ctypes.data_as(C.POINTER(C.c_int64)), d2.ctypes.data_as(C.POINTER(C.c_double)),
      gap.ctypes.data_as(C.POINTER(C.c_double)))
    del keep
    return ids, d2, gap


def recall(result_ids: np.ndarray, exact_ids: np.ndarray) -> float:
    """recall@k = |result ∩ exact| / k averaged over queries (padding ids -1 never match)."""
    nq, k = exact_ids.shape
    hits = 0
    for r, e in zip(result_ids, exact_ids):
        hits += len(set(int(v) for v in r if v >= 0) & set(int(v) for v in e))
    return hits / float(nq * k) if nq else 1.0
