"""Relocation and rebuild (§5.1; Table 1):
after a grouped build (Algorithm 1), every point is searched for (beam-1 descent, 1-NN); a
point the search does not return is "reassigned to that partition" the search reached, and
the index is rebuilt over the relocated data layer; the error rate is recorded after every
build.

Each build and each exhaustive point search runs in libmask's kernels (K12, K9).  Between
builds the loop does the relocation bookkeeping on the host (reading G8): a found
point keeps its data-layer group, a missed one targets the group of the partition its search
reached (group-major prototype id // nCentroids); the new data-layer order lists the target
groups in order with the points of a group ordered by the iteration's seeded keys (the rebuild
seed policy seed = base + i, passed in by the caller), and the rebuild splits that order into
the same number of balanced groups.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import numpy as np

from . import api


def _groups_of(order: np.ndarray, n_groups: int) -> np.ndarray:
    n = order.size
    base, rem = divmod(n, n_groups)
    sizes = np.full(n_groups, base, np.int64)
    sizes[n_groups - rem:] += 1
    g = np.empty(n, np.int64)
    g[order] = np.repeat(np.arange(n_groups), sizes)
    return g


def relocate_and_rebuild(X, length_group: int, n_centroids: int, iters: int, perm: np.ndarray, iterations: int,
                         keys_fn: Callable[[int, int], np.ndarray],
                         hook: Optional[Callable] = None) -> List[float]:
    """Error rates of the first build and of each of ``iterations`` relocation rebuilds.

    X: device tensor (n x d fp32); perm: the first build's data-layer order; keys_fn(i, n): the
    order keys of iteration i (i >= 1).  hook(i, order, index, found, reached_group) is called
    after every build's point search (tests); the index is freed afterwards."""
    n = int(X.shape[0])
    depth, layer_k = api.grouped_depth(n, length_group, n_centroids)
    if depth < 1:
        raise ValueError("no centroid layer: fewer points than length_group")
    n_groups = layer_k[0] // n_centroids
    order = np.ascontiguousarray(perm, np.int64)
    errors = []
    for i in range(iterations + 1):
        idx = api.build_grouped(X, length_group, n_centroids, iters, perm=order)
        ids, _ = idx.query(X, knn=1, beam=1)  # exhaustive point search (K9)
        got = ids[:, 0].cpu().numpy()
        found = got == np.arange(n)
        errors.append(float(np.mean(~found)))
        lab1 = idx.labels(1)
        reached = np.where(got >= 0, lab1[np.maximum(got, 0)] // n_centroids, -1)
        if hook is not None:
            hook(i, order, idx, found, reached)
        idx.free()
        if i == iterations:
            break
        # found points, and searches that reached no partition (reached < 0), stay in place
        target = np.where(found | (reached < 0), _groups_of(order, n_groups), reached)
        keys = np.asarray(keys_fn(i + 1, n), np.int64)
        order = np.lexsort((keys, target)).astype(np.int64)
    return errors
