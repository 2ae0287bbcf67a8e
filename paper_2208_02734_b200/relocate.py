"""Relocation and rebuild (§5.1; Table 1):
after a grouped build (Algorithm 1), every point is searched for (beam-1 descent, 1-NN); a
point the search does not return is "reassigned to that partition" the search reached, and
the index is rebuilt over the relocated data layer; the error rate is recorded after every
build.

Each build (K12), each exhaustive point search (K9) and each relocation step (mask_relocate,
reading G8: found points keep their data-layer group, a missed one targets the group of the
partition its search reached, the next order lists the target groups in order with a group's
points ordered by the iteration's seeded keys) runs in libmask's kernels; this loop only
marshals arguments (the grouped build takes its data-layer order as a host array).
"""
from __future__ import annotations

from typing import Callable, List, Optional

import numpy as np
import torch

from . import api


def relocate_and_rebuild(X, length_group: int, n_centroids: int, iters: int, perm: np.ndarray, iterations: int,
                         keys_fn: Callable[[int, int], np.ndarray],
                         hook: Optional[Callable] = None) -> List[float]:
    """Error rates of the first build and of each of ``iterations`` relocation rebuilds.

    X: device tensor (n x d fp32); perm: the first build's data-layer order; keys_fn(i, n): the
    order keys of iteration i (i >= 1).  hook(i, order, index, found, reached_group) is called
    after every build's point search (tests; numpy views of the library's outputs); the index is
    freed afterwards."""
    n = int(X.shape[0])
    depth, _ = api.grouped_depth(n, length_group, n_centroids)
    if depth < 1:
        raise ValueError("no centroid layer: fewer points than length_group")
    dev = X.device
    order = torch.from_numpy(np.ascontiguousarray(perm, np.int64)).to(dev)
    errors = []
    for i in range(iterations + 1):
        idx = api.build_grouped(X, length_group, n_centroids, iters, perm=order.cpu().numpy())
        ids, _ = idx.query(X, knn=1, beam=1)  # exhaustive point search (K9)
        got = ids[:, 0].contiguous()
        keys = torch.from_numpy(np.ascontiguousarray(keys_fn(i + 1, n), np.int64)).to(dev) if i < iterations \
            else torch.zeros(n, dtype=torch.int64, device=dev)
        nxt, reached, misses = api.relocate(idx, got, order, keys, n_centroids)
        errors.append(misses / n)
        if hook is not None:
            found = (got == torch.arange(n, device=dev)).cpu().numpy()
            hook(i, order.cpu().numpy(), idx, found, reached.cpu().numpy())
        idx.free()
        if i == iterations:
            break
        order = nxt
    return errors
