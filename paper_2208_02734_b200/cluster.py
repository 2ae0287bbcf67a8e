"""The paper's distributed mode (§3.4 "Indexing distributed datasets", P:995-1034;
SURVEY §8(f) NEXT-3), on B200s: one node = one GPU.

* build: every node builds its own multilevel index over its own rows with ``comm=None`` --
  no collective at all (the zero-communication counter, ``collective_count()``, must not move;
  P:1005-1008 "each node can work with its own data partitions, in parallel with the rest of
  nodes").
* register: "just the top level centroids from each node need to be recorded":
  the registry is the concatenation of the nodes' top-level prototypes with children
  (``mask_top_prototypes``) and their node numbers; node n's rows get global ids
  ``id_base[n] + local id`` (id bases = exclusive prefix of the node row counts).
* query: K14 routes every query to the nodes with a registered centroid closer than epsilon
  (strict; epsilon = inf = all nodes), each routed node runs its own descent (K9)
  on the queries routed to it, and K14 merges the answers by (d^2, node, id).

``LocalCluster`` holds several node indexes in one process (e.g. partitions sharing one GPU);
``DistCluster`` is one node per ``torch.distributed`` rank (NCCL on B200s): queries are sharded
by batch, all-gathered so that every node can answer the ones routed to it, and the answers go
back to each query's owner with one ``all_to_all`` before the merge.  The exchange helpers are
plain ``torch.distributed`` plumbing (tested with ``gloo`` on CPU); every distance, routing
decision and merge runs in libmask's kernels.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import api


class Registry:
    """Coordinator metadata: registered top-level centroids (device R x d fp32), their node
    numbers (device int32), and the nodes' global id bases."""

    def __init__(self, tops: Sequence[np.ndarray], id_bases: Sequence[int], device):
        self.n_nodes = len(tops)
        d = next((t.shape[1] for t in tops if t.ndim == 2 and t.shape[0]), 1)
        rows = [np.asarray(t, np.float32).reshape(-1, d) for t in tops]
        self.counts = [r.shape[0] for r in rows]
        protos = np.concatenate(rows, axis=0) if sum(self.counts) else np.zeros((0, d), np.float32)
        self.protos = torch.from_numpy(np.ascontiguousarray(protos)).to(device)
        self.node_of = torch.from_numpy(np.repeat(np.arange(self.n_nodes, dtype=np.int32), self.counts)).to(device)
        self.id_bases = [int(b) for b in id_bases]

    def route(self, queries, epsilon: float, stream=None) -> torch.Tensor:
        return api.route(self.protos, self.node_of, self.n_nodes, queries, epsilon, stream=stream)


def _stats(routed: torch.Tensor) -> dict:
    per_q = routed.sum(dim=1)
    nq = int(routed.shape[0])
    return dict(queries=nq, nodes=int(routed.shape[1]), routed_pairs=int(per_q.sum()),
                skipped_pairs=int(routed.numel() - per_q.sum()), empty_route=int((per_q == 0).sum()))


class LocalCluster:
    """Several independent node indexes in one process (§3.4 with co-located nodes)."""

    def __init__(self, nodes: Sequence[api.Index], id_bases: Sequence[int], device, build_collectives: int = 0):
        self.nodes = list(nodes)
        self.registry = Registry([nd.top_prototypes() for nd in self.nodes], id_bases, device)
        self.build_collectives = build_collectives

    @classmethod
    def build(cls, parts: Sequence, levels: Sequence[int], iters: int, inits: Sequence[Sequence[np.ndarray]],
              id_bases: Optional[Sequence[int]] = None, **kw) -> "LocalCluster":
        """One independent ``mask_build`` per part (comm=None); ``inits[n]`` = part n's init
        indices per level.  Records the NCCL calls the builds issued (zero by construction)."""
        c0 = api.collective_count()
        nodes = [api.build(p, levels, iters, inits[n], **kw) for n, p in enumerate(parts)]
        c1 = api.collective_count()
        if id_bases is None:
            sizes = [int(p.shape[0]) if isinstance(p, torch.Tensor) else p.rows for p in parts]
            id_bases = np.concatenate([[0], np.cumsum(sizes)[:-1]]).tolist()
        p0 = parts[0]
        dev = p0.device if isinstance(p0, torch.Tensor) else p0.row_ptr.device
        return cls(nodes, id_bases, dev, build_collectives=c1 - c0)

    def knn(self, queries, knn: int = 10, epsilon: float = math.inf, beam: int = 1, stream=None):
        """Route, answer per routed node, merge.  Returns ids (global, int64), d2, routed, stats."""
        routed = self.registry.route(queries, epsilon, stream=stream)
        answers = [nd.query_routed(queries, routed, n, self.registry.id_bases[n], knn=knn, beam=beam, stream=stream)
                   for n, nd in enumerate(self.nodes)]
        ids = torch.stack([a[0] for a in answers])
        d2 = torch.stack([a[1] for a in answers])
        out_i, out_d = api.merge(ids, d2, stream=stream)
        return out_i, out_d, routed, _stats(routed)

    def free(self) -> None:
        for nd in self.nodes:
            nd.free()


# ---------------------------------------------------------------- torch.distributed plumbing
def gather_registry(top: np.ndarray, n_rows: int, dim: int, group=None, device="cpu") -> Tuple[List[np.ndarray], List[int]]:
    """All-gather every node's registered centroids (variable counts) and row counts; returns
    (tops per node, id bases).  Plain torch.distributed plumbing."""
    import torch.distributed as dist
    W = dist.get_world_size(group)
    meta = torch.tensor([top.shape[0], n_rows], dtype=torch.int64, device=device)
    metas = [torch.empty_like(meta) for _ in range(W)]
    dist.all_gather(metas, meta, group=group)
    counts = [int(m[0]) for m in metas]
    rows = [int(m[1]) for m in metas]
    cap = max(max(counts), 1)
    buf = torch.zeros((cap, dim), dtype=torch.float32, device=device)
    if top.shape[0]:
        buf[:top.shape[0]] = torch.from_numpy(np.ascontiguousarray(top, np.float32)).to(device)
    bufs = [torch.empty_like(buf) for _ in range(W)]
    dist.all_gather(bufs, buf, group=group)
    tops = [b[:c].cpu().numpy() for b, c in zip(bufs, counts)]
    bases = np.concatenate([[0], np.cumsum(rows)[:-1]]).astype(np.int64).tolist()
    return tops, bases


def gather_queries(q_local: torch.Tensor, group=None) -> Tuple[torch.Tensor, List[int]]:
    """All-gather the batch-sharded dense queries: (Q_all, per-rank counts)."""
    import torch.distributed as dist
    W = dist.get_world_size(group)
    n = torch.tensor([q_local.shape[0]], dtype=torch.int64, device=q_local.device)
    ns = [torch.empty_like(n) for _ in range(W)]
    dist.all_gather(ns, n, group=group)
    counts = [int(x) for x in ns]
    cap = max(max(counts), 1)
    buf = torch.zeros((cap, q_local.shape[1]), dtype=q_local.dtype, device=q_local.device)
    buf[:q_local.shape[0]] = q_local
    bufs = [torch.empty_like(buf) for _ in range(W)]
    dist.all_gather(bufs, buf, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)]), counts


def return_answers(ids: torch.Tensor, d2: torch.Tensor, counts: Sequence[int], group=None):
    """Send this node's answers for every query back to the query's owner (one all_to_all);
    returns (ids, d2) of shape (W, n_own, k): node-major answers for the owner's queries."""
    import torch.distributed as dist
    W = dist.get_world_size(group)
    r = dist.get_rank(group)
    k = ids.shape[1]
    own = counts[r]
    out_i = torch.empty((W * own, k), dtype=ids.dtype, device=ids.device)
    out_d = torch.empty((W * own, k), dtype=d2.dtype, device=d2.device)
    dist.all_to_all_single(out_i, ids.contiguous(), [own] * W, list(counts), group=group)
    dist.all_to_all_single(out_d, d2.contiguous(), [own] * W, list(counts), group=group)
    return out_i.view(W, own, k), out_d.view(W, own, k)


class DistCluster:
    """One §3.4 node per torch.distributed rank (one GPU each)."""

    def __init__(self, index: api.Index, registry: Registry, group=None, build_collectives: int = 0):
        self.index = index
        self.registry = registry
        self.group = group
        self.build_collectives = build_collectives

    @classmethod
    def build(cls, data_local, levels: Sequence[int], iters: int, init_idx: Sequence[np.ndarray], group=None,
              **kw) -> "DistCluster":
        import torch.distributed as dist
        c0 = api.collective_count()
        idx = api.build(data_local, levels, iters, init_idx, **kw)  # comm=None: independent
        c1 = api.collective_count()
        dev = data_local.device
        tops, bases = gather_registry(idx.top_prototypes(), int(data_local.shape[0]), int(data_local.shape[1]),
                                      group=group, device=dev)
        reg = Registry(tops, bases, dev)
        assert reg.n_nodes == dist.get_world_size(group)
        return cls(idx, reg, group, build_collectives=c1 - c0)

    def knn(self, q_local: torch.Tensor, knn: int = 10, epsilon: float = math.inf, beam: int = 1, stream=None):
        """This rank's query shard -> (ids, d2) of its queries after the cluster-wide search."""
        import torch.distributed as dist
        r = dist.get_rank(self.group)
        Q, counts = gather_queries(q_local, self.group)
        routed = self.registry.route(Q, epsilon, stream=stream)
        ids, d2 = self.index.query_routed(Q, routed, r, self.registry.id_bases[r], knn=knn, beam=beam, stream=stream)
        ai, ad = return_answers(ids, d2, counts, self.group)
        out_i, out_d = api.merge(ai, ad, stream=stream)
        lo = sum(counts[:r])
        return out_i, out_d, _stats(routed[lo:lo + counts[r]])

    def free(self) -> None:
        self.index.free()


__all__ = ["Registry", "LocalCluster", "DistCluster", "gather_registry", "gather_queries", "return_answers"]
