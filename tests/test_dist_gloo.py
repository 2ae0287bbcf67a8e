"""World-size-2 `gloo` tests (CPU) of the row-sharded data-parallel Lloyd step that mask_build
runs over NCCL on B200s (BASELINE.json north_star: points sharded, prototypes replicated, one
allreduce of [sums | counts] per iteration; queries sharded by batch).

Each rank owns rows shard.row_range(N, W, r) of the same seeded dataset; the per-rank partial
cluster sums/counts (FP64 oracle) are combined with all_reduce(SUM) and turned into means,
which must equal the single-process oracle update; the init-row gather (owners contribute
their rows, everyone else zeros, then SUM) must reproduce Y[init_idx] exactly; the
batch-sharded query results concatenated in rank order must equal the unsharded ones.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_2208_02734_b200.shard import query_range, row_range


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = datagen.CONFIGS[2].scaled(256)
        X = datagen.data(cfg).astype(np.float64)
        N, d = X.shape
        lo, hi = row_range(N, world, rank)
        Xl = datagen.data(cfg, lo, hi - lo).astype(np.float64)
        assert np.array_equal(Xl, X[lo:hi])  # block-seeded generator: shards are slices
        k = cfg.levels[0]
        init = datagen.init_indices(cfg.cid, 1, N, k)
        # ---- init gather: owners contribute their rows, the rest zeros, then SUM
        P0 = np.zeros((k, d))
        own = (init >= lo) & (init < hi)
        P0[own] = Xl[init[own] - lo]
        t = torch.from_numpy(P0)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        P = t.numpy()
        assert np.array_equal(P, X[init])
        # ---- three data-parallel Lloyd iterations
        for _ in range(3):
            lab, _, _ = oracle.assign(Xl, P)
            S, cnt = oracle.cluster_sums(Xl, lab, k)
            tS, tc = torch.from_numpy(S), torch.from_numpy(cnt)
            dist.all_reduce(tS, op=dist.ReduceOp.SUM)
            dist.all_reduce(tc, op=dist.ReduceOp.SUM)
            P_new, _ = oracle.means_from_sums(tS.numpy(), tc.numpy(), P)
            # reference: the unsharded update
            lab_all, _, _ = oracle.assign(X, P)
            P_ref, _ = oracle.means(X, lab_all, P)
            np.testing.assert_allclose(P_new, P_ref, rtol=1e-12, atol=1e-12)
            P = P_new
        # ---- batch-sharded queries over a replicated index
        idx = oracle.build_index(X, [init, datagen.init_indices(cfg.cid, 2, k, cfg.levels[1])], 3)
        Q = datagen.queries(cfg, count=37)
        qlo, qhi = query_range(len(Q), world, rank)
        ids, d2, _ = oracle.query(idx.P, idx.offsets, idx.members, X, Q[qlo:qhi], 5, 1)
        parts = [None] * world
        dist.all_gather_object(parts, (qlo, ids))
        if rank == 0:
            got = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])], axis=0)
            ref, _, _ = oracle.query(idx.P, idx.offsets, idx.members, X, Q, 5, 1)
            np.testing.assert_array_equal(got, ref)
            open(os.path.join(out_dir, "ok"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_data_parallel_lloyd_and_query_sharding_gloo(tmp_path):
    oracle.build()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").exists()


def _cluster_worker(rank, world, port, out_dir):
    """§3.4 distributed mode host plumbing: each rank is a node with its own index
    (the oracle's, built from its rows only), the registry / query / answer exchanges of
    paper_2208_02734_b200.cluster, and the merge, against the single-process oracle."""
    from paper_2208_02734_b200.cluster import gather_queries, gather_registry, return_answers
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = datagen.gaussian_clouds(61, 120, radius=15.0, sigma=1.0).astype(np.float64)
        X = X[datagen.group_perm(61, X.shape[0])]
        n = X.shape[0]
        bounds = [(r * n // world, (r + 1) * n // world) for r in range(world)]
        levels = [(12, 3), (10, 5)]  # different top sizes per node: ragged registry
        nodes = []
        for r, (lo, hi) in enumerate(bounds):
            k1, k2 = levels[r]
            idx = oracle.build_index(X[lo:hi], [datagen.init_indices(62 + r, 1, hi - lo, k1),
                                                datagen.init_indices(62 + r, 2, k1, k2)], 6)
            nodes.append(dict(P=idx.P, offsets=idx.offsets, members=idx.members, X=X[lo:hi], id_base=lo))
        me = nodes[rank]
        top = oracle.top_registry(me["P"][-1], me["offsets"][-1]).astype(np.float32)
        tops, bases = gather_registry(top, bounds[rank][1] - bounds[rank][0], 2)
        assert bases == [lo for lo, _ in bounds]
        for nd, tp in zip(nodes, tops):
            np.testing.assert_array_equal(tp, oracle.top_registry(nd["P"][-1], nd["offsets"][-1]).astype(np.float32))
        Q = datagen.gaussian_clouds(63, 5, radius=15.0, sigma=1.0).astype(np.float32)  # 40 queries
        qlo, qhi = query_range(len(Q), world, rank)
        Qall, counts = gather_queries(torch.from_numpy(Q[qlo:qhi]))
        assert np.array_equal(Qall.numpy(), Q)
        for eps in (np.inf, 4.0):
            # this node answers the queries routed to it (the rest padded), global ids
            ids, d2, _ = oracle.query(me["P"], me["offsets"], me["members"], me["X"], Qall.numpy(), 5, 1)
            ids = np.where(ids >= 0, ids + me["id_base"], -1)
            for i in range(len(Q)):
                if rank not in oracle.route(tops, Qall.numpy()[i], eps)[0]:
                    ids[i], d2[i] = -1, np.inf
            ai, ad = return_answers(torch.from_numpy(ids), torch.from_numpy(d2), counts)
            assert ai.shape == (world, qhi - qlo, 5)
            got = [oracle.merge([(ai[n, i].numpy(), ad[n, i].numpy()) for n in range(world)], range(world), 5)
                   for i in range(qhi - qlo)]
            ref_i, ref_d, _, _ = oracle.cluster_query(nodes, Q, 5, 1, eps)
            np.testing.assert_array_equal(np.stack([g[0] for g in got]), ref_i[qlo:qhi])
            np.testing.assert_array_equal(np.stack([g[1] for g in got]), ref_d[qlo:qhi])
        dist.barrier()
        if rank == 0:
            open(os.path.join(out_dir, "ok"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_distributed_mode_exchanges_gloo(tmp_path):
    oracle.build()
    port = _free_port()
    mp.spawn(_cluster_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").exists()


def _host_coll_worker(rank, world, port, out_dir):
    """The host transport of libmask's communicator (api.host_collective, the function
    mask_comm_init_host calls) over gloo: every kind and dtype the library issues."""
    import ctypes as C

    from paper_2208_02734_b200 import _lib
    from paper_2208_02734_b200.api import host_collective

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for dt, code in [(np.float32, 0),
                         (np.float64, 1), (np.int32, 2), (np.int64, 3), (np.uint64, 4)]:
            a = (np.arange(6) + 10 * rank).astype(dt)
            assert host_collective(_lib.MASK_COLL_ALLREDUCE, a.ctypes.data, None, a.size, code, _lib.MASK_COLL_SUM) == 0
            np.testing.assert_array_equal(a, sum((np.arange(6) + 10 * r) for r in range(world)).astype(dt))
            b = (np.arange(4) * (rank + 1)).astype(dt)
            assert host_collective(_lib.MASK_COLL_ALLREDUCE, b.ctypes.data, None, b.size, code, _lib.MASK_COLL_MAX) == 0
            np.testing.assert_array_equal(b, (np.arange(4) * world).astype(dt))
            c = np.full(5, rank + 7, dt)
            assert host_collective(_lib.MASK_COLL_BROADCAST, c.ctypes.data, None, c.size, code, world - 1) == 0
            np.testing.assert_array_equal(c, np.full(5, world - 1 + 7, dt))
            s = np.full(3, rank, dt)
            g = np.zeros(3 * world, dt)
            assert host_collective(_lib.MASK_COLL_ALLGATHER, g.ctypes.data, s.ctypes.data, 3, code, 0) == 0
            np.testing.assert_array_equal(g, np.repeat(np.arange(world), 3).astype(dt))
        # u64 sums beyond 2^63 keep their bits (summed as int64 two's complement)
        u = np.array([2 ** 63 + rank], np.uint64)
        assert host_collective(_lib.MASK_COLL_ALLREDUCE, u.ctypes.data, None, 1, 4, _lib.MASK_COLL_SUM) == 0
        assert int(u[0]) == (world * 2 ** 63 + sum(range(world))) % 2 ** 64
        # an unknown kind is reported as a failure (the library turns it into MASK_ERR_NCCL)
        z = np.zeros(1, np.float32)
        assert host_collective(9, z.ctypes.data, None, 1, 0, 0) != 0
        open(os.path.join(out_dir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


def test_host_collective_transport_gloo(tmp_path):
    world = 2
    mp.spawn(_host_coll_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"ok{r}").exists()
