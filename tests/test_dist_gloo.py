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
