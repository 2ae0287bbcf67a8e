"""The row-sharded multi-GPU build path of libmask (world > 1), run for real with two ranks.

The round's GPU boxes have one B200, so the two processes share it and their communicator is
libmask's host transport (mask_comm_init_host over gloo): the library drains its stream and
hands each collective's buffer to torch.distributed, so every world > 1 branch of mask_build
executes -- the parameter-hash agreement, the owner-gather init allreduce, the ONE packed
allreduce per Lloyd iteration (sums | counts | J | changed), the no-change stop decided from the
combined statistics, the end-of-level-1 label and row gathers, the rank-0 broadcast of the
upper levels -- while no kernel waits on another rank's kernel.  (With NCCL on an 8-GPU box the
same calls go to ncclAllReduce / ncclBroadcast / ncclAllGather.)

Checked against the FP64 oracle: the sharded build's level trajectories (labels of both shards
concatenated in rank order) by parity.check_trajectory, identical replicas on both ranks,
child lists over all N rows, batch-sharded queries vs the oracle descent, and the
argument-agreement error."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import datagen  # noqa: E402


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, cid, div, T, sparse_ok):
    import paper_2208_02734_b200 as mk
    from paper_2208_02734_b200.shard import query_range, row_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    comm = mk.Comm.host()
    try:
        cfg = datagen.CONFIGS[cid].scaled(div)
        inits = datagen.all_init_indices(cfg)
        lo, hi = row_range(cfg.n, world, rank)
        if cfg.sparse:
            rp, col, val = datagen.data(cfg, lo, hi - lo)
            data = mk.Csr(torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda(), torch.from_numpy(val).cuda(),
                          cfg.dim)
        else:
            data = torch.from_numpy(datagen.data(cfg, lo, hi - lo)).cuda()
        n0 = mk.collective_count()
        idx = mk.build(data, cfg.levels, T, inits, flags=mk.MASK_TRACE_PASSES, comm=comm, n_global=cfg.n,
                       row_offset=lo)
        ncoll = mk.collective_count() - n0
        out = {"ncoll": ncoll, "lo": lo, "hi": hi}
        for l in range(1, len(cfg.levels) + 1):
            out[f"P{l}"] = idx.prototypes(l)
            out[f"lab{l}"] = idx.labels(l)
            off, mem = idx.children(l)
            out[f"off{l}"], out[f"mem{l}"] = off, mem
            seq = idx.passes(l)
            out[f"npass{l}"] = len(seq)
            for t, (P, lab) in enumerate(seq):
                out[f"tP{l}_{t}"] = P
                out[f"tL{l}_{t}"] = lab
        # queries sharded by batch (no communication)
        if not cfg.sparse:
            Q = datagen.queries(cfg, count=256)
            qlo, qhi = query_range(len(Q), world, rank)
            ids, d2 = idx.query(torch.from_numpy(Q[qlo:qhi]).cuda(), knn=10)
            out["qids"], out["qd2"] = ids.cpu().numpy(), d2.cpu().numpy()
        idx.free()
        # ranks disagreeing on the parameters: MASK_ERR_ARG on every rank
        bad = [a.copy() for a in inits]
        if rank == 1:
            bad[0] = bad[0][::-1].copy()
        try:
            mk.build(data, cfg.levels, T, bad, comm=comm, n_global=cfg.n, row_offset=lo)
            out["mismatch"] = "no error"
        except mk.MaskError as e:
            out["mismatch"] = str(e)
        # the farthest-point empty repair is single-GPU: MASK_ERR_UNSUPPORTED on every rank
        try:
            mk.build(data, cfg.levels, T, inits, comm=comm, n_global=cfg.n, row_offset=lo, empty="farthest")
            out["farthest"] = "no error"
        except mk.MaskError as e:
            out["farthest"] = str(e)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **out)
    finally:
        comm.free()
        dist.destroy_process_group()


def _run(tmp_path, cid, div, T, world=2):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), cid, div, T, True), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]


@pytest.mark.parametrize("cid,div,T", [(2, 64, 25), (3, 512, 20), (4, 64, 10)])
def test_sharded_build_two_ranks(tmp_path, cid, div, T):
    import oracle
    from parity import check_queries, check_trajectory

    cfg = datagen.CONFIGS[cid].scaled(div)
    inits = datagen.all_init_indices(cfg)
    res = _run(tmp_path, cid, div, T)
    r0, r1 = res
    L = len(cfg.levels)
    # replicas: identical prototypes, labels (all N after the gather) and child lists
    for l in range(1, L + 1):
        np.testing.assert_array_equal(r0[f"P{l}"], r1[f"P{l}"])
        np.testing.assert_array_equal(r0[f"lab{l}"], r1[f"lab{l}"])
        np.testing.assert_array_equal(r0[f"off{l}"], r1[f"off{l}"])
        np.testing.assert_array_equal(r0[f"mem{l}"], r1[f"mem{l}"])
    assert len(r0["lab1"]) == cfg.n
    # collectives per build: the level-1 loop issues one allreduce per Lloyd iteration
    passes1 = int(r0["npass1"])
    updates = passes1 - 1
    assert r0["ncoll"] == r1["ncoll"]
    # hash (1) + init (1) + one per loop pass that ran (<= updates + 1) + final stats (1) +
    # gathers (2 scalars + labels/rows per rank) + upper-level broadcasts (2 per level)
    assert r0["ncoll"] >= updates + 3
    # level trajectories: the shards' labels concatenated in rank order = the global labels
    if cfg.sparse:
        rp, col, val = datagen.data(cfg)
        Y = (rp, col, val)
    else:
        X = datagen.data(cfg)
        Y = X.astype(np.float64)
    for l in range(1, L + 1):
        npass = int(r0[f"npass{l}"])
        assert npass == int(r1[f"npass{l}"])
        gpu = []
        for t in range(npass):
            if l == 1:  # both ranks finalize the same combined sums: bitwise-equal prototypes
                np.testing.assert_array_equal(r0[f"tP{l}_{t}"], r1[f"tP{l}_{t}"])
            lab = np.concatenate([r0[f"tL{l}_{t}"], r1[f"tL{l}_{t}"]]) if l == 1 else r0[f"tL{l}_{t}"]
            gpu.append((r0[f"tP{l}_{t}"], lab))
        csr_dim = cfg.dim if (cfg.sparse and l == 1) else None
        ref = oracle.lloyd(Y, inits[l - 1], T, csr_dim=csr_dim, trace=True).passes
        check_trajectory(Y, gpu, ref, csr_dim=csr_dim, what=f"{cfg.name} 2 ranks level {l}")
        np.testing.assert_array_equal(r0[f"lab{l}"], gpu[-1][1])
        Y = r0[f"P{l}"].astype(np.float64)
        o_ref, m_ref = oracle.children(r0[f"lab{l}"], cfg.levels[l - 1])
        np.testing.assert_array_equal(r0[f"off{l}"], o_ref)
        np.testing.assert_array_equal(r0[f"mem{l}"], m_ref)
    # batch-sharded queries = the oracle descent over the (replicated) index
    if not cfg.sparse:
        Q = datagen.queries(cfg, count=256)
        ids = np.concatenate([r0["qids"], r1["qids"]])
        d2 = np.concatenate([r0["qd2"], r1["qd2"]])
        P = [r0[f"P{l}"].astype(np.float64) for l in range(1, L + 1)]
        rids, rd2, gap = oracle.query(P, [r0[f"off{l}"] for l in range(1, L + 1)],
                                      [r0[f"mem{l}"] for l in range(1, L + 1)], X, Q, 10, 1)
        check_queries(ids, d2, rids, rd2, gap, what=f"{cfg.name} 2-rank queries")
    for r in res:
        assert "MASK_ERR_ARG" in str(r["mismatch"]) and "disagree" in str(r["mismatch"])
        assert "MASK_ERR_UNSUPPORTED" in str(r["farthest"])
