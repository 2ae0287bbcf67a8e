"""GPU parity of the §3.4 distributed mode through the C-ABI:
independent per-node builds (zero NCCL calls), the registry of top-level prototypes with
children, K14 routing against the oracle's strict-epsilon rule, the routed per-node descents and
the (d^2, node, id) merge against ``oracle.cluster_query`` over the GPU-built node structures
(the build itself is covered by test_gpu_parity).  Queries whose routing distance lies within
1e-5 relative of epsilon, or whose descent meets a near tie, are exempt (FP32 vs FP64)."""
import math

import numpy as np
import pytest

import datagen
import oracle
from parity import TIE_REL, check_queries

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402
from paper_2208_02734_b200.cluster import LocalCluster  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _split(n, W, sizes=None):
    if sizes is None:
        return [(r * n // W, (r + 1) * n // W) for r in range(W)]
    b = np.concatenate([[0], np.cumsum(sizes)])
    return [(int(b[r]), int(b[r + 1])) for r in range(len(sizes))]


def _oracle_nodes(cl, parts_np, bounds, csr=False):
    nodes = []
    for nd, Xp, (lo, _) in zip(cl.nodes, parts_np, bounds):
        L = nd.num_levels
        ch = [nd.children(l) for l in range(1, L + 1)]
        nodes.append(dict(P=[nd.prototypes(l) for l in range(1, L + 1)], offsets=[c[0] for c in ch],
                          members=[c[1] for c in ch], X=Xp, id_base=lo))
    return nodes


def _route_gap(nodes, Qv, eps):
    tops = [oracle.top_registry(nd["P"][-1], nd["offsets"][-1]) for nd in nodes]
    return np.array([oracle.route(tops, q, eps)[1] for q in Qv])


def _check(cl, onodes, Q, Qv, knn, beam, eps, csr_dim=None, Qdev=None):
    ids, d2, routed, stats = cl.knn(Qdev if Qdev is not None else t(Q), knn=knn, epsilon=eps, beam=beam)
    ids_ref, d2_ref, routed_ref, gap = oracle.cluster_query(onodes, Q, knn, beam, eps, csr_dim=csr_dim)
    rgap = _route_gap(onodes, Qv, eps)
    r = routed.cpu().numpy().astype(bool)
    ok = (r == routed_ref).all(axis=1) | (rgap < TIE_REL)
    assert ok.all(), f"routing differs on {np.nonzero(~ok)[0][:5].tolist()}"
    check_queries(ids.cpu().numpy(), d2.cpu().numpy(), ids_ref, d2_ref, gap, what=f"cluster eps={eps} beam={beam}")
    assert stats["routed_pairs"] == int(r.sum()) and stats["empty_route"] == int((~r.any(axis=1)).sum())
    return ids, d2, r


def test_cluster_paper_example_eight_clouds():
    # Figure "cluster": clouds split into random partitions, one per node, so any
    # cloud appears in every node; 4 nodes, small per-node hierarchies
    X = datagen.gaussian_clouds(31, 500, radius=20.0, sigma=1.0)
    perm = datagen.group_perm(31, X.shape[0])
    X = X[perm]
    W = 4
    bounds = _split(X.shape[0], W)
    parts = [X[lo:hi] for lo, hi in bounds]
    levels = [16, 4]
    inits = [[datagen.init_indices(300 + r, 1, hi - lo, 16), datagen.init_indices(300 + r, 2, 16, 4)]
             for r, (lo, hi) in enumerate(bounds)]
    c0 = mk.collective_count()
    cl = LocalCluster.build([t(p) for p in parts], levels, 10, inits)
    assert cl.build_collectives == 0 and mk.collective_count() == c0  # zero-communication build
    assert cl.registry.n_nodes == W and sum(cl.registry.counts) <= W * 4
    onodes = _oracle_nodes(cl, parts, bounds)
    Q = datagen.gaussian_clouds(32, 25, radius=20.0, sigma=1.0)
    for eps in (math.inf, 6.0, 2.5, 1.0):
        for beam in (1, 3):
            _check(cl, onodes, Q, Q.astype(np.float64), 10, beam, eps)
    # eps = inf equals the merge of the nodes' own mask_query answers (broadcast equivalence)
    ids, d2, _, _ = cl.knn(t(Q), knn=10, epsilon=math.inf)
    own = [nd.query(t(Q), knn=10) for nd in cl.nodes]
    gi = torch.stack([torch.where(a[0] >= 0, a[0] + lo, a[0]) for a, (lo, _) in zip(own, bounds)])
    mi, md = mk.merge(gi, torch.stack([a[1] for a in own]))
    assert torch.equal(mi, ids) and torch.equal(md, d2)
    # eps = 0 routes nowhere (strict): all padding, every query flagged in the stats
    ids, d2, routed, stats = cl.knn(t(Q), knn=10, epsilon=0.0)
    assert (ids == -1).all() and torch.isinf(d2).all() and stats["empty_route"] == Q.shape[0]
    cl.free()


def test_cluster_ragged_nodes_and_single_node():
    cfg = datagen.CONFIGS[2].scaled(512)
    X = datagen.data(cfg)
    n = X.shape[0]
    sizes = [n - 9 - 700, 700, 9]  # one node smaller than k_nn: its answers are padded
    bounds = _split(n, 3, sizes)
    parts = [X[lo:hi] for lo, hi in bounds]
    levels = [4, 2]
    inits = [[datagen.init_indices(310 + r, 1, hi - lo, 4), datagen.init_indices(310 + r, 2, 4, 2)]
             for r, (lo, hi) in enumerate(bounds)]
    cl = LocalCluster.build([t(p) for p in parts], levels, 8, inits)
    onodes = _oracle_nodes(cl, parts, bounds)
    Q = datagen.queries(cfg, count=70)
    d_top = np.sqrt(((Q[:, None, :].astype(np.float64) - cl.registry.protos.cpu().numpy()[None]) ** 2).sum(-1))
    for eps in (math.inf, float(np.median(d_top)), float(np.percentile(d_top, 10))):
        _check(cl, onodes, Q, Q.astype(np.float64), 10, 2, eps)
    cl.free()
    # one node: the cluster answer is that node's own descent
    one = LocalCluster.build([t(X)], [32, 4], 6, [[datagen.init_indices(320, 1, n, 32), datagen.init_indices(320, 2, 32, 4)]])
    ids, d2, _, _ = one.knn(t(Q), knn=7)
    ids0, d20 = one.nodes[0].query(t(Q), knn=7)
    assert torch.equal(ids, ids0) and torch.equal(d2, d20)
    one.free()


def test_cluster_sparse_nodes():
    # C4-shaped CSR nodes: CSR routing (||c||^2 + sum q_p^2 - 2 q_p c_p) and CSR descents
    rp, col, val = datagen.random_csr(330, 2400, 500, 10)
    W, dim = 2, 500
    bounds = _split(2400, W)
    parts_np, parts = [], []
    for lo, hi in bounds:
        prp = rp[lo:hi + 1] - rp[lo]
        pc, pv = col[rp[lo]:rp[hi]], val[rp[lo]:rp[hi]]
        parts_np.append((prp, pc, pv))
        parts.append(mk.Csr(t(prp), t(pc), t(pv), dim))
    inits = [[datagen.init_indices(331 + r, 1, hi - lo, 24), datagen.init_indices(331 + r, 2, 24, 4)]
             for r, (lo, hi) in enumerate(bounds)]
    cl = LocalCluster.build(parts, [24, 4], 5, inits)
    onodes = _oracle_nodes(cl, parts_np, bounds)
    qrp, qcol, qval = datagen.random_csr(332, 60, dim, 10)
    Qv = np.zeros((60, dim))
    for i in range(60):
        Qv[i, qcol[qrp[i]:qrp[i + 1]]] = qval[qrp[i]:qrp[i + 1]]
    d_top = np.sqrt(((Qv[:, None, :] - cl.registry.protos.cpu().numpy()[None]) ** 2).sum(-1))
    for eps in (math.inf, float(np.median(d_top.min(axis=1)))):
        _check(cl, onodes, (qrp, qcol, qval), Qv, 5, 1, eps, csr_dim=dim,
               Qdev=mk.Csr(t(qrp), t(qcol), t(qval), dim))
    cl.free()


def test_route_and_merge_arguments():
    reg = t(np.zeros((2, 3), np.float32))
    node = t(np.array([0, 1], np.int32))
    Q = t(np.ones((4, 3), np.float32))
    with pytest.raises(mk.MaskError):
        mk.route(reg, node, 2, Q, -1.0)
    with pytest.raises(mk.MaskError):
        mk.route(reg, node, 0, Q, 1.0)
    r = mk.route(reg, node, 2, Q, math.inf)
    assert r.shape == (4, 2) and (r == 1).all()
    r = mk.route(reg, node, 2, Q[:0], 1.0)
    assert r.shape == (0, 2)
    with pytest.raises(mk.MaskError):
        mk.merge(torch.zeros((65, 1, 1), dtype=torch.int64, device="cuda"),
                 torch.zeros((65, 1, 1), dtype=torch.float32, device="cuda"))
    # merge: (d^2, node, id) order, equal distances resolved by the node number
    ids = t(np.array([[[5, 9, -1]], [[100, 101, 102]]], np.int64))
    d2 = t(np.array([[[1.0, 2.0, np.inf]], [[1.0, 1.5, 2.0]]], np.float32))
    mi, md = mk.merge(ids, d2)
    assert mi.cpu().tolist() == [[5, 100, 101]] and md.cpu().tolist() == [[1.0, 1.0, 1.5]]


def test_dist_cluster_nccl_single_rank():
    # DistCluster through its NCCL exchanges (registry all-gather, query all-gather, answer
    # all_to_all) in a one-rank process group; equal to LocalCluster over the same partition
    import os
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(here, "_dist_cluster_main.py")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "DIST_CLUSTER_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_merge_at_the_node_limit():
    # 64 nodes (the K14 merge limit) with random sorted answers: (d^2, node, id) merge = a
    # host sort of the union
    rng = np.random.default_rng(5)
    W, nq, k = 64, 40, 7
    d2 = np.sort(rng.integers(0, 30, size=(W, nq, k)).astype(np.float32), axis=2)
    ids = rng.integers(0, 10**6, size=(W, nq, k)).astype(np.int64)
    ids[:, :, -1] = np.where(rng.random((W, nq)) < 0.3, -1, ids[:, :, -1])
    d2 = np.where(ids < 0, np.inf, d2).astype(np.float32)
    for n in range(W):  # every node's answer sorted by (d^2, id), padding last (the contract)
        for q in range(nq):
            o = np.lexsort((np.where(ids[n, q] < 0, np.iinfo(np.int64).max, ids[n, q]), d2[n, q]))
            ids[n, q], d2[n, q] = ids[n, q][o], d2[n, q][o]
    mi, md = mk.merge(t(ids), t(d2))
    mi, md = mi.cpu().numpy(), md.cpu().numpy()
    for q in range(nq):
        cand = sorted((float(d2[n, q, r]), n, int(ids[n, q, r])) for n in range(W) for r in range(k) if ids[n, q, r] >= 0)
        ref = cand[:k]
        assert [c[2] for c in ref] == mi[q][:len(ref)].tolist()
        assert np.allclose([c[0] for c in ref], md[q][:len(ref)])
