"""GPU parity of dynamic insertion through the C-ABI: the
partition each new point joins equals the oracle's insertion path over the same index (tie
window exempt), child lists are rebuilt with the new rows, prototypes are unchanged, and an
inserted vector is found by a subsequent query (insert closure)."""
import numpy as np
import pytest

import datagen
import oracle
from parity import TIE_REL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402


@pytest.mark.parametrize("cid,div,borrow", [(2, 64, False), (1, 2, True), (3, 1024, False)])
def test_insert_parity_and_closure(cid, div, borrow):
    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    Xd = torch.from_numpy(X).cuda()
    idx = mk.build(Xd, cfg.levels, 5, datagen.all_init_indices(cfg), flags=mk.MASK_BORROW_DATA if borrow else 0)
    L = idx.num_levels
    P = [idx.prototypes(l) for l in range(1, L + 1)]
    ch = [idx.children(l) for l in range(1, L + 1)]
    new = datagen.queries(cfg, count=300)
    part = idx.insert(torch.from_numpy(new).cuda()).cpu().numpy()
    n = X.shape[0]
    for i, q in enumerate(new):
        j, gap = oracle.descend_leaf([p.astype(np.float64) for p in P], [c[0] for c in ch], [c[1] for c in ch], q)
        assert part[i] == j or gap < TIE_REL, f"point {i}: partition {part[i]} vs oracle {j}"
    for l in range(1, L + 1):
        np.testing.assert_array_equal(idx.prototypes(l), P[l - 1])  # prototypes unchanged
    lab = idx.labels(1)
    assert lab.shape[0] == n + len(new)
    np.testing.assert_array_equal(lab[n:], part)
    off, mem = idx.children(1)
    o_ref, m_ref = oracle.children(lab, cfg.levels[0])
    np.testing.assert_array_equal(off, o_ref)
    np.testing.assert_array_equal(mem, m_ref)
    ids, d2 = idx.query(torch.from_numpy(new).cuda(), knn=1)
    ids = ids.cpu().numpy()[:, 0]
    np.testing.assert_array_equal(ids, np.arange(n, n + len(new)))  # closure: found at distance 0
    assert float(d2.max()) == 0.0
    # a second insertion continues the ids
    part2 = idx.insert(np.ascontiguousarray(new[:5] + 1e-3))
    assert part2.shape == (5,) and idx.labels(1).shape[0] == n + len(new) + 5
    idx.free()


def _index_state(idx):
    L = idx.num_levels
    return ([idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)],
            [idx.labels(l).astype(np.int64) for l in range(1, L + 1)])


@pytest.mark.parametrize("cid,div,thr", [(2, 64, 300), (3, 2048, 100), (5, 4096, 120)])
def test_split_partitions_parity(cid, div, thr):
    """Partition split + local rebuild (reading S1).  Each split partition's local
    Lloyd run is (a) the library's own level build of those rows from the same seeded init --
    pinned by rebuilding it with mask_build (MASK_TRACE_PASSES) and comparing -- and (b) checked
    pass by pass against the FP64 oracle's run (parity.check_trajectory: in sync within 1e-4, or
    parting only at a near-tie row, D15).  The index around it: the new ids and their
    level-2 parents equal oracle.split_partitions', every other partition and upper level is
    untouched, child lists = {i : labels = j}, and queries over the rebuilt index equal the
    oracle descent over it."""
    from parity import check_assignment, check_queries, check_trajectory, rel_l2

    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    idx = mk.build(torch.from_numpy(X).cuda(), cfg.levels, 6, datagen.all_init_indices(cfg))
    P0, L0 = _index_state(idx)
    nsplit = idx.split(thr, iters=8, seed=11)
    Pr, Lr, split = oracle.split_partitions(P0, L0, X, threshold=thr, T=8, seed=11)
    assert nsplit == len(split) and nsplit > 0
    P1, L1 = _index_state(idx)
    assert P1[0].shape == Pr[0].shape
    k1 = P0[0].shape[0]
    counts = np.bincount(L0[0], minlength=k1)
    X64 = X.astype(np.float64)
    nxt = k1
    for j in split:
        rows = np.nonzero(L0[0] == j)[0]
        s_j = -(-int(counts[j]) // thr)
        ids = [j] + list(range(nxt, nxt + s_j - 1))
        nxt += s_j - 1
        init = mk.seeded_init(11 + j, 1, len(rows), s_j)
        np.testing.assert_array_equal(init, oracle.seeded_init(11 + j, 1, len(rows), s_j))
        loc = mk.build(torch.from_numpy(np.ascontiguousarray(X[rows])).cuda(), [s_j], 8, [init],
                       flags=mk.MASK_TRACE_PASSES)
        # (a) the split ran the library's level build on these rows
        assert rel_l2(P1[0][ids], loc.prototypes(1)) <= 1e-6, f"partition {j}: split != local build"
        loc_lab = np.asarray(ids)[loc.labels(1)]
        if not np.array_equal(L1[0][rows], loc_lab):
            check_assignment(X64[rows], P1[0][ids], np.searchsorted(ids, L1[0][rows]), what=f"split {j} labels")
        # (b) the local build against the oracle's Lloyd run, pass by pass
        ref = oracle.lloyd(X64[rows], init, 8, trace=True).passes
        check_trajectory(X64[rows], loc.passes(1), ref, what=f"split partition {j}")
        loc.free()
        if len(P1) > 1:
            assert np.all(L1[1][ids] == Lr[1][ids])  # new prototypes under j's parent
    for l in range(1, len(P1)):
        np.testing.assert_array_equal(P1[l], P0[l])  # upper levels untouched
        np.testing.assert_array_equal(L1[l], Lr[l])
    same = np.isin(L0[0], split, invert=True)
    np.testing.assert_array_equal(L1[0][same], L0[0][same])
    untouched = np.setdiff1d(np.arange(k1), split)
    np.testing.assert_array_equal(P1[0][untouched], P0[0][untouched])
    for l in range(1, len(P1) + 1):
        off, mem = idx.children(l)
        o_ref, m_ref = oracle.children(L1[l - 1], P1[l - 1].shape[0])
        np.testing.assert_array_equal(off, o_ref)
        np.testing.assert_array_equal(mem, m_ref)
    Q = datagen.queries(cfg, count=200)
    ch = [idx.children(l) for l in range(1, len(P1) + 1)]
    rids, rd2, gap = oracle.query(P1, [c[0] for c in ch], [c[1] for c in ch], X, Q, 10, 2)
    ids_q, d2 = idx.query(torch.from_numpy(Q).cuda(), knn=10, beam=2)
    check_queries(ids_q.cpu().numpy(), d2.cpu().numpy(), rids, rd2, gap, what="queries after the split")
    assert idx.split(thr * 1000, iters=8) == 0  # nothing above the threshold: no change
    idx.free()


def test_insert_then_split_restores_the_partition_size():
    """The paper's scenario: many new points land in one region, its partition grows past the
    threshold, and the split rebuilds only that part; inserted points stay findable."""
    cfg = datagen.CONFIGS[2].scaled(64)
    X = datagen.data(cfg)
    idx = mk.build(torch.from_numpy(X).cuda(), cfg.levels, 6, datagen.all_init_indices(cfg))
    P1 = idx.prototypes(1)
    rng = np.random.default_rng(5)
    new = (P1[7] + 0.3 * rng.standard_normal((2000, cfg.dim))).astype(np.float32)
    part = idx.insert(torch.from_numpy(new).cuda()).cpu().numpy()
    k_before = idx.level_info(1)["k"]
    big = np.bincount(idx.labels(1), minlength=k_before).max()
    thr = 600
    assert big > thr
    ns = idx.split(thr, iters=10, seed=3)
    assert ns >= 1 and idx.level_info(1)["k"] > k_before
    sizes = np.bincount(idx.labels(1), minlength=idx.level_info(1)["k"])
    assert sizes.sum() == X.shape[0] + len(new)
    assert sizes.max() < big
    ids, d2 = idx.query(torch.from_numpy(new[:50]).cuda(), knn=1, beam=4)
    assert float(d2.cpu().numpy().min()) == 0.0
    idx.free()
