"""Pins for the FP64 oracle (oracle/) against things other than itself.

Each test pins the oracle to a value the paper/SPEC prints for a worked example, a closed
form, a special case that reduces to a library routine (scipy / numpy), brute force on a
tiny input, or an invariant of the method.  Chosen so that a dropped term, a wrong sign,
a wrong index, a transposed operand or a wrong tie rule fails at least one of them.
"""
import json
import os

import numpy as np
import pytest
from scipy.spatial.distance import cdist

import datagen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ distances
def test_dist_345_triangle():
    # SPEC.md:51 [TRIVIAL]: L2 (0,0)-(3,4) = 5  -> squared 25 (D9)
    assert oracle.dist2([0.0, 0.0], [3.0, 4.0]) == 25.0
    assert oracle.dist2([3.0, 4.0], [0.0, 0.0]) == 25.0
    assert oracle.dist2([1.5, -2.0], [1.5, -2.0]) == 0.0


def test_dist_matches_scipy():
    rng = np.random.default_rng(0)
    a = rng.standard_normal((7, 13))
    b = rng.standard_normal((5, 13))
    ref = cdist(a, b, "sqeuclidean")
    for i in range(7):
        for j in range(5):
            assert oracle.dist2(a[i], b[j]) == pytest.approx(ref[i, j], rel=1e-14)


def test_sparse_dense_identity_equals_densified():
    # sparse-dense distance == densified result (<= 1e-12 relative)
    rp, col, val = datagen.random_csr(5, 20, 300, 12)
    P = np.random.default_rng(1).standard_normal((9, 300))
    dense = np.zeros((20, 300))
    for i in range(20):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    ref = cdist(dense, P, "sqeuclidean")
    L = oracle.lib()
    for i in range(20):
        c = np.ascontiguousarray(col[rp[i]:rp[i + 1]], np.int32)
        v = np.ascontiguousarray(val[rp[i]:rp[i + 1]], np.float64)
        for j in range(9):
            cn2 = float(np.dot(P[j], P[j]))
            got = L.orc_dist2_csr_dense(c.size, c, v, np.ascontiguousarray(P[j]), cn2)
            assert got == pytest.approx(ref[i, j], rel=1e-12)
    # sparse {} vs (3,4): SPEC.md:61 distance from origin
    got = L.orc_dist2_csr_dense(0, np.zeros(1, np.int32), np.zeros(1), np.array([3.0, 4.0]), 25.0)
    assert got == 25.0
    # sparse-sparse union form == densified
    for i in range(19):
        a0, a1, b0, b1 = rp[i], rp[i + 1], rp[i + 1], rp[i + 2]
        got = L.orc_dist2_csr_csr(a1 - a0, np.ascontiguousarray(col[a0:a1]), np.ascontiguousarray(val[a0:a1], np.float64),
                                  b1 - b0, np.ascontiguousarray(col[b0:b1]), np.ascontiguousarray(val[b0:b1], np.float64))
        assert got == pytest.approx(float(((dense[i] - dense[i + 1]) ** 2).sum()), rel=1e-12)


# ------------------------------------------------------------------ assignment
def test_assign_brute_force_scipy():
    rng = np.random.default_rng(2)
    for n, d, k in [(50, 3, 7), (200, 16, 33), (31, 1, 5), (64, 9, 64)]:
        Y = rng.standard_normal((n, d))
        P = rng.standard_normal((k, d))
        lab, b1, b2 = oracle.assign(Y, P)
        D = cdist(Y, P, "sqeuclidean")
        assert np.array_equal(lab, D.argmin(axis=1))  # numpy argmin also returns the first minimum
        Ds = np.sort(D, axis=1)
        np.testing.assert_allclose(b1, Ds[:, 0], rtol=1e-13)
        if k > 1:
            np.testing.assert_allclose(b2, Ds[:, 1], rtol=1e-13)


def test_assign_ties_lowest_ordinal():
    # exact match -> that centroid; equidistant -> lowest ordinal (D4)
    lab, b1, _ = oracle.assign([[0.0, 0.0]], [[0.0, 0.0], [5.0, 5.0]])
    assert lab[0] == 0 and b1[0] == 0.0
    lab, _, _ = oracle.assign([[0.0, 0.0]], [[5.0, 5.0], [1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]])
    assert lab[0] == 1
    # duplicated prototypes: the lower copy wins
    lab, _, _ = oracle.assign([[2.0, 2.0]], [[9.0, 9.0], [2.0, 2.1], [2.0, 2.1]])
    assert lab[0] == 1


def test_assign_k1_second_is_inf():
    lab, b1, b2 = oracle.assign([[1.0], [2.0]], [[0.0]])
    assert list(lab) == [0, 0] and np.all(np.isinf(b2))


# ------------------------------------------------------------------ update
def test_means_against_numpy_add_at():
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((500, 6))
    k = 40
    lab = rng.integers(0, k - 3, size=500).astype(np.int32)  # last 3 clusters empty
    P_old = rng.standard_normal((k, 6))
    P_new, cnt = oracle.means(Y, lab, P_old)
    S = np.zeros((k, 6))
    np.add.at(S, lab, Y)
    c = np.bincount(lab, minlength=k)
    assert np.array_equal(cnt, c)
    nz = c > 0
    np.testing.assert_allclose(P_new[nz], S[nz] / c[nz, None], rtol=1e-13)
    assert np.array_equal(P_new[~nz], P_old[~nz])  # empty clusters keep their prototype (D5)


def test_cluster_sums_csr_equals_densified():
    rp, col, val = datagen.random_csr(7, 60, 50, 5)
    dense = np.zeros((60, 50))
    for i in range(60):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    lab = (np.arange(60) % 7).astype(np.int32)
    S1, c1 = oracle.cluster_sums_csr((rp, col, val), 50, lab, 7)
    S2, c2 = oracle.cluster_sums(dense, lab, 7)
    assert np.array_equal(c1, c2)
    np.testing.assert_allclose(S1, S2, rtol=0, atol=1e-15)


# ------------------------------------------------------------------ Lloyd
def test_golden_spec_s107_trajectories():
    g = json.load(open(os.path.join(GOLDEN, "spec_s107_two_clusters.json")))
    Y = np.array(g["points"], np.float64)
    for case in g["cases"]:
        r = oracle.lloyd(Y, np.array(case["init"]), T=10)
        np.testing.assert_array_equal(r.P, np.array(case["final_P"]))
        np.testing.assert_array_equal(r.labels, case["labels_per_pass"][-1])
        np.testing.assert_array_equal(r.J[:-1], case["J_per_pass"])  # passes before the final one
        assert r.J[-1] == case["final_J"]
        assert r.updates == case["updates"]
        # the per-pass labels: pass 0 from the init prototypes
        lab0, _, _ = oracle.assign(Y, Y[case["init"]])
        np.testing.assert_array_equal(lab0, case["labels_per_pass"][0])


def test_lloyd_empty_cluster_keeps_prototype_and_ties():
    # hand-derived: points 0,0,5 with both inits at 0 -> pass 0 all ties -> label 0 (lowest);
    # P0 <- mean(0,0,5)=5/3, P1 empty keeps 0; pass 1: 0,0 -> P1, 5 -> P0; P0 <- 5, P1 <- 0.
    Y = np.array([[0.0], [0.0], [5.0]])
    r = oracle.lloyd(Y, np.array([0, 1]), T=10)
    np.testing.assert_array_equal(r.P, [[5.0], [0.0]])
    np.testing.assert_array_equal(r.labels, [1, 1, 0])
    assert r.J[0] == 25.0 and r.J[-1] == 0.0


def test_lloyd_k1_is_global_mean():
    # SPEC.md:109 [TRIVIAL]: k = 1 -> the componentwise mean, labels all 0
    Y = datagen.random_dense(4, 300, 5, scale=3.0, offset=1.0).astype(np.float64)
    r = oracle.lloyd(Y, np.array([17]), T=3)
    np.testing.assert_allclose(r.P[0], Y.mean(axis=0), rtol=1e-12)
    assert np.all(r.labels == 0)
    assert r.J[-1] == pytest.approx(((Y - Y.mean(axis=0)) ** 2).sum(), rel=1e-12)


def test_lloyd_k_equals_n_identity():
    # SPEC.md:108 [TRIVIAL]: k = |points|, distinct points -> each point its own prototype, J = 0
    Y = datagen.random_dense(5, 40, 3).astype(np.float64)
    r = oracle.lloyd(Y, np.arange(40), T=5)
    np.testing.assert_array_equal(r.P, Y)
    np.testing.assert_array_equal(r.labels, np.arange(40))
    assert r.J[-1] == 0.0


def test_lloyd_monotone_and_fixed_point():
    # inertia non-increasing; labels = brute-force nearest; converged P = member means
    Y = datagen.blobs(6, 2000, 4, 8).astype(np.float64)
    idx = datagen.init_indices(99, 1, 2000, 50)
    r = oracle.lloyd(Y, idx, T=200)
    assert np.all(np.diff(r.J) <= 1e-12 * r.J[:-1])
    D = cdist(Y, r.P, "sqeuclidean")
    np.testing.assert_array_equal(r.labels, D.argmin(axis=1))
    assert r.changed[-1] == 0  # converged inside 200 iterations
    S = np.zeros_like(r.P)
    np.add.at(S, r.labels, Y)
    c = np.bincount(r.labels, minlength=50)
    np.testing.assert_allclose(r.P[c > 0], S[c > 0] / c[c > 0, None], rtol=1e-12)


def test_lloyd_T0_is_plain_assignment():
    Y = datagen.blobs(8, 300, 2, 4).astype(np.float64)
    idx = np.array([5, 60, 7])
    r = oracle.lloyd(Y, idx, T=0)
    np.testing.assert_array_equal(r.P, Y[idx])
    np.testing.assert_array_equal(r.labels, cdist(Y, Y[idx], "sqeuclidean").argmin(axis=1))
    assert r.updates == 0 and len(r.J) == 1


def test_lloyd_tol_stop():
    Y = datagen.blobs(9, 1000, 3, 5).astype(np.float64)
    idx = datagen.init_indices(98, 1, 1000, 20)
    r_inf = oracle.lloyd(Y, idx, T=3, tol=1e9)  # any displacement <= tol -> one update
    assert r_inf.updates == 1


def test_lloyd_csr_equals_densified():
    rp, col, val = datagen.random_csr(10, 120, 40, 6)
    dense = np.zeros((120, 40))
    for i in range(120):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    idx = datagen.init_indices(97, 1, 120, 9)
    a = oracle.lloyd((rp, col, val), idx, T=6, csr_dim=40)
    b = oracle.lloyd(dense, idx, T=6)
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_allclose(a.P, b.P, rtol=0, atol=1e-13)
    np.testing.assert_allclose(a.J, b.J, rtol=1e-12)


def test_children_lists():
    lab = np.array([2, 0, 2, 1, 2, 0], np.int32)
    off, mem = oracle.children(lab, 4)
    assert list(off) == [0, 2, 3, 6, 6]
    assert list(mem) == [1, 5, 3, 0, 2, 4]


# ------------------------------------------------------------------ queries
def _exact_numpy(X, Q, k):
    D = cdist(Q, X, "sqeuclidean")
    ids = np.array([np.lexsort((np.arange(X.shape[0]), row))[:k] for row in D])
    return ids, np.take_along_axis(D, ids, axis=1)


def test_knn_exact_against_numpy():
    X = datagen.blobs(11, 400, 3, 5).astype(np.float64)
    Q = datagen.blobs(12, 30, 3, 5).astype(np.float64)
    ids, d2, _ = oracle.knn_exact(X, Q, 7)
    ids2, d22 = _exact_numpy(X, Q, 7)
    np.testing.assert_array_equal(ids, ids2)
    np.testing.assert_allclose(d2, d22, rtol=1e-13)
    # ties by id: duplicated points
    Xd = np.array([[0.0], [1.0], [1.0], [1.0], [3.0]])
    ids, _, _ = oracle.knn_exact(Xd, np.array([[1.0]]), 3)
    assert list(ids[0]) == [1, 2, 3]


def test_query_single_level_k1_is_exact_knn():
    # SURVEY §8(c) pins: L=1, k_1=1 -> the leaf is all N points -> result = exact k-NN, recall 1
    X = datagen.blobs(13, 500, 2, 6).astype(np.float64)
    Q = datagen.blobs(14, 40, 2, 6).astype(np.float64)
    idx = oracle.build_index(X, [np.array([3])], T=2)
    ids, d2, _ = oracle.query(idx.P, idx.offsets, idx.members, X, Q, 10, 1)
    eids, ed2, _ = oracle.knn_exact(X, Q, 10)
    np.testing.assert_array_equal(ids, eids)
    assert oracle.recall(ids, eids) == 1.0


def test_query_wide_beam_is_exact_knn():
    # beam >= max_l k_l -> every partition scanned -> exact k-NN
    X = datagen.blobs(15, 800, 3, 8).astype(np.float64)
    Q = datagen.blobs(16, 25, 3, 8).astype(np.float64)
    inits = [datagen.init_indices(96, 1, 800, 40), datagen.init_indices(96, 2, 40, 6)]
    idx = oracle.build_index(X, inits, T=5)
    ids, _, _ = oracle.query(idx.P, idx.offsets, idx.members, X, Q, 5, beam=40)
    eids, _, _ = oracle.knn_exact(X, Q, 5)
    np.testing.assert_array_equal(ids, eids)


def test_query_identity_levels_self_query():
    # P:1864-1867 "1:1 ratio ... renders perfect accuracy (exact search)": identity levels
    X = datagen.random_dense(17, 64, 4).astype(np.float64)
    inits = [np.arange(64), np.arange(64)]
    idx = oracle.build_index(X, inits, T=3)
    ids, d2, _ = oracle.query(idx.P, idx.offsets, idx.members, X, X, 1, 1)
    np.testing.assert_array_equal(ids[:, 0], np.arange(64))
    assert np.all(d2 == 0.0)


def test_query_padding_and_descent_invariants():
    X = datagen.blobs(18, 300, 2, 5).astype(np.float64)
    Q = datagen.blobs(19, 20, 2, 5).astype(np.float64)
    inits = [datagen.init_indices(95, 1, 300, 60), datagen.init_indices(95, 2, 60, 7)]
    idx = oracle.build_index(X, inits, T=4)
    ids, d2, _ = oracle.query(idx.P, idx.offsets, idx.members, X, Q, 50, 1)
    eids, ed2, _ = oracle.knn_exact(X, Q, 1)
    for q in range(20):
        valid = ids[q] >= 0
        # padded with (-1, +inf) after the partition is exhausted (D8)
        assert np.all(np.isinf(d2[q][~valid]))
        assert np.all(np.diff(d2[q][valid]) >= 0)
        # one-sided approximation: top hit never closer than the true NN
        assert d2[q][0] >= ed2[q][0]
        # every hit lies in the single level-1 partition that was reached
        lab1 = idx.levels[0].labels
        assert len(set(lab1[ids[q][valid]].tolist())) == 1
        # the reached level-1 prototype is the nearest non-empty child of the nearest top prototype
        P2, P1 = idx.P[1], idx.P[0]
        off2, mem2 = idx.offsets[1], idx.members[1]
        off1 = idx.offsets[0]
        top = [j for j in range(P2.shape[0]) if off2[j + 1] > off2[j]]
        t = min(top, key=lambda j: (oracle.dist2(Q[q], P2[j]), j))
        ch = [int(j) for j in mem2[off2[t]:off2[t + 1]] if off1[j + 1] > off1[j]]
        c = min(ch, key=lambda j: (oracle.dist2(Q[q], P1[j]), j))
        assert lab1[ids[q][0]] == c


def test_query_sparse_matches_densified():
    rp, col, val = datagen.random_csr(20, 150, 60, 6)
    qrp, qcol, qval = datagen.random_csr(21, 12, 60, 6)
    dense = np.zeros((150, 60))
    for i in range(150):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    qd = np.zeros((12, 60))
    for i in range(12):
        qd[i, qcol[qrp[i]:qrp[i + 1]]] = qval[qrp[i]:qrp[i + 1]]
    inits = [datagen.init_indices(94, 1, 150, 15), datagen.init_indices(94, 2, 15, 3)]
    idx = oracle.build_index((rp, col, val), inits, T=4, csr_dim=60)
    a_ids, a_d2, _ = oracle.query(idx.P, idx.offsets, idx.members, (rp, col, val), (qrp, qcol, qval), 5, 1,
                                  dim=60, x_csr=True, q_csr=True)
    b_ids, b_d2, _ = oracle.query(idx.P, idx.offsets, idx.members, dense, qd, 5, 1)
    np.testing.assert_array_equal(a_ids, b_ids)
    np.testing.assert_allclose(a_d2, b_d2, rtol=1e-12, atol=1e-15)
    e1, _, _ = oracle.knn_exact((rp, col, val), (qrp, qcol, qval), 5, csr=True)
    e2, _, _ = oracle.knn_exact(dense, qd, 5)
    np.testing.assert_array_equal(e1, e2)


def test_recall_definition():
    assert oracle.recall(np.array([[1, 2, 3]]), np.array([[3, 2, 9]])) == pytest.approx(2 / 3)
    assert oracle.recall(np.array([[-1, -1]]), np.array([[0, 1]])) == 0.0


# ------------------------------------------------------------------ grouped construction (NEXT-1)
def _golden_grouped():
    with open(os.path.join(GOLDEN, "paper_grouped_depth.json")) as f:
        return json.load(f)


def test_grouped_depth_matches_paper_tables():
    # PAPER.md P:1457-1467 and P:1506-1516 (Tree depth column, 80,000 points)
    g = _golden_grouped()
    for row in g["depth_by_params"]:
        layers = oracle.grouped_layer_sizes(g["n_points"], row["length_group"], row["n_centroids"])
        assert len(layers) == row["tree_depth"], row


def test_grouped_first_layer_of_the_1600_point_example():
    # 1,600 points, lengthGroup 16, nCentroids 8 -> 100 groups, 800 centroids
    ex = _golden_grouped()["first_layer_example"]
    X = datagen.gaussian_clouds(1, ex["n_points"] // 8, 30.0)
    idx = oracle.build_grouped(X, ex["length_group"], ex["n_centroids"], 5, datagen.group_perm(2, X.shape[0]))
    assert oracle.grouped_layer_sizes(ex["n_points"], ex["length_group"], ex["n_centroids"])[0][1] == ex["groups"]
    assert idx.levels[0].P.shape[0] == ex["first_layer_centroids"]
    # top layer holds at most lengthGroup centroids ("less than or equal to")
    assert idx.levels[-1].P.shape[0] <= ex["length_group"]


def test_grouped_structure_and_per_group_clustering():
    # SPEC index invariants: each group's child lists partition the group's chunk; every item is
    # labelled with its nearest prototype of its own group (brute force, lowest ordinal on ties)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((203, 3))
    lg, nc = 20, 6
    perm = datagen.group_perm(4, X.shape[0])
    idx = oracle.build_grouped(X, lg, nc, 100, perm)
    Y, order = X, perm
    for lv, (n, g) in zip(idx.levels, oracle.grouped_layer_sizes(X.shape[0], lg, nc)):
        base, rem = divmod(n, g)
        start = 0
        for gi in range(g):
            size = base + (1 if gi >= g - rem else 0)
            items = np.sort(order[start:start + size])
            start += size
            assert set(np.unique(lv.labels[items]) // nc) == {gi}
            protos = lv.P[gi * nc:(gi + 1) * nc]
            d = cdist(Y[items], protos, "sqeuclidean")
            np.testing.assert_array_equal(lv.labels[items] - gi * nc, np.argmin(d, axis=1))
            for c in range(nc):  # converged: non-empty prototypes are their members' means
                mem = items[lv.labels[items] == gi * nc + c]
                if mem.size:
                    np.testing.assert_allclose(protos[c], Y[mem].mean(axis=0), rtol=1e-12, atol=1e-12)
        Y, order = lv.P, np.arange(lv.P.shape[0])


def test_grouped_single_centroid_groups_are_group_means():
    # nCentroids = 1: each group's prototype is the mean of its chunk (closed form); 43 points in
    # groups of 10 -> 4 groups of sizes 10, 11, 11, 11 (balanced split, remainder in the last groups)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((43, 2))
    perm = datagen.group_perm(6, 43)
    idx = oracle.build_grouped(X, 10, 1, 3, perm)
    assert len(idx.levels) == 1
    chunks = [perm[0:10], perm[10:21], perm[21:32], perm[32:43]]
    for gi, ch in enumerate(chunks):
        np.testing.assert_allclose(idx.levels[0].P[gi], X[ch].mean(axis=0), rtol=1e-13)
        assert np.all(idx.levels[0].labels[ch] == gi)
    with pytest.raises(ValueError):
        oracle.grouped_layer_sizes(100, 10, 10)


def test_grouped_no_overlap_clouds_point_search_error_zero():
    # X_GNO (8 well-separated clouds x 200 points, lengthGroup 16,
    # nCentroids 8): "able to correctly find all points without errors" -> 0.0 %.  Read as the
    # cloud-level error of the descent (G7): the point returned for every self-query
    # lies in the query's own cloud.
    X = datagen.gaussian_clouds(31, 200, 40.0, 1.0)
    idx = oracle.build_grouped(X, 16, 8, 20, datagen.group_perm(32, X.shape[0]))
    assert len(idx.levels) == 7  # P:1250-1251 "final depth of 8 layers" = 7 centroid layers + data
    ids, _, _ = oracle.query(idx.P, idx.offsets, idx.members, X, X, 1, 1)
    cloud = np.repeat(np.arange(8), 200)
    assert np.mean(cloud[ids[:, 0]] != cloud) == 0.0


# ------------------------------------------------------------------ range search (NEXT-2)
def _small_index(seed=3, n=600, d=3, levels=(40, 6)):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) * np.array([3.0, 1.0, 0.5])[:d]
    inits = [datagen.init_indices(seed, 1, n, levels[0]), datagen.init_indices(seed, 2, levels[0], levels[1])]
    return X, oracle.build_index(X, inits, 10)


def test_range_cover_mode_equals_brute_force():
    # SPEC range_query [DERIVED]: cover-expanded pruning is lossless by the triangle inequality,
    # so the result equals the brute-force range scan over the whole dataset
    X, idx = _small_index()
    cov = oracle.cover_radii(idx, X)
    rng = np.random.default_rng(4)
    for q in rng.standard_normal((25, 3)) * 2:
        for r in (0.3, 1.0, 2.5):
            ids, d2 = oracle.range_query(idx.P, idx.offsets, idx.members, X, q, r, cover=cov)
            bd = cdist(q[None], X, "sqeuclidean")[0]
            ref = np.nonzero(bd <= r * r)[0]
            ref = ref[np.lexsort((ref, bd[ref]))]
            np.testing.assert_array_equal(ids, ref)


def test_range_paper_mode_is_a_subset_and_zero_radius_finds_duplicates():
    X, idx = _small_index()
    cov = oracle.cover_radii(idx, X)
    rng = np.random.default_rng(5)
    for q in rng.standard_normal((20, 3)) * 2:
        a, _ = oracle.range_query(idx.P, idx.offsets, idx.members, X, q, 1.5)
        b, _ = oracle.range_query(idx.P, idx.offsets, idx.members, X, q, 1.5, cover=cov)
        assert set(a.tolist()) <= set(b.tolist())  # SPEC: candidate-set monotonicity
    # radius 0 at an indexed point, cover mode: exactly that point (distinct data)
    ids, d2 = oracle.range_query(idx.P, idx.offsets, idx.members, X, X[17], 0.0, cover=cov)
    np.testing.assert_array_equal(ids, [17])
    assert d2[0] == 0.0


def test_cover_radii_bound_every_descendant():
    X, idx = _small_index()
    cov = oracle.cover_radii(idx, X)
    # level 1: exact max member distance; level 2: >= the distance to every data row below
    lab1 = idx.levels[0].labels
    for j in range(idx.levels[0].P.shape[0]):
        mem = X[lab1 == j]
        exp = np.sqrt(((mem - idx.levels[0].P[j]) ** 2).sum(axis=1)).max() if len(mem) else 0.0
        assert cov[0][j] == pytest.approx(exp, rel=1e-12, abs=0)
    lab2 = idx.levels[1].labels
    for j in range(idx.levels[1].P.shape[0]):
        rows = np.nonzero(np.isin(lab1, np.nonzero(lab2 == j)[0]))[0]
        if rows.size:
            assert np.sqrt(((X[rows] - idx.levels[1].P[j]) ** 2).sum(axis=1)).max() <= cov[1][j] * (1 + 1e-12)


# ------------------------------------------------------------------ insertion (NEXT-4)
def test_insertion_closure_and_descent_matches_query_path():
    # P:963-982 + SPEC insert [TRIVIAL]: insert then point query of the same vector -> found, and
    # the insertion path is the beam-1 query path (its partition holds the k-NN answer)
    X, idx = _small_index(seed=6)
    rng = np.random.default_rng(7)
    new = rng.standard_normal((30, 3)) * 2
    labels = [lv.labels.copy() for lv in idx.levels]
    leafs = [oracle.descend_leaf(idx.P, idx.offsets, idx.members, q)[0] for q in new]
    X2 = np.concatenate([X, new])
    lab1 = np.concatenate([labels[0], np.array(leafs, np.int32)])
    off1, mem1 = oracle.children(lab1, idx.levels[0].P.shape[0])
    offs = [off1] + idx.offsets[1:]
    mems = [mem1] + idx.members[1:]
    ids, d2, _ = oracle.query(idx.P, offs, mems, X2, new, 1, 1)
    np.testing.assert_array_equal(ids[:, 0], np.arange(X.shape[0], X2.shape[0]))
    assert np.all(d2[:, 0] == 0.0)
    # the leaf reached is the partition a beam-1 k-NN query of a pre-existing row scans
    for i in rng.choice(X.shape[0], 20, replace=False):
        j, _ = oracle.descend_leaf(idx.P, idx.offsets, idx.members, X[i])
        rows = idx.members[0][idx.offsets[0][j]:idx.offsets[0][j + 1]]
        got, _, _ = oracle.query(idx.P, idx.offsets, idx.members, X, X[i:i + 1], 1, 1)
        assert got[0, 0] in rows


# ------------------------------------------------------------------ distributed mode (NEXT-3)
def _node_indexes(X, W, levels=(12, 3), seed=41, T=6):
    """W independent indexes over contiguous row ranges of X (global id = range start + local)."""
    n = X.shape[0]
    nodes = []
    for r in range(W):
        lo, hi = r * n // W, (r + 1) * n // W
        Xl = X[lo:hi]
        inits = [datagen.init_indices(seed + r, 1, hi - lo, levels[0]),
                 datagen.init_indices(seed + r, 2, levels[0], levels[1])]
        idx = oracle.build_index(Xl, inits, T)
        nodes.append(dict(P=idx.P, offsets=idx.offsets, members=idx.members, X=Xl, id_base=lo))
    return nodes


def test_route_matches_library_distances_and_limits():
    # §3.4: routed(q) = {n : min_c ||q - c|| < eps}; checked against scipy's cdist,
    # eps = inf -> every node, eps = 0 -> no node (strict, reading C1), monotone in eps
    rng = np.random.default_rng(7)
    tops = [rng.standard_normal((m, 3)) * 4 for m in (5, 1, 9)]
    tops.append(np.zeros((0, 3)))  # a node that registered nothing
    Q = rng.standard_normal((60, 3)) * 4
    R = np.concatenate(tops[:3])
    owner = np.repeat(np.arange(3), [5, 1, 9])
    D = cdist(Q, R)
    for eps in (0.5, 2.0, 3.7, 8.0):
        for i, q in enumerate(Q):
            got, _ = oracle.route(tops, q, eps)
            assert got == sorted(set(owner[D[i] < eps].tolist()))
    for q in Q[:10]:
        assert oracle.route(tops, q, np.inf)[0] == [0, 1, 2, 3]
        assert oracle.route(tops, q, 0.0)[0] == []
        prev = set()
        for eps in np.linspace(0, 12, 25):
            cur = set(oracle.route(tops, q, eps)[0])
            assert prev <= cur
            prev = cur
    # strict: a query exactly on a centroid is not routed at eps = 0 but is at any eps > 0
    assert oracle.route(tops, tops[1][0], 0.0)[0] == []
    assert 1 in oracle.route(tops, tops[1][0], 1e-9)[0]


def test_route_node_exclusive_region():
    # SPEC route [DERIVED]: node n holds cloud n only (clouds 40 apart, sigma 1); a query near
    # cloud n's centre with eps = half the centre spacing reaches exactly node n
    X = datagen.gaussian_clouds(5, 150, radius=40.0, sigma=1.0, clouds=4).astype(np.float64)
    nodes = _node_indexes(X, 4, levels=(10, 2))
    tops = [oracle.top_registry(nd["P"][-1], nd["offsets"][-1]) for nd in nodes]
    centres = 40.0 * np.stack([np.cos(np.arange(4) * np.pi / 2), np.sin(np.arange(4) * np.pi / 2)], 1)
    spacing = 40.0 * np.sqrt(2.0)
    rng = np.random.default_rng(3)
    for n in range(4):
        for _ in range(5):
            q = centres[n] + rng.standard_normal(2) * 0.5
            assert oracle.route(tops, q, spacing / 2)[0] == [n]


def test_cluster_broadcast_with_wide_beam_is_exact_knn():
    # eps = inf and beam >= every k_l: each node's descent scans all its rows, so the merged
    # answer is the exact k-NN of the union with global ids (brute force, ties by (d^2, id))
    X = datagen.blobs(21, 600, 3, 6).astype(np.float64)
    Q = datagen.blobs(22, 30, 3, 6).astype(np.float64)
    nodes = _node_indexes(X, 3)
    ids, d2, routed, _ = oracle.cluster_query(nodes, Q, 7, beam=12, epsilon=np.inf)
    assert routed.all()
    eids, ed2, _ = oracle.knn_exact(X, Q, 7)
    np.testing.assert_array_equal(ids, eids)
    np.testing.assert_allclose(d2, ed2, rtol=1e-13)


def test_cluster_single_node_and_tight_epsilon():
    X = datagen.blobs(23, 500, 2, 5).astype(np.float64)
    Q = datagen.blobs(24, 40, 2, 5).astype(np.float64)
    # one node: the cluster answer is that node's own descent (no merge)
    one = _node_indexes(X, 1)
    ids, d2, _, _ = oracle.cluster_query(one, Q, 5, 1, np.inf)
    ids0, d20, _ = oracle.query(one[0]["P"], one[0]["offsets"], one[0]["members"], X, Q, 5, 1)
    np.testing.assert_array_equal(ids, ids0)
    # a tight eps routes fewer nodes: results are drawn only from the routed nodes, queries
    # with no routed node get the padding, and recall cannot exceed the broadcast's
    nodes = _node_indexes(X, 4)
    ids_all, _, _, _ = oracle.cluster_query(nodes, Q, 5, 1, np.inf)
    ids_t, d2_t, routed, _ = oracle.cluster_query(nodes, Q, 5, 1, 0.6)
    assert routed.sum() < routed.size
    lo = np.array([nd["id_base"] for nd in nodes] + [X.shape[0]])
    for i in range(len(Q)):
        own = np.searchsorted(lo, ids_t[i][ids_t[i] >= 0], side="right") - 1
        assert set(own.tolist()) <= set(np.nonzero(routed[i])[0].tolist())
        if not routed[i].any():
            assert (ids_t[i] == -1).all() and np.isinf(d2_t[i]).all()
    eids, _, _ = oracle.knn_exact(X, Q, 5)
    assert oracle.recall(ids_t, eids) <= oracle.recall(ids_all, eids)


# ------------------------------------------------------------------ seeded initialisation (D2)
def test_seeded_init_is_a_uniform_sample_without_replacement():
    # k distinct indices in range; k = n gives every index; the first SplitMix64 outputs of the
    # published reference seed 0 (state increments from 0) pin the generator itself
    for (n, k) in ((10, 10), (1000, 5), (57, 56), (1, 1)):
        v = oracle.seeded_init(3, 1, n, k)
        assert len(v) == k and len(set(v.tolist())) == k and v.min() >= 0 and v.max() < n
    assert sorted(oracle.seeded_init(9, 2, 40, 40).tolist()) == list(range(40))
    # SplitMix64 from state 0: 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4 (Steele et al.'s sequence)
    import oracle as o
    state, outs = 0, []
    for _ in range(2):
        state = (state + 0x9E3779B97F4A7C15) & o._M64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & o._M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & o._M64
        outs.append(z ^ (z >> 31))
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]
    # level 1 with seed = -level * golden starts from state 0: its first draw is u(n-k+1) of
    # the first output above
    n, k = 1000, 3
    seed = (-1 * 0x9E3779B97F4A7C15) & o._M64
    assert oracle.seeded_init(seed, 1, n, k)[0] == 0xE220A8397B1DCDAF % (n - k + 1)
    # uniformity: each index of [0, 20) is chosen with probability k/n = 1/4 over many seeds
    cnt = np.zeros(20)
    for s in range(4000):
        cnt[oracle.seeded_init(s, 1, 20, 5)] += 1
    p = 5 / 20
    sd = np.sqrt(4000 * p * (1 - p))
    assert np.all(np.abs(cnt - 4000 * p) < 5 * sd), cnt


# ------------------------------------------------------------------ relocation and rebuild (NEXT-4)
def test_relocation_loop_definitions():
    X = datagen.gaussian_clouds(5, 100, radius=12.0, sigma=2.0)
    perm = datagen.group_perm(5, X.shape[0])
    # iterations = 0: the single entry is the first build's exhaustive error (SPEC)
    e0 = oracle.relocate_and_rebuild(X, 16, 8, 8, perm, 0, 3, datagen.relocation_keys)
    idx = oracle.build_grouped(X, 16, 8, 8, perm=perm)
    assert e0 == [oracle.exhaustive_error(idx, X)]
    # a relocation step: found points keep their group, missed points land in the reached
    # group, the order is by (target group, key), and every point appears once
    n, g = 103, 6
    order = np.random.default_rng(1).permutation(n)
    found = np.random.default_rng(2).random(n) < 0.5
    reached = np.random.default_rng(3).integers(0, g, n)
    keys = np.random.default_rng(4).permutation(n)
    new = oracle.relocation_order(order, g, found, reached, keys)
    assert sorted(new.tolist()) == list(range(n))
    base, rem = divmod(n, g)
    cur = np.empty(n, int)
    pos = 0
    for gi in range(g):
        size = base + (1 if gi >= g - rem else 0)
        cur[order[pos:pos + size]] = gi
        pos += size
    target = np.where(found, cur, reached)
    assert np.all(np.diff(target[new]) >= 0)
    for gi in range(g):
        members = new[target[new] == gi]
        assert np.all(np.diff(keys[members]) > 0)


def test_relocation_lowers_the_self_miss_rate():
    # §5.1 / Table 1: relocating the points not found makes the groups follow the search paths,
    # so some rebuild reaches a lower error than the first build (the paper: 40.5 -> 30.31 %)
    X = datagen.gaussian_clouds(5, 200, radius=12.0, sigma=2.0)
    perm = datagen.group_perm(5, X.shape[0])
    e = oracle.relocate_and_rebuild(X, 16, 8, 10, perm, 4, 100, datagen.relocation_keys)
    assert len(e) == 5 and min(e[1:]) < e[0]


# ------------------------------------------------------------------ NEXT-4 partition split (reading S1)
def test_split_partitions_worked_example():
    """Hand-derived: a partition {0, 1, 2, 100, 101, 102} on a line with threshold 3 splits into
    s = 2 groups; whatever the two seeded init rows are, Lloyd separates the two clusters (an
    init inside one cluster pulls the far cluster to the other prototype at the first update:
    e.g. init (0, 1): {0} | {1, 2, 100, 101, 102} -> prototypes (0, 61.2) -> {0,1,2} | {100,101,102}),
    so the prototypes are 1 and 101; the other partition {50} and the level-2 labels stay."""
    X = np.array([[0.0], [1.0], [2.0], [100.0], [101.0], [102.0], [50.0]])
    P = [np.array([[51.0], [50.0]]), np.array([[40.0]])]
    labels = [np.array([0, 0, 0, 0, 0, 0, 1]), np.array([0, 0])]
    for seed in range(5):
        P2, L2, split = oracle.split_partitions(P, labels, X, threshold=3, T=5, seed=seed)
        assert split == [0]
        assert P2[0].shape == (3, 1) and P2[0][1, 0] == 50.0
        assert sorted([P2[0][0, 0], P2[0][2, 0]]) == [1.0, 101.0]
        a, b = L2[0][:3], L2[0][3:6]
        assert len(set(a)) == 1 and len(set(b)) == 1 and {a[0], b[0]} == {0, 2}
        assert P2[0][a[0], 0] == 1.0 and P2[0][b[0], 0] == 101.0
        assert L2[0][6] == 1
        np.testing.assert_array_equal(L2[1], [0, 0, 0])  # the new prototype's parent = j's parent
        np.testing.assert_array_equal(P2[1], P[1])


def test_split_partitions_invariants():
    """Random data: the split partitions' rows are exactly covered by the new groups, every new
    prototype is the mean of its members (numpy), every member sits at its nearest new prototype
    (scipy cdist), other partitions and upper levels are untouched, and s = ceil(n_j / threshold)."""
    from scipy.spatial.distance import cdist

    X = datagen.blobs(77, 3000, 5, 12)
    k1 = 12
    labels0 = oracle.assign(X, X[datagen.init_indices(78, 1, 3000, k1)])[0].astype(np.int64)
    P1 = np.stack([X[labels0 == j].mean(axis=0) for j in range(k1)])
    labels1 = np.arange(k1) % 3
    P2l = np.stack([P1[labels1 == j].mean(axis=0) for j in range(3)])
    thr = 300
    counts = np.bincount(labels0, minlength=k1)
    P2, L2, split = oracle.split_partitions([P1, P2l], [labels0, labels1], X, threshold=thr, T=8, seed=9)
    assert split == [j for j in range(k1) if counts[j] > thr] and split
    n_new = sum(-(-int(counts[j]) // thr) - 1 for j in split)
    assert P2[0].shape[0] == k1 + n_new and L2[1].shape[0] == k1 + n_new
    np.testing.assert_array_equal(P2[1], P2l)
    nxt = k1
    for j in range(k1):
        rows = np.nonzero(labels0 == j)[0]
        if j not in split:
            np.testing.assert_array_equal(P2[0][j], P1[j])
            np.testing.assert_array_equal(L2[0][rows], j)
            continue
        s = -(-int(counts[j]) // thr)
        ids = [j] + list(range(nxt, nxt + s - 1))
        nxt += s - 1
        assert set(L2[0][rows].tolist()) <= set(ids)
        for g in ids:
            mem = rows[L2[0][rows] == g]
            if mem.size:
                np.testing.assert_allclose(P2[0][g], X[mem].astype(np.float64).mean(axis=0), rtol=1e-12, atol=1e-12)
            assert L2[1][g] == labels1[j]
        D = cdist(X[rows].astype(np.float64), P2[0][ids], "sqeuclidean")
        near = np.array(ids)[D.argmin(axis=1)]
        np.testing.assert_array_equal(L2[0][rows], near)
    # nothing above the threshold: nothing changes
    P3, L3, sp3 = oracle.split_partitions([P1, P2l], [labels0, labels1], X, threshold=int(counts.max()), T=8, seed=9)
    assert sp3 == [] and np.array_equal(P3[0], P1) and np.array_equal(L3[0], labels0)


# ------------------------------------------------------------------ hand-derived pins (round 2)
def _hand_index(P_levels, labels_levels):
    """An oracle.Index from explicit prototypes and labels (child lists = {i : labels = j})."""
    levels, offs, mems = [], [], []
    for P, lab in zip(P_levels, labels_levels):
        P = np.asarray(P, np.float64)
        lab = np.asarray(lab, np.int32)
        levels.append(oracle.LevelResult(P, lab, np.zeros(1), np.zeros(1, np.int64), 0))
        o, m = oracle.children(lab, P.shape[0])
        offs.append(o)
        mems.append(m)
    return oracle.Index(levels, offs, mems, P_levels[0].shape[1] if np.ndim(P_levels[0]) == 2 else 1)


def test_range_paper_mode_hand_derived():
    """Algorithm 3 on a hand-built 1-D index: rows 0, 1, 10, 11, 20, 21; level-1
    prototypes 0.5 {0,1}, 10.5 {10,11}, 20.5 {20,21}; top prototypes 5.5 {c0, c1}, 20.5 {c2}.
    q = 9, r = 4: top keeps 5.5 (3.5 <= 4), drops 20.5; level 1 keeps 10.5 (1.5), drops 0.5 (8.5)
    -> rows 10, 11 (d^2 1, 4).  q = 5.8, r = 4.3: top keeps 5.5; level 1 drops 0.5 (5.3) and
    10.5 (4.7) -> nothing, although row 10 lies at 4.2 (the paper's rule is lossy); cover mode
    (cover(10.5) = 0.5: 4.7 <= 4.8) finds it."""
    X = np.array([[0.0], [1.0], [10.0], [11.0], [20.0], [21.0]])
    idx = _hand_index([np.array([[0.5], [10.5], [20.5]]), np.array([[5.5], [20.5]])],
                      [np.array([0, 0, 1, 1, 2, 2]), np.array([0, 0, 1])])
    ids, d2 = oracle.range_query(idx.P, idx.offsets, idx.members, X, np.array([9.0]), 4.0)
    np.testing.assert_array_equal(ids, [2, 3])
    np.testing.assert_array_equal(d2, [1.0, 4.0])
    ids, _ = oracle.range_query(idx.P, idx.offsets, idx.members, X, np.array([5.8]), 4.3)
    assert ids.size == 0
    cov = oracle.cover_radii(idx, X)
    np.testing.assert_allclose(cov[0], [0.5, 0.5, 0.5])
    np.testing.assert_allclose(cov[1], [5.5, 0.5])  # 5.5 -> farthest row below it: 0 or 11
    ids, d2 = oracle.range_query(idx.P, idx.offsets, idx.members, X, np.array([5.8]), 4.3, cover=cov)
    np.testing.assert_array_equal(ids, [2])
    np.testing.assert_allclose(d2, [4.2 ** 2])


def test_exhaustive_error_hand_derived_and_identity():
    """The point-search error (SPEC exhaustive_error): on a hand-built 1-D index with
    rows 0, 3, 4 and level-1 prototypes 0 {row 0} and 10 {rows 3, 4}, points 3 and 4 descend to
    prototype 0 (3 < 7, 4 < 6) and are answered with row 0: error 2/3.  An identity index (every
    point its own prototype) is exact search: error 0."""
    X = np.array([[0.0], [3.0], [4.0]])
    idx = _hand_index([np.array([[0.0], [10.0]])], [np.array([0, 1, 1])])
    assert oracle.exhaustive_error(idx, X) == pytest.approx(2.0 / 3.0)
    Xr = datagen.blobs(21, 300, 4, 5)
    ident = oracle.build_index(Xr, [np.arange(300), np.arange(300)], 3)
    assert oracle.exhaustive_error(ident, Xr) == 0.0


# ---------------------------------------------------------------- empty-cluster repair (D5b)
def test_lloyd_farthest_reseed_worked_example():
    """SPEC S:128 reading D5b, derived by hand.  Y = (0,0), (0,0), (1,0), (10,0), init rows
    {0, 1}: both prototypes (0,0), every row ties -> prototype 0 (D4), prototype 1 is empty.
    Pass 0: J0 = 0 + 0 + 1 + 100 = 101; P0 <- mean of all = (2.75, 0); the farthest row from its
    prototype is row 3 (d = 100) -> P1 <- (10, 0).  Pass 1: rows 0-2 -> 0 (7.5625, 7.5625,
    3.0625), row 3 -> 1 (0): J1 = 18.1875; P0 <- (1/3, 0).  Pass 2: no label change -> stop.
    Final J = 2/9 + 4/9 = 2/3.  Under "keep" prototype 1 stays at (0,0) and wins rows 0-2 in
    pass 1 instead."""
    Y = np.array([[0, 0], [0, 0], [1, 0], [10, 0]], np.float64)
    r = oracle.lloyd(Y, np.array([0, 1]), 10, empty="farthest")
    np.testing.assert_allclose(r.P, [[1 / 3, 0], [10, 0]], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(r.labels, [0, 0, 0, 1])
    np.testing.assert_allclose(r.J, [101.0, 18.1875, 2 / 3, 2 / 3], rtol=1e-15)
    assert r.updates == 2
    keep = oracle.lloyd(Y, np.array([0, 1]), 10)
    assert not np.allclose(keep.P, r.P)
    # keep: pass 1 puts rows 0-2 on the unmoved prototype 1 at (0,0) (0, 0, 1 against 7.5625,
    # 7.5625, 3.0625) and row 3 on prototype 0
    np.testing.assert_array_equal(oracle.lloyd(Y, np.array([0, 1]), 1).labels, [1, 1, 1, 0])


def test_lloyd_farthest_reseed_order_and_ties():
    """Several empty prototypes take the farthest rows in ascending j; equal distances go to
    the lower row index.  Y = (0,0) x3, (1,0), (7,0), (-9,0), init rows {0, 1, 2}: all rows ->
    prototype 0, prototypes 1 and 2 empty; farthest (d desc): row 5 (81), row 4 (49) ->
    P1 = (-9,0), P2 = (7,0).  Ties: Y = (0,0), (0,0), (-5,0), (5,0), init {0, 1}: rows 2 and 3
    are both at 25 -> row 2 (lower index) -> P1 = (-5,0); pass 1 moves row 3 nowhere (25/9 vs
    100) and P0 <- (5/3, 0)."""
    Y = np.array([[0, 0], [0, 0], [0, 0], [1, 0], [7, 0], [-9, 0]], np.float64)
    r = oracle.lloyd(Y, np.array([0, 1, 2]), 1, empty="farthest", trace=True)
    P1 = r.passes[1][0]  # the prototypes the final pass used = after the one update
    # P0 = mean of all six rows = (-1/6, 0); the two empties take rows 5 and 4
    np.testing.assert_allclose(P1, [[-1 / 6, 0], [-9, 0], [7, 0]], rtol=0, atol=1e-15)
    Y2 = np.array([[0, 0], [0, 0], [-5, 0], [5, 0]], np.float64)
    r2 = oracle.lloyd(Y2, np.array([0, 1]), 10, empty="farthest")
    np.testing.assert_allclose(r2.P, [[5 / 3, 0], [-5, 0]], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(r2.labels, [0, 0, 1, 0])


def test_lloyd_farthest_csr_equals_dense_and_no_empty_is_keep():
    """The CSR path re-seeds with the densified row; without empty clusters the policy does
    not change the trajectory."""
    rng = np.random.default_rng(5)
    D = np.where(rng.random((300, 40)) < 0.2, rng.random((300, 40)), 0.0)
    D[:40] = D[0]  # 40 identical rows: an init on them leaves empty clusters
    init = np.arange(12)
    rp = np.concatenate([[0], np.cumsum((D != 0).sum(1))]).astype(np.int64)
    col = np.nonzero(D)[1].astype(np.int32)
    val = D[D != 0].astype(np.float32).astype(np.float64)
    D = np.zeros_like(D)
    for i in range(D.shape[0]):
        D[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    a = oracle.lloyd(D, init, 8, empty="farthest")
    b = oracle.lloyd((rp, col, val), init, 8, csr_dim=40, empty="farthest")
    np.testing.assert_allclose(a.P, b.P, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(a.labels, b.labels)
    assert not np.allclose(a.P, oracle.lloyd(D, init, 8).P)  # the repair did change the run
    Y = rng.standard_normal((500, 3))
    init2 = rng.choice(500, 8, replace=False)
    np.testing.assert_array_equal(oracle.lloyd(Y, init2, 6, empty="farthest").P, oracle.lloyd(Y, init2, 6).P)
