"""GPU parity: the CUDA path (through the C-ABI) against the FP64 oracle on the same seeded
inputs, element by element, at sizes the oracle finishes in seconds (several tiles and a
ragged tail), plus edge cases.  Marked `gpu` (run on a B200)."""
import numpy as np
import pytest

import datagen
import oracle
from parity import check_assignment, check_prototypes, check_queries, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_native_library_is_the_one_loaded():
    import paper_2208_02734_b200._lib as L

    lib = L.load()
    assert mk.device_ok(), "libmask reports no sm_100 device"
    import os

    maps = open("/proc/self/maps").read()
    assert os.path.realpath(L.LIB_PATH) in maps


# ------------------------------------------------------------------ assignment (K1/K2)
ASSIGN_SHAPES = [
    (1000, 2, 100), (1037, 3, 7), (4099, 16, 300), (500, 17, 33), (257, 64, 1), (300, 128, 300),
    (2049, 8, 129), (777, 1, 5), (3000, 32, 64), (1500, 64, 513), (640, 96, 40), (300, 128, 257),
    # one prototype tile, many row blocks (one TMEM A buffer for d > 64): every issuer keeps
    # the per-block A phases in step
    (5000, 128, 100), (3000, 96, 128), (4100, 64, 128), (2000, 40, 192),
]


@pytest.mark.parametrize("n,d,k", ASSIGN_SHAPES)
@pytest.mark.parametrize("flags", [0, mk.MASK_FORCE_SIMT])
def test_assign_parity(n, d, k, flags):
    X = datagen.blobs(100 + d, n, d, max(2, k // 4), spread=10.0)
    P = X[datagen.init_indices(50 + d, 1, n, k)]
    P = P + datagen.random_dense(7 + k, k, d, scale=0.1)  # prototypes that are not data rows
    lab, d2, nf = mk.assign(t(X), t(P), flags=flags)
    check_assignment(X, P, lab.cpu().numpy(), d2.cpu().numpy(), what=f"assign n={n} d={d} k={k}")


def test_assign_exact_ties_take_lowest_ordinal():
    X = np.array([[0.0, 0.0], [1.0, 1.0], [2.0, 2.0]] * 50, np.float32)
    P = np.array([[5.0, 5.0], [1.0, 1.0], [1.0, 1.0], [0.0, 0.0], [0.0, 0.0]], np.float32)
    for flags in (0, mk.MASK_FORCE_SIMT):
        lab, d2, _ = mk.assign(t(X), t(P), flags=flags)
        lab = lab.cpu().numpy()
        assert np.all(lab[0::3] == 3) and np.all(lab[1::3] == 1) and np.all(lab[2::3] == 1)


# ------------------------------------------------------------------ update (K5/K7)
@pytest.mark.parametrize("n,d,k", [(5000, 2, 100), (4099, 16, 300), (1000, 17, 50), (3000, 64, 129), (700, 128, 33)])
def test_update_parity(n, d, k):
    X = datagen.blobs(200 + d, n, d, 7)
    P_in = datagen.random_dense(300 + d, k, d)
    rng = np.random.default_rng(n)
    labels = rng.integers(0, max(1, k - 5), size=n).astype(np.int32)  # last clusters empty
    P_out, counts, md = mk.update(t(X), t(labels), t(P_in))
    P_ref, cnt_ref = oracle.means(X.astype(np.float64), labels, P_in.astype(np.float64))
    assert np.array_equal(counts.cpu().numpy(), cnt_ref)
    got = P_out.cpu().numpy()
    check_prototypes(got, P_ref, what="update")
    empty = cnt_ref == 0
    assert np.array_equal(got[empty], P_in[empty])  # D5: empty keeps its prototype exactly
    ref_md = np.sqrt(((P_ref - P_in) ** 2).sum(axis=1)).max()
    assert md == pytest.approx(ref_md, rel=1e-4)


# ------------------------------------------------------------------ build (levels + Lloyd)
def _step_parity_build(X, levels, T, inits, flags=0, csr=None, tol=0.0):
    """Build with the step-parity hook; check every pass's assignment and every update
    against the oracle applied to the GPU's own P_t (SURVEY §8(c) step mode)."""
    passes = {}

    def cb(level, p, P, labels):
        passes.setdefault(level, []).append((P, labels))

    data = X if csr is None else csr
    idx = mk.build(data, levels, T, inits, tol=tol, flags=flags, iter_cb=cb)
    Y = None
    for l in range(1, len(levels) + 1):
        if l == 1:
            if csr is None:
                Y = X.astype(np.float64)
            else:
                rp, col, val = [a.cpu().numpy() if hasattr(a, "cpu") else a for a in (csr.row_ptr, csr.col, csr.val)]
                Y = np.zeros((rp.size - 1, csr.dim))
                for i in range(rp.size - 1):
                    Y[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
        else:
            Y = idx.prototypes(l - 1).astype(np.float64)
        seq = passes[l]
        # init prototypes = the seeded rows
        np.testing.assert_array_equal(seq[0][0], Y[inits[l - 1]].astype(np.float32))
        for p_i, (P, lab) in enumerate(seq):
            check_assignment(Y, P, lab, what=f"level {l} pass {p_i}")
            if p_i + 1 < len(seq):
                P_next = seq[p_i + 1][0]
                if not np.array_equal(P_next, P):  # an update happened between the passes
                    P_ref, _ = oracle.means(Y, lab, P.astype(np.float64))
                    check_prototypes(P_next, P_ref, what=f"level {l} update after pass {p_i}")
        # stored labels = the final pass
        np.testing.assert_array_equal(idx.labels(l), seq[-1][1])
        np.testing.assert_array_equal(idx.prototypes(l), seq[-1][0])
        # children = {i : labels[i] = j} ascending
        off, mem = idx.children(l)
        o_ref, m_ref = oracle.children(seq[-1][1], levels[l - 1])
        np.testing.assert_array_equal(off, o_ref)
        np.testing.assert_array_equal(mem, m_ref)
        tr = idx.trace(l)
        assert len(tr["J"]) == len(seq)
    return idx, passes


def _e2e_compare(idx, X, levels, T, inits, csr_dim=None, data=None):
    ref = oracle.build_index(X if data is None else data, inits, T, csr_dim=csr_dim)
    errs = []
    for l in range(1, len(levels) + 1):
        errs.append(check_prototypes(idx.prototypes(l), ref.levels[l - 1].P, what=f"e2e level {l}"))
    return ref, errs


def test_build_C1_full_step_and_e2e():
    cfg = datagen.CONFIGS[1]
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    idx, passes = _step_parity_build(X, cfg.levels, cfg.iters, inits)
    ref, errs = _e2e_compare(idx, X, cfg.levels, cfg.iters, inits)
    # trace: J_t of the GPU vs the oracle's when the trajectories agree
    trg = idx.trace(1)
    if len(trg["J"]) == len(ref.levels[0].J):
        np.testing.assert_allclose(trg["J"], ref.levels[0].J, rtol=1e-4)
    # queries: oracle descends the GPU-built index
    Q = datagen.queries(cfg)
    _query_parity(idx, X, Q, cfg.levels, knn=cfg.knn, beam=1)
    idx.free()


def _query_parity(idx, X, Q, levels, knn, beam, Qdev=None, csr=False, dim=None):
    L = len(levels)
    P = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
    ch = [idx.children(l) for l in range(1, L + 1)]
    ids_ref, d2_ref, gap = oracle.query(P, [c[0] for c in ch], [c[1] for c in ch], X, Q, knn, beam,
                                        dim=dim, x_csr=csr, q_csr=csr)
    qin = Qdev if Qdev is not None else t(Q)
    ids, d2 = idx.query(qin, knn=knn, beam=beam)
    ids = ids.cpu().numpy()
    d2 = d2.cpu().numpy()
    nd, ne = check_queries(ids, d2, ids_ref, d2_ref, gap, what=f"query beam={beam}")
    # host-memory query path gives the same answer
    if not csr:
        ids_h, d2_h = idx.query(np.ascontiguousarray(Q, np.float32), knn=knn, beam=beam)
        np.testing.assert_array_equal(ids_h, ids)
    if not csr:
        eids, _, _ = oracle.knn_exact(X, Q, knn)
        ok = gap >= 1e-5
        r_gpu = oracle.recall(ids[ok], eids[ok])
        r_ref = oracle.recall(ids_ref[ok], eids[ok])
        assert r_gpu == r_ref
    return nd, ne


@pytest.mark.parametrize("cid,div,T", [(1, 1, 20), (2, 64, 25), (3, 2048, 20)])
def test_build_fused_small_levels_step(cid, div, T):
    """Levels small enough for the fused single-launch Lloyd loop (K11) in step mode over the
    pass trace of the production build (MASK_TRACE_PASSES; no iteration callback, so K11 runs):
    every pass's labels = nearest prototype of the P_t it used (tie window), every update =
    FP64 member means of those labels (1e-4), J of the final pass, child lists."""
    cfg = datagen.CONFIGS[cid].scaled(div) if div > 1 else datagen.CONFIGS[cid]
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    idx = mk.build(t(X), cfg.levels, T, inits, flags=mk.MASK_TIME_KERNELS | mk.MASK_TRACE_PASSES)
    Y = X.astype(np.float64)
    for l in range(1, len(cfg.levels) + 1):
        assert idx.timing(l)["assign_kernel"] == "K11-fused-small-level", f"level {l}: expected K11"
        seq = idx.passes(l)
        np.testing.assert_array_equal(seq[0][0], Y[inits[l - 1]].astype(np.float32))
        for p_i, (P, lab) in enumerate(seq):
            check_assignment(Y, P, lab, what=f"level {l} pass {p_i}")
            if p_i + 1 < len(seq) and not np.array_equal(seq[p_i + 1][0], P):
                P_ref, _ = oracle.means(Y, lab, P.astype(np.float64))
                check_prototypes(seq[p_i + 1][0], P_ref, what=f"level {l} update after pass {p_i}")
        P, lab = seq[-1]
        np.testing.assert_array_equal(idx.labels(l), lab)
        np.testing.assert_array_equal(idx.prototypes(l), P)
        off, mem = idx.children(l)
        o_ref, m_ref = oracle.children(lab, cfg.levels[l - 1])
        np.testing.assert_array_equal(off, o_ref)
        np.testing.assert_array_equal(mem, m_ref)
        tr = idx.trace(l)
        assert len(tr["J"]) == len(seq)
        d2 = ((Y - P.astype(np.float64)[lab]) ** 2).sum()
        assert tr["J"][-1] == pytest.approx(d2, rel=1e-5)
        Y = P.astype(np.float64)
    idx.free()


@pytest.mark.parametrize("cid,div", [(2, 64), (3, 256), (5, 2048)])
def test_build_scaled_replicas_step_and_queries(cid, div):
    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    T = min(cfg.iters, 8)
    idx, _ = _step_parity_build(X, cfg.levels, T, inits)
    Q = datagen.queries(cfg, count=200)
    _query_parity(idx, X, Q, cfg.levels, knn=10, beam=1)
    _query_parity(idx, X, Q, cfg.levels, knn=5, beam=3)
    idx.free()


def test_build_edge_cases():
    X = datagen.blobs(300, 1001, 5, 9)
    # k = n at level 1 with identity init: every point its own prototype, J = 0
    idx = mk.build(t(X), [1001, 1], 3, [np.arange(1001), np.array([7])])
    np.testing.assert_array_equal(idx.prototypes(1), X)
    np.testing.assert_array_equal(idx.labels(1), np.arange(1001))
    assert idx.trace(1)["J"][-1] == 0.0
    # level 2 with k = 1: the mean of the level-1 prototypes
    np.testing.assert_allclose(idx.prototypes(2)[0], X.astype(np.float64).mean(axis=0), rtol=1e-5, atol=1e-5)
    # self-queries on the identity index return the point itself
    ids, d2 = idx.query(t(X[:50]), knn=1)
    np.testing.assert_array_equal(ids.cpu().numpy()[:, 0], np.arange(50))
    idx.free()
    # L = 1, k = 1: the leaf is the whole dataset -> exact k-NN, recall 1
    idx = mk.build(t(X), [1], 2, [np.array([3])])
    Q = datagen.blobs(301, 64, 5, 9)
    ids, d2 = idx.query(t(Q), knn=10)
    eids, ed2, gap = oracle.knn_exact(X, Q, 10)
    ok = gap >= 1e-5
    np.testing.assert_array_equal(ids.cpu().numpy()[ok], eids[ok])
    idx.free()
    # T = 0: labels are the plain assignment to the init rows
    inits = [datagen.init_indices(5, 1, 1001, 40)]
    idx = mk.build(t(X), [40], 0, inits)
    check_assignment(X, X[inits[0]], idx.labels(1))
    assert idx.level_info(1)["updates"] == 0
    idx.free()
    # a partition smaller than k_nn is padded with (-1, +inf)
    idx = mk.build(t(X), [500], 3, [datagen.init_indices(6, 1, 1001, 500)])
    ids, d2 = idx.query(t(X[:20]), knn=32)
    ids = ids.cpu().numpy()
    d2 = d2.cpu().numpy()
    assert (ids < 0).any()
    assert np.all(np.isinf(d2[ids < 0]))
    idx.free()


def test_empty_cluster_keeps_prototype():
    # duplicated data rows -> duplicated init prototypes -> the higher copy gets no members
    X = datagen.blobs(310, 2000, 3, 4)
    X[1] = X[0]
    inits = [np.array([0, 1] + list(range(2, 30)))]
    idx, passes = _step_parity_build(X, [30], 5, inits)
    tr = idx.trace(1)
    assert tr["empties"][0] >= 1
    # after the first update the empty prototype is still the init row (D5)
    np.testing.assert_array_equal(passes[1][1][0][1], X[1])
    idx.free()


def test_nonfinite_and_argument_errors():
    X = datagen.blobs(320, 100, 4, 3)
    X[5, 2] = np.nan
    with pytest.raises(mk.MaskError) as e:
        mk.build(t(X), [4], 2, [np.arange(4)], flags=mk.MASK_VALIDATE_FINITE)
    assert e.value.code == -2
    X[5, 2] = 0.0
    idx = mk.build(t(X), [4], 2, [np.arange(4)])
    with pytest.raises(mk.MaskError):
        idx.query(t(X[:, :3]), knn=3)  # dim mismatch
    with pytest.raises(mk.MaskError):
        idx.query(t(X[:3]), knn=0)
    with pytest.raises(mk.MaskError):
        idx.query(t(X[:3]), knn=3, beam=0)
    idx.free()


def test_host_memory_build_matches_device_build():
    cfg = datagen.CONFIGS[2].scaled(256)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    a = mk.build(t(X), cfg.levels, 4, inits)
    b = mk.build(X, cfg.levels, 4, inits)
    for l in range(1, len(cfg.levels) + 1):
        assert rel_l2(a.prototypes(l), b.prototypes(l)) < 1e-5
    a.free()
    b.free()


# ------------------------------------------------------------------ sparse (K3/K6)
def _csr_dev(rp, col, val, dim):
    return mk.Csr(t(rp), t(col), t(val), dim)


def test_sparse_assign_and_build_parity():
    rp, col, val = datagen.random_csr(400, 3000, 600, 12)
    dense = np.zeros((3000, 600))
    for i in range(3000):
        dense[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    inits = [datagen.init_indices(401, 1, 3000, 64), datagen.init_indices(401, 2, 64, 8)]
    csr = _csr_dev(rp, col, val, 600)
    P = dense[inits[0]].astype(np.float32) + datagen.random_dense(3, 64, 600, scale=0.01)
    lab, d2, _ = mk.assign(csr, t(P))
    check_assignment(dense, P, lab.cpu().numpy(), d2.cpu().numpy(), what="csr assign")
    idx, _ = _step_parity_build(None, [64, 8], 5, inits, csr=csr)
    qrp, qcol, qval = datagen.random_csr(402, 100, 600, 12)
    _query_parity(idx, (rp, col, val), (qrp, qcol, qval), [64, 8], knn=10, beam=1,
                  Qdev=_csr_dev(qrp, qcol, qval, 600), csr=True, dim=600)
    idx.free()


def test_sparse_C4_shaped_replica():
    cfg = datagen.CONFIGS[4].scaled(256)
    rp, col, val = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    csr = _csr_dev(rp, col, val, cfg.dim)
    idx, _ = _step_parity_build(None, cfg.levels, 4, inits, csr=csr)
    idx.free()


def test_seeded_init_when_no_indices_are_given():
    # init_idx = NULL: mask_build draws D2's indices from `seed` (mask_seeded_init); with T = 0
    # every level's prototypes are exactly the drawn rows of its input
    cfg = datagen.CONFIGS[2].scaled(256)
    X = datagen.data(cfg)
    seed = 20221004
    idx = mk.build(t(X), cfg.levels, 0, None, seed=seed)
    Y = X
    for l, k in enumerate(cfg.levels, start=1):
        sel = oracle.seeded_init(seed, l, Y.shape[0], k)
        P = idx.prototypes(l)
        np.testing.assert_array_equal(P, Y[sel])
        Y = P
    idx.free()
    # a Lloyd build from the seed equals the build from the same indices passed explicitly
    inits = [oracle.seeded_init(seed, 1, X.shape[0], cfg.levels[0])]
    for l in range(1, len(cfg.levels)):
        inits.append(oracle.seeded_init(seed, l + 1, cfg.levels[l - 1], cfg.levels[l]))
    a = mk.build(t(X), cfg.levels, 4, None, seed=seed)
    b = mk.build(t(X), cfg.levels, 4, inits)
    for l in range(1, len(cfg.levels) + 1):
        assert rel_l2(a.prototypes(l), b.prototypes(l)) < 1e-5
    a.free()
    b.free()


def test_partition_ordered_rows_give_identical_queries():
    # the leaf scans read the partition-ordered copy of the rows by default; without it
    # (MASK_NO_PARTITION_COPY) they gather through the member ids: same arithmetic, same answers
    cfg = datagen.CONFIGS[3].scaled(2048)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    Q = t(datagen.queries(cfg, count=300))
    a = mk.build(t(X), cfg.levels, 4, inits)
    ids_a, d2_a = {}, {}
    for beam in (1, 3, 8):
        ids_a[beam], d2_a[beam] = a.query(Q, knn=10, beam=beam)
    # the same index structure read without the copy: rebuild with identical prototypes is not
    # guaranteed (atomics), so compare against the oracle descent over this index instead
    L = len(cfg.levels)
    ch = [a.children(l) for l in range(1, L + 1)]
    for beam in (1, 3, 8):
        ref_i, ref_d, gap = oracle.query([a.prototypes(l) for l in range(1, L + 1)], [c[0] for c in ch],
                                         [c[1] for c in ch], X, datagen.queries(cfg, count=300), 10, beam)
        check_queries(ids_a[beam].cpu().numpy(), d2_a[beam].cpu().numpy(), ref_i, ref_d, gap,
                      what=f"partition-ordered leaf scan beam {beam}")
    a.free()
    b = mk.build(t(X), cfg.levels, 4, inits, flags=mk._lib.MASK_NO_PARTITION_COPY)
    chb = [b.children(l) for l in range(1, L + 1)]
    for beam in (1, 3, 8, 64):  # member-id gathers (beam 64: the wide-beam kernel's path)
        ids_b, d2_b = b.query(Q, knn=10, beam=beam)
        ref_i, ref_d, gap = oracle.query([b.prototypes(l) for l in range(1, L + 1)], [c[0] for c in chb],
                                         [c[1] for c in chb], X, datagen.queries(cfg, count=300), 10, beam)
        check_queries(ids_b.cpu().numpy(), d2_b.cpu().numpy(), ref_i, ref_d, gap,
                      what=f"member-id leaf scan beam {beam}")
    b.free()


def test_displacement_trace_matches_the_prototype_steps():
    # mask_get_displacement: dmax_t = max_j ||c_j^(t+1) - c_j^(t)|| (the tolerance-stop
    # quantity, D3), checked against the prototypes the step hook exported for every pass
    cfg = datagen.CONFIGS[2].scaled(256)
    X = datagen.data(cfg)
    seen = {}
    idx = mk.build(t(X), cfg.levels, 6, datagen.all_init_indices(cfg),
                   iter_cb=lambda l, p, P, lab: seen.__setitem__((l, p), P.astype(np.float64)))
    for lv in range(1, len(cfg.levels) + 1):
        tr = idx.trace(lv)
        passes = sorted(p for (l, p) in seen if l == lv)
        assert len(tr["dmax"]) == len(tr["J"]) == len(passes)
        for p in passes[:-1]:
            ref = np.sqrt(((seen[(lv, p + 1)] - seen[(lv, p)]) ** 2).sum(axis=1)).max()
            assert abs(tr["dmax"][p] - ref) <= 1e-5 * ref + 1e-6, (lv, p, tr["dmax"][p], ref)
        assert tr["dmax"][passes[-1]] == 0.0
    idx.free()


@pytest.mark.parametrize("knn,beam", [(32, 32), (1, 32), (32, 1), (17, 5)])
def test_query_limits_match_the_oracle(knn, beam):
    # the largest k_nn and beam the ABI accepts (32 each), ragged values, over a 3-level index
    # with small partitions (answers padded where a partition holds fewer than k_nn rows)
    cfg = datagen.CONFIGS[3].scaled(4096)
    X = datagen.data(cfg)
    idx = mk.build(t(X), cfg.levels, 5, datagen.all_init_indices(cfg))
    Q = datagen.queries(cfg, count=120)
    _query_parity(idx, X, Q, cfg.levels, knn=knn, beam=beam)
    idx.free()


def test_sparse_queries_with_a_beam():
    rp, col, val = datagen.random_csr(410, 2500, 700, 14)
    inits = [datagen.init_indices(411, 1, 2500, 48), datagen.init_indices(411, 2, 48, 6)]
    idx = mk.build(_csr_dev(rp, col, val, 700), [48, 6], 5, inits)
    qrp, qcol, qval = datagen.random_csr(412, 80, 700, 14)
    for beam in (2, 6):
        _query_parity(idx, (rp, col, val), (qrp, qcol, qval), [48, 6], knn=10, beam=beam,
                      Qdev=_csr_dev(qrp, qcol, qval, 700), csr=True, dim=700)
    idx.free()


def test_sparse_queries_longer_than_the_staged_limit():
    """CSR queries with more non-zeros than the kernel stages in shared memory (1024) are
    answered in full from global memory: identical to the oracle descent (no truncation)."""
    d = 6000
    rp, col, val = datagen.random_csr(420, 2000, d, 20)
    inits = [datagen.init_indices(421, 1, 2000, 40), datagen.init_indices(421, 2, 40, 5)]
    idx = mk.build(_csr_dev(rp, col, val, d), [40, 5], 5, inits)
    # 30 queries: a mix of 1500- and 3000-non-zero rows plus short ones
    parts = [datagen.random_csr(422, 10, d, 1500), datagen.random_csr(423, 10, d, 3000),
             datagen.random_csr(424, 10, d, 20)]
    qrp = np.concatenate([[0]] + [p[0][1:] + sum(q[0][-1] for q in parts[:i]) for i, p in enumerate(parts)])
    qcol = np.concatenate([p[1] for p in parts])
    qval = np.concatenate([p[2] for p in parts])
    assert np.diff(qrp).max() > 1024
    for beam in (1, 3):
        _query_parity(idx, (rp, col, val), (qrp.astype(np.int64), qcol, qval), [40, 5], knn=10, beam=beam,
                      Qdev=_csr_dev(qrp.astype(np.int64), qcol, qval, d), csr=True, dim=d)
    idx.free()


def test_csr_structure_errors_are_reported():
    """Invalid CSR input (include/mask.h mask_matrix) is MASK_ERR_ARG from the device-side check,
    for device and host data, builds, queries and mask_assign; the valid matrix still builds."""
    rp, col, val = datagen.random_csr(430, 300, 200, 6)
    inits = [datagen.init_indices(431, 1, 300, 12)]
    bad_order = col.copy()
    bad_order[[6, 7]] = bad_order[[7, 6]]  # row 1: columns not increasing
    bad_range = col.copy()
    bad_range[20] = 200  # column index == dim
    bad_rp = rp.copy()
    bad_rp[5] = bad_rp[4] - 1  # row_ptr decreasing
    for c, r, msg in [(bad_order, rp, "strictly increasing"), (bad_range, rp, "out of range"), (col, bad_rp, "row_ptr")]:
        for dev in (True, False):
            data = _csr_dev(r, c, val, 200) if dev else mk.Csr(r, c, val, 200)
            with pytest.raises(mk.MaskError, match=msg):
                mk.build(data, [12], 2, inits)
        with pytest.raises(mk.MaskError, match=msg):
            mk.assign(_csr_dev(r, c, val, 200), t(np.zeros((4, 200), np.float32)))
    idx = mk.build(_csr_dev(rp, col, val, 200), [12], 2, inits)
    for c, r, msg in [(bad_order, rp, "strictly increasing"), (bad_range, rp, "out of range")]:
        with pytest.raises(mk.MaskError, match=msg):
            idx.query(_csr_dev(r, c, val, 200), knn=3)
        with pytest.raises(mk.MaskError, match=msg):
            idx.query(mk.Csr(r, c, val, 200), knn=3)
    idx.free()


@pytest.mark.parametrize("d", [16, 32, 64, 128])
def test_near_ties_are_decided_exactly(d):
    """Rows placed on the bisector of two prototypes (midpoint + noise orthogonal to their
    difference): the 3xTF32 scores cannot order them, K1 flags them with their two candidates and
    K4 decides between the two in FP64 (the oracle's arithmetic): every label then equals the
    oracle's argmin (lowest index on exact ties), with no tie-window exemption."""
    rng = np.random.default_rng(d)
    k, n = 300, 4096
    P = (rng.standard_normal((k, d)) * 4.0).astype(np.float32)
    a = rng.integers(0, k, n)
    b = (a + 1 + rng.integers(0, k - 1, n)) % k
    diff = P[a].astype(np.float64) - P[b]
    z = rng.standard_normal((n, d))
    z -= (z * diff).sum(1, keepdims=True) / (diff * diff).sum(1, keepdims=True) * diff
    X = ((P[a].astype(np.float64) + P[b]) / 2 + 0.05 * z).astype(np.float32)
    lab, d2, nf = mk.assign(t(X), t(P))
    ref, b1, b2 = oracle.assign(X.astype(np.float64), P.astype(np.float64))
    assert nf > n // 4, f"expected most rows flagged, got {nf}"
    got = lab.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} labels differ from the oracle (rows {bad[:5].tolist()})"


@pytest.mark.parametrize("cid,div,knn,beam", [(3, 256, 10, 40), (3, 256, 32, 256), (2, 64, 10, 100), (5, 2048, 5, 64)])
def test_wide_beam_queries_match_the_oracle(cid, div, knn, beam):
    """Beams above 32 (shared-memory merge-path selection): the same result lists as the
    oracle's descent with the same beam, and recall not below the 32-wide beam's."""
    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    idx = mk.build(t(X), cfg.levels, 6, datagen.all_init_indices(cfg))
    Q = datagen.queries(cfg, count=150)
    _query_parity(idx, X, Q, cfg.levels, knn=knn, beam=beam)
    eids, _, _ = oracle.knn_exact(X, Q, knn)
    wide, _ = idx.query(t(Q), knn=knn, beam=beam)
    narrow, _ = idx.query(t(Q), knn=knn, beam=32)
    # (not a strict superset: a wider candidate set can push a narrow beam's pick out)
    assert oracle.recall(wide.cpu().numpy(), eids) >= oracle.recall(narrow.cpu().numpy(), eids) - 0.02
    with pytest.raises(mk.MaskError):
        idx.query(t(Q), knn=knn, beam=257)
    idx.free()


@pytest.mark.parametrize("cid,div,nq,knn,beam", [(3, 256, 1024, 10, 64), (3, 256, 8192, 10, 8), (2, 64, 2048, 10, 32),
                                                 (5, 2048, 1024, 5, 100), (3, 4096, 700, 32, 97)])
def test_leaf_grouped_queries_match_the_oracle(monkeypatch, cid, div, nq, knn, beam):
    """Large batches (nq x beam >= 65,536, or forced) take the leaf-grouped path: descent ->
    (query, leaf) pairs sorted by leaf -> each leaf's rows staged once for all its queries ->
    per-query merge.  Same result lists as the oracle's descent, and the same ids as the
    per-query kernel wherever the oracle's k-th/(k+1)-th gap is clear."""
    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    idx = mk.build(t(X), cfg.levels, 6, datagen.all_init_indices(cfg))
    Q = datagen.queries(cfg, count=nq)
    monkeypatch.setenv("MASK_QUERY_GROUPED", "0")
    p_ids, p_d2 = idx.query(t(Q), knn=knn, beam=beam)
    p_ids, p_d2 = p_ids.cpu().numpy(), p_d2.cpu().numpy()
    monkeypatch.setenv("MASK_QUERY_GROUPED", "1")
    # with and without the grouped step into level 1, with and without the two-phase leaf scan
    # (the last run splits the grouped level step into many query chunks: a tiny candidate budget)
    # (and one with grouped steps from the top level down)
    for gl, tau, budget, top in (("0", "1", None, "0"), ("1", "1", None, "0"), ("1", "0", None, "0"),
                                 ("1", "1", "3000", "0"), ("1", "1", None, "1")):
        monkeypatch.setenv("MASK_GROUPED_LEVEL", gl)
        monkeypatch.setenv("MASK_LEAF_TAU", tau)
        monkeypatch.setenv("MASK_GROUPED_FROM_TOP", top)
        if budget:
            monkeypatch.setenv("MASK_QUERY_CAND_BUDGET", budget)
        else:
            monkeypatch.delenv("MASK_QUERY_CAND_BUDGET", raising=False)
        try:
            _query_parity(idx, X, Q, cfg.levels, knn=knn, beam=beam)
        except AssertionError as e:
            raise AssertionError(f"MASK_GROUPED_LEVEL={gl} MASK_LEAF_TAU={tau}: {e}") from None
        g_ids, g_d2 = idx.query(t(Q), knn=knn, beam=beam)
        g_ids, g_d2 = g_ids.cpu().numpy(), g_d2.cpu().numpy()
        fin = np.isfinite(p_d2)
        np.testing.assert_array_equal(np.isfinite(g_d2), fin)
        np.testing.assert_allclose(g_d2[fin], p_d2[fin], rtol=1e-5, atol=1e-6)
        same = (g_ids == p_ids).all(1)
        assert same.mean() > 0.99, f"gl={gl} tau={tau}: {(~same).sum()} queries differ between grouped and per-query"
    idx.free()


def _dup_data(seed, n, d, ndup, copies):
    """Rows 0 .. ndup*copies-1 are `copies` copies of `ndup` points (so an init on the first
    rows holds duplicate prototypes and leaves clusters empty), the rest Gaussian."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)).astype(np.float32)
    base = rng.standard_normal((ndup, d)).astype(np.float32)
    X[:ndup * copies] = np.repeat(base, copies, axis=0)
    return X


@pytest.mark.parametrize("d,k,extra", [(16, 64, 0), (64, 96, 0), (64, 96, mk.MASK_FORCE_SIMT), (3, 40, 0)])
def test_empty_farthest_reseed_trajectory(d, k, extra):
    """MASK_EMPTY_FARTHEST (D5b) on data whose init leaves prototypes empty: the
    production build's level-1 trajectory against the oracle's with the same policy (every
    pass's prototypes, so every re-seed's rows, within 1e-4; tie-window rule of D15)."""
    from parity import check_trajectory
    X = _dup_data(700 + d, 6000, d, 30, 8)
    init = [np.arange(k, dtype=np.int64), datagen.init_indices(701, 2, k, 8)]
    idx = mk.build(t(X), [k, 8], 12, init, flags=mk.MASK_BORROW_DATA | mk.MASK_TRACE_PASSES | extra,
                   empty="farthest")
    ref = oracle.lloyd(X.astype(np.float64), init[0], 12, trace=True, empty="farthest")
    assert (np.bincount(ref.passes[0][1], minlength=k) == 0).sum() > 0  # the repair did run
    check_trajectory(X.astype(np.float64), idx.passes(1), ref.passes, what=f"farthest d={d}")
    keep = oracle.lloyd(X.astype(np.float64), init[0], 12)
    assert rel_l2(idx.prototypes(1), keep.P) > 1e-3  # differs from the keep policy's run
    idx.free()


def test_empty_farthest_reseed_csr():
    """The CSR path re-seeds with densified rows (K6 update, K3 assignment)."""
    from parity import check_trajectory
    rp, col, val = datagen.random_csr(720, 4000, 300, 12)
    # unit rows are all at d^2 ~ 2 from prototypes they share no column with: scale each row so
    # the farthest-row order is decided well outside the 1e-5 tie window (D5b reading)
    scale = np.random.default_rng(721).uniform(0.5, 2.0, 4000).astype(np.float32)
    val = (val * np.repeat(scale, np.diff(rp))).astype(np.float32)
    # rows 0..159: 8 copies of rows 0..19
    dense_rows = []
    for i in range(20):
        dense_rows.append((col[rp[i]:rp[i + 1]], val[rp[i]:rp[i + 1]]))
    rows = [dense_rows[i // 8] for i in range(160)] + [(col[rp[i]:rp[i + 1]], val[rp[i]:rp[i + 1]])
                                                       for i in range(160, 4000)]
    rp2 = np.concatenate([[0], np.cumsum([len(c) for c, _ in rows])]).astype(np.int64)
    col2 = np.concatenate([c for c, _ in rows]).astype(np.int32)
    val2 = np.concatenate([v for _, v in rows]).astype(np.float32)
    k = 48
    init = [np.arange(k, dtype=np.int64)]
    idx = mk.build(_csr_dev(rp2, col2, val2, 300), [k], 10, init, flags=mk.MASK_TRACE_PASSES, empty="farthest")
    ref = oracle.lloyd((rp2, col2, val2), init[0], 10, csr_dim=300, trace=True, empty="farthest")
    assert (np.bincount(ref.passes[0][1], minlength=k) == 0).sum() > 0
    check_trajectory((rp2, col2, val2), idx.passes(1), ref.passes, csr_dim=300, what="farthest CSR")
    idx.free()
