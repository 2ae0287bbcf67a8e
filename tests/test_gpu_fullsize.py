"""Full-size parity at BASELINE.json sizes, in the launch configuration bench.py times
(mask_build of the whole config through the C-ABI, device data, default flags), checked on
sampled outputs the oracle computes one by one (SURVEY.md §8(c) "Coverage per config"):

* step mode: at checked passes, the GPU labels of sampled rows vs the oracle's assignment of
  those rows to the GPU's own P_t (tie window 1e-5), and P_{t+1} vs the oracle's FP64 member
  means of the GPU's full label vector (1e-4 relative L2, BASELINE.json north_star);
* upper levels in full; child lists vs {i : labels[i] = j};
* queries: a sample of the config's queries, oracle descent over the GPU-built index.
"""
import numpy as np
import pytest

import datagen
import oracle
from parity import check_assignment, check_prototypes, check_queries

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402


def _full_config(cid, sample_rows, checked, n_queries):
    cfg = datagen.CONFIGS[cid]
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    rng = np.random.default_rng(cid)
    rows = np.sort(rng.choice(cfg.n, sample_rows, replace=False))
    seen = {}

    def cb(level, p, P, labels):
        if level == 1:
            seen[p] = (P, labels)
        else:
            seen[(level, p)] = (P, labels)

    Xd = torch.from_numpy(X).to("cuda:0")
    idx = mk.build(Xd, cfg.levels, cfg.iters, inits, flags=mk.MASK_BORROW_DATA, iter_cb=cb)
    passes = sorted(p for p in seen if isinstance(p, int))
    assert len(passes) == idx.level_info(1)["passes"]
    last = passes[-1]
    check_passes = sorted({0, 1, last // 2, last - 1, last} & set(passes)) if checked is None else checked
    X64 = X.astype(np.float64)
    for p in check_passes:
        P, lab = seen[p]
        check_assignment(X64[rows], P, lab[rows], what=f"{cfg.name} level 1 pass {p}")
        if p + 1 in seen and not np.array_equal(seen[p + 1][0], P):
            P_ref, _ = oracle.means(X64, lab, P.astype(np.float64))
            check_prototypes(seen[p + 1][0], P_ref, what=f"{cfg.name} level 1 update after pass {p}")
    np.testing.assert_array_equal(idx.labels(1), seen[last][1])
    # upper levels: every pass in full
    for l in range(2, len(cfg.levels) + 1):
        Y = idx.prototypes(l - 1).astype(np.float64)
        lp = sorted(p for (lv, p) in [key for key in seen if isinstance(key, tuple)] if lv == l)
        for p in lp:
            P, lab = seen[(l, p)]
            check_assignment(Y, P, lab, what=f"{cfg.name} level {l} pass {p}")
            if (l, p + 1) in seen and not np.array_equal(seen[(l, p + 1)][0], P):
                P_ref, _ = oracle.means(Y, lab, P.astype(np.float64))
                check_prototypes(seen[(l, p + 1)][0], P_ref, what=f"{cfg.name} level {l} update {p}")
    # child lists
    for l in range(1, len(cfg.levels) + 1):
        off, mem = idx.children(l)
        o_ref, m_ref = oracle.children(idx.labels(l), cfg.levels[l - 1])
        np.testing.assert_array_equal(off, o_ref)
        np.testing.assert_array_equal(mem, m_ref)
    # queries (sample), oracle descent over the GPU-built index
    Q = datagen.queries(cfg)
    qs = np.sort(rng.choice(len(Q), n_queries, replace=False))
    ids, d2 = idx.query(torch.from_numpy(Q).to("cuda:0"), knn=cfg.knn)
    ids, d2 = ids.cpu().numpy()[qs], d2.cpu().numpy()[qs]
    L = len(cfg.levels)
    P = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
    ch = [idx.children(l) for l in range(1, L + 1)]
    rids, rd2, gap = oracle.query(P, [c[0] for c in ch], [c[1] for c in ch], X, Q[qs], cfg.knn, 1)
    check_queries(ids, d2, rids, rd2, gap, what=f"{cfg.name} queries")
    idx.free()


def test_C2_full_size_bench_configuration():
    _full_config(2, sample_rows=4096, checked=None, n_queries=2000)


def test_C3_full_size():
    _full_config(3, sample_rows=4096, checked=[0, 10, 20], n_queries=500)


def test_C4_full_size_sparse():
    """C4 at full size (1e6 CSR rows, d = 10,000, ~0.5 % non-zeros, k = 8192/256): step-mode
    parity of sampled rows at checked passes, FP64 update checks, child lists, queries."""
    cfg = datagen.CONFIGS[4]
    rp, col, val = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    rng = np.random.default_rng(4)
    rows = np.sort(rng.choice(cfg.n, 1024, replace=False))
    seen = {}

    def cb(level, p, P, labels):
        if level == 1 and p in (0, 1, 7):
            seen[p] = (P, labels)
        elif level == 1:
            seen[p] = (None, None)

    dev = "cuda:0"
    csr = mk.Csr(torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev), torch.from_numpy(val).to(dev), cfg.dim)
    T = 8
    idx = mk.build(csr, cfg.levels, T, inits, flags=mk.MASK_BORROW_DATA, iter_cb=cb)
    for p in (0, 1, 7):
        if p not in seen or seen[p][0] is None:
            continue
        P, lab = seen[p]
        sub_rp = np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])])
        sub_col = np.concatenate([col[rp[r]:rp[r + 1]] for r in rows])
        sub_val = np.concatenate([val[rp[r]:rp[r + 1]] for r in rows])
        dense = np.zeros((len(rows), cfg.dim))
        for i in range(len(rows)):
            dense[i, sub_col[sub_rp[i]:sub_rp[i + 1]]] = sub_val[sub_rp[i]:sub_rp[i + 1]]
        check_assignment(dense, P, lab[rows], what=f"C4 level 1 pass {p}")
        if p == 0 and 1 in seen and seen[1][0] is not None:
            S, cnt = oracle.cluster_sums_csr((rp, col, val), cfg.dim, lab, cfg.levels[0])
            P_ref, _ = oracle.means_from_sums(S, cnt, P.astype(np.float64))
            check_prototypes(seen[1][0], P_ref, what="C4 level 1 update after pass 0")
    off, mem = idx.children(1)
    o_ref, m_ref = oracle.children(idx.labels(1), cfg.levels[0])
    np.testing.assert_array_equal(off, o_ref)
    qrp, qcol, qval = datagen.queries(cfg, count=200)
    ids, d2 = idx.query(mk.Csr(torch.from_numpy(qrp).to(dev), torch.from_numpy(qcol).to(dev),
                               torch.from_numpy(qval).to(dev), cfg.dim), knn=cfg.knn)
    L = len(cfg.levels)
    P = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
    ch = [idx.children(l) for l in range(1, L + 1)]
    rids, rd2, gap = oracle.query(P, [c[0] for c in ch], [c[1] for c in ch], (rp, col, val), (qrp, qcol, qval),
                                  cfg.knn, 1, dim=cfg.dim, x_csr=True, q_csr=True)
    check_queries(ids.cpu().numpy(), d2.cpu().numpy(), rids, rd2, gap, what="C4 queries")
    tm = idx.timing(1)
    print("C4 level-1 timing", tm)
    idx.free()
