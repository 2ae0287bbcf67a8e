"""GPU parity of the grouped construction (Algorithm 1) against
the FP64 oracle on the same seeded inputs and split permutation: layer sizes, per-group
clustering (labels = nearest prototype of the item's own group, prototypes = member means
after convergence), child lists, and the exhaustive point-search error of the GPU-built index
(oracle descent over the same index, tie window)."""
import numpy as np
import pytest

import datagen
import oracle
from parity import TIE_REL, check_prototypes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402


def _check_layers(idx, X, lg, nc, perm):
    layers = oracle.grouped_layer_sizes(X.shape[0], lg, nc)
    assert idx.num_levels == len(layers)
    Y, order = X.astype(np.float64), perm
    for l, (n, g) in enumerate(layers, start=1):
        P = idx.prototypes(l).astype(np.float64)
        lab = idx.labels(l)
        assert P.shape[0] == g * nc and lab.shape[0] == n
        base, rem = divmod(n, g)
        start = 0
        means = np.empty_like(P)
        for gi in range(g):
            size = base + (1 if gi >= g - rem else 0)
            items = order[start:start + size]
            start += size
            protos = P[gi * nc:(gi + 1) * nc]
            ref, b1, b2 = oracle.assign(Y[items], protos)
            got = lab[items] - gi * nc
            assert got.min() >= 0 and got.max() < nc, f"layer {l} group {gi}: label outside the group"
            bad = (got != ref) & ~((b2 - b1) < TIE_REL * b2)
            assert not bad.any(), f"layer {l} group {gi}: {int(bad.sum())} labels differ"
            m, _ = oracle.means(Y[items], got.astype(np.int32), protos)
            means[gi * nc:(gi + 1) * nc] = m
        check_prototypes(P, means, what=f"layer {l} prototypes vs member means")
        off, mem = idx.children(l)
        o_ref, m_ref = oracle.children(lab, g * nc)
        np.testing.assert_array_equal(off, o_ref)
        np.testing.assert_array_equal(mem, m_ref)
        Y, order = P, np.arange(P.shape[0])


@pytest.mark.parametrize("lg,nc,n,d", [(16, 8, 1600, 2), (10, 5, 20000, 2), (30, 15, 9001, 3), (64, 20, 50000, 16)])
def test_grouped_build_parity(lg, nc, n, d):
    if d == 2 and n % 8 == 0:
        X = datagen.gaussian_clouds(7, n // 8, 12.0, 2.0)
    else:
        X = datagen.random_dense(8, n, d)
    perm = datagen.group_perm(9, n)
    T = 60  # tiny groups: converged well before the cap, so prototypes are member means
    idx = mk.build_grouped(torch.from_numpy(X).cuda(), lg, nc, T, perm)
    assert [idx.level_info(l)["k"] for l in range(1, idx.num_levels + 1)] == mk.grouped_depth(n, lg, nc)[1]
    _check_layers(idx, X, lg, nc, perm)
    # exhaustive point search of every element: the GPU's answers vs the oracle's
    # descent over the same GPU-built index
    ids, d2 = idx.query(torch.from_numpy(X).cuda(), knn=1)
    ids = ids.cpu().numpy()[:, 0]
    L = idx.num_levels
    P = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
    ch = [idx.children(l) for l in range(1, L + 1)]
    rids, _, gap = oracle.query(P, [c[0] for c in ch], [c[1] for c in ch], X, X, 1, 1)
    ok = gap >= TIE_REL
    np.testing.assert_array_equal(ids[ok], rids[ok, 0])
    err_gpu = float(np.mean(ids != np.arange(n)))
    err_ref = float(np.mean(rids[:, 0] != np.arange(n)))
    assert abs(err_gpu - err_ref) <= (~ok).mean() + 1e-12
    idx.free()


def test_grouped_argument_errors():
    X = torch.from_numpy(datagen.random_dense(1, 100, 2)).cuda()
    with pytest.raises(mk.MaskError):
        mk.build_grouped(X, 10, 10, 5)  # ratio 1:1 never shrinks
    with pytest.raises(mk.MaskError):
        mk.build_grouped(X, 200, 5, 5)  # fewer points than a group
    with pytest.raises(mk.MaskError):
        mk.build_grouped(X, 10, 5, 5, np.zeros(100, np.int64))  # not a permutation


def test_relocation_and_rebuild_parity():
    # §5.1 relocation loop (NEXT-4): every build is Algorithm 1 over the loop's order (same
    # checks as above), every point search agrees with the oracle's descent over that index
    # (tie window), and every next order is the oracle's relocation step applied to the
    # search results (independent implementations of reading G8)
    from paper_2208_02734_b200.relocate import relocate_and_rebuild
    lg, nc = 16, 8
    X = datagen.gaussian_clouds(11, 200, 12.0, 2.0)
    n = X.shape[0]
    perm = datagen.group_perm(11, n)
    g = oracle.grouped_layer_sizes(n, lg, nc)[0][1]
    recs = []

    def hook(i, order, idx, found, reached):
        _check_layers(idx, X, lg, nc, order)
        L = idx.num_levels
        ch = [idx.children(l) for l in range(1, L + 1)]
        ids, _, gap = oracle.query([idx.prototypes(l) for l in range(1, L + 1)], [c[0] for c in ch],
                                   [c[1] for c in ch], X, X, 1, 1)
        f_ref = ids[:, 0] == np.arange(n)
        bad = (f_ref != found) & (gap >= TIE_REL)
        assert not bad.any(), f"iteration {i}: {int(bad.sum())} point searches differ"
        sure = (f_ref == found) & (gap >= TIE_REL) & ~found
        r_ref = np.where(ids[:, 0] >= 0, idx.labels(1)[np.maximum(ids[:, 0], 0)] // nc, -1)
        assert np.array_equal(r_ref[sure], reached[sure]), f"iteration {i}: reached partitions differ"
        recs.append((order.copy(), found.copy(), reached.copy()))

    keys = lambda i, m: datagen.relocation_keys(77, i, m)  # noqa: E731
    errs = relocate_and_rebuild(torch.from_numpy(X).cuda(), lg, nc, 30, perm, 3, keys, hook=hook)
    assert len(errs) == 4 and len(recs) == 4
    for i, (order, found, reached) in enumerate(recs):
        assert errs[i] == float(np.mean(~found))
        if i + 1 < len(recs):
            np.testing.assert_array_equal(recs[i + 1][0], oracle.relocation_order(order, g, found, reached,
                                                                                  keys(i + 1, n)))
    assert min(errs[1:]) < errs[0]  # relocation helps (Table 1's trend)
