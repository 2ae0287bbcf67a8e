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
