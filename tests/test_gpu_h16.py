"""GPU parity of K1's 3xFP16 path (kind::f16, d = 64 / 128; DESIGN.md §6 K1 "3xFP16") against the
FP64 oracle and against the 3xTF32 path (MASK_TC_TF32): the data scale is chosen per level from
max |x|, so very large and very small magnitudes must give the same exact labels; near ties are
decided by K4 with the oracle's arithmetic in both paths.  Marked `gpu`."""
import numpy as np
import pytest

import datagen
from parity import check_assignment, check_prototypes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import oracle  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("n,d,k,scale", [(3000, 64, 700, 1.0), (2500, 128, 300, 1.0), (2000, 64, 257, 3.0e4),
                                         (2000, 128, 129, 2.0e-5), (700, 64, 1, 1.0)])
def test_h16_assign_matches_oracle_and_tf32(n, d, k, scale):
    X = (datagen.blobs(91, n, d, 12, spread=6.0, sigma=1.0) * scale).astype(np.float32)
    init = datagen.init_indices(91, 1, n, k)
    P = (X[init] + datagen.random_dense(92, k, d, scale=0.05 * scale)).astype(np.float32)
    lab, d2, _ = mk.assign(t(X), t(P))
    check_assignment(X, P, lab.cpu().numpy(), d2.cpu().numpy(), what=f"3xFP16 n={n} d={d} k={k} x{scale:g}")
    lab_t, _, _ = mk.assign(t(X), t(P), flags=mk.MASK_TC_TF32)
    assert np.array_equal(lab.cpu().numpy(), lab_t.cpu().numpy()), "3xFP16 and 3xTF32 labels differ"


def test_h16_build_reports_kernel_and_matches_oracle():
    cfg = datagen.CONFIGS[3].scaled(256)  # C3 rows (d = 64), k = 256 / 4 / ...
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    idx = mk.build(t(X), cfg.levels, 6, inits, flags=mk.MASK_TIME_KERNELS)
    assert idx.timing(1)["assign_kernel"] == "K1-tcgen05-3xfp16"
    ref = oracle.build_index(X, inits, 6)
    for l in range(1, len(cfg.levels) + 1):
        check_prototypes(idx.prototypes(l), ref.levels[l - 1].P, what=f"3xFP16 build level {l}")
    idx.free()
