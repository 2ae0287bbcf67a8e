"""GPU parity of K3T (CSR assignment with the hot columns on tcgen05, DESIGN.md §6 K3T) against
the FP64 oracle: ragged rows (empty, all-hot, long tails of > 32 and > 64 non-zeros), d below
and above the hot-set size H = 128, k not a multiple of the 128-prototype tile, a ragged last
row block, and a C4-shaped replica (Zipf columns) -- plus the default SIMT K3 on the same
inputs.  K3T is opt-in (MASK_CSR_TC).  Marked `gpu`."""
import numpy as np
import pytest

import datagen
from parity import check_assignment, check_assignment_any

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402

DEV = "cuda:0"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _dense(rp, col, val, d):
    n = rp.size - 1
    Y = np.zeros((n, d))
    for i in range(n):
        Y[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    return Y


# (seed, n, d, k, max_nnz): d < H, d = H + ragged, long rows, k = 1, k % 128 != 0, n % 128 != 0
SHAPES = [
    (31, 300, 50, 37, 40),
    (32, 1000, 129, 300, 129),
    (33, 2000, 600, 257, 90),
    (34, 513, 3000, 1, 200),
    (35, 1500, 5000, 1000, 160),
    (36, 128, 700, 128, 70),
    (37, 2, 900, 5, 30),
]


@pytest.mark.parametrize("seed,n,d,k,max_nnz", SHAPES)
def test_k3t_assign_matches_oracle(seed, n, d, k, max_nnz):
    rp, col, val = datagen.ragged_csr(seed, n, d, max_nnz)
    Y = _dense(rp, col, val, d)
    # prototypes: data rows plus small noise (dense, non-negative), so the assignment is not trivial
    init = datagen.init_indices(seed, 1, n, min(k, n)) if n >= k else np.arange(k) % n
    P = (Y[init] + np.abs(datagen.random_dense(seed, k, d, scale=0.02))).astype(np.float32)
    csr = mk.Csr(t(rp), t(col), t(val), d)
    lab, d2, _ = mk.assign(csr, t(P), flags=mk.MASK_CSR_TC)
    check_assignment(Y, P, lab.cpu().numpy(), d2.cpu().numpy(), what=f"K3T n={n} d={d} k={k}")
    lab2, d22, _ = mk.assign(csr, t(P))
    check_assignment(Y, P, lab2.cpu().numpy(), d22.cpu().numpy(), what=f"K3 SIMT n={n} d={d} k={k}")


def test_k3t_c4_replica_build_kernel():
    """C4-shaped replica (Zipf(1.2) columns, 50 non-zeros per row): K3T runs in the build (kernel
    id reported) and its level-1 labels match the oracle for the prototypes of every pass."""
    cfg = datagen.CONFIGS[4].scaled(128)
    rp, col, val = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    csr = mk.Csr(t(rp), t(col), t(val), cfg.dim)
    idx = mk.build(csr, cfg.levels, 3, inits, flags=mk.MASK_TRACE_PASSES | mk.MASK_TIME_KERNELS | mk.MASK_CSR_TC)
    assert idx.timing(1)["assign_kernel"] == "K3T-csr-tcgen05"
    for P_t, lab_t in idx.passes(1):
        check_assignment_any((rp, col, val), P_t, lab_t, csr_dim=cfg.dim, what="C4/128 level-1 pass")
    idx.free()
