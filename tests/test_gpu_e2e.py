"""End-to-end parity of whole builds at the configs' iteration counts (BASELINE.json
north_star: "Prototypes must agree within 1e-4 relative L2 error per level"; SURVEY.md §8(c)
"End-to-end ... from the same init"; PAPER.md P:641-668 levels, P:654-655 Lloyd).

Every build here is the production path in the bench's launch configuration (device data,
MASK_BORROW_DATA | MASK_TIME_ASSIGN, fused small levels (K11), label sort, K1/K3/K4, no
iteration callback); MASK_TRACE_PASSES only copies each pass's prototypes and labels aside on
the device.  Each level's trajectory is compared with the FP64 oracle's Lloyd run from the same
level input and init rows by ``parity.check_trajectory``: in-sync passes must agree within
1e-4; if the label sequences part, the first differing pass must be a near-tie decision inside
the oracle's own 1e-5 window, and every later GPU pass is checked in step mode (D15).
The whole-index comparison against ``oracle.build_index`` is asserted at 1e-4 per level while
level 1 stays in sync.  ``MASK_E2E_REPORT=<path>`` appends one JSON line per level."""
import json
import os

import numpy as np
import pytest

import datagen
import oracle
from parity import PROTO_REL, check_trajectory, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402

DEV = "cuda:0"
BENCH_FLAGS = mk.MASK_BORROW_DATA | mk.MASK_TIME_ASSIGN


def _report(rec):
    path = os.environ.get("MASK_E2E_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _e2e(cfg, extra_flags=0, expect_kernels=None, whole_index=True):
    sparse = cfg.sparse
    inits = datagen.all_init_indices(cfg)
    if sparse:
        rp, col, val = datagen.data(cfg)
        data = mk.Csr(torch.from_numpy(rp).to(DEV), torch.from_numpy(col).to(DEV), torch.from_numpy(val).to(DEV),
                      cfg.dim)
        Y1 = (rp, col, val)
    else:
        X = datagen.data(cfg)
        data = torch.from_numpy(X).to(DEV)
        Y1 = X.astype(np.float64)
    idx = mk.build(data, cfg.levels, cfg.iters, inits, flags=BENCH_FLAGS | mk.MASK_TRACE_PASSES | extra_flags)
    reports = []
    Y = Y1
    chain = []  # the oracle's own levels (each from the oracle's previous level): build_index
    for l in range(1, len(cfg.levels) + 1):
        csr_dim = cfg.dim if (sparse and l == 1) else None
        gpu = idx.passes(l)
        res = oracle.lloyd(Y, inits[l - 1], cfg.iters, csr_dim=csr_dim, trace=True)
        ref = res.passes
        if l == 1:
            chain.append(res.P)  # level 1: the same input on both sides
        rep = check_trajectory(Y, gpu, ref, csr_dim=csr_dim, what=f"{cfg.name} level {l}")
        tm = idx.timing(l)
        rep.update(config=cfg.name, level=l, T=cfg.iters, flags=int(extra_flags), kernel=tm["assign_kernel"])
        if expect_kernels:
            assert tm["assign_kernel"] == expect_kernels[l - 1], f"level {l}: ran {tm['assign_kernel']}"
        # stored labels / prototypes are the final pass
        np.testing.assert_array_equal(idx.labels(l), gpu[-1][1])
        np.testing.assert_array_equal(idx.prototypes(l), gpu[-1][0])
        reports.append(rep)
        _report(rep)
        Y = idx.prototypes(l).astype(np.float64)  # the next level's input as the GPU built it
    if whole_index:
        # the whole index against oracle.build_index's chain (each level from the oracle's own
        # previous level; level 1 shares the run above): held to 1e-4 per level while every
        # level below stayed in sync
        for l in range(2, len(cfg.levels) + 1):
            chain.append(oracle.lloyd(chain[-1], inits[l - 1], cfg.iters).P)
        for l in range(1, len(cfg.levels) + 1):
            e = rel_l2(idx.prototypes(l), chain[l - 1])
            reports[l - 1]["whole_index_rel_l2"] = e
            if all(r["diverged_at"] is None for r in reports[:l]):
                assert e <= PROTO_REL, f"{cfg.name} level {l}: whole-index prototype rel L2 {e:.3e}"
    idx.free()
    return reports


def test_e2e_C1_full_fused():
    """C1 at full size (T = 20): both levels run the fused small-level loop (K11)."""
    cfg = datagen.CONFIGS[1]
    _e2e(cfg, expect_kernels=["K11-fused-small-level", "K11-fused-small-level"])


def test_e2e_C1_full_per_pass():
    cfg = datagen.CONFIGS[1]
    _e2e(cfg, extra_flags=mk.MASK_NO_FUSED)


@pytest.mark.parametrize("extra", [0, mk.MASK_NO_FUSED])
def test_e2e_C2_div64_T25(extra):
    """The C2/64 replica at the config's T = 25 (level 1 of 15,625 rows, k = 64: K11 by
    default, the per-pass kernels with MASK_NO_FUSED)."""
    cfg = datagen.CONFIGS[2].scaled(64)
    _e2e(cfg, extra_flags=extra)


def test_e2e_fused_vs_per_pass_small_levels():
    """The fused loop (K11) and the per-pass kernels run the same Lloyd iteration: on the C2/64
    replica their level-1 trajectories agree pass for pass while both stay in sync with the
    oracle, and their final prototypes agree within 1e-4 when neither diverged."""
    cfg = datagen.CONFIGS[2].scaled(64)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    a = mk.build(torch.from_numpy(X).to(DEV), cfg.levels, cfg.iters, inits, flags=BENCH_FLAGS | mk.MASK_TRACE_PASSES)
    b = mk.build(torch.from_numpy(X).to(DEV), cfg.levels, cfg.iters, inits,
                 flags=BENCH_FLAGS | mk.MASK_TRACE_PASSES | mk.MASK_NO_FUSED)
    assert a.timing(1)["assign_kernel"] == "K11-fused-small-level"
    assert b.timing(1)["assign_kernel"] != "K11-fused-small-level"
    pa, pb = a.passes(1), b.passes(1)
    for t in range(min(len(pa), len(pb))):
        assert rel_l2(pa[t][0], pb[t][0]) <= PROTO_REL, f"pass {t}"
        if not np.array_equal(pa[t][1], pb[t][1]):
            break
    else:
        assert len(pa) == len(pb)
        for l in range(1, len(cfg.levels) + 1):
            assert rel_l2(a.prototypes(l), b.prototypes(l)) <= PROTO_REL
    a.free()
    b.free()


@pytest.mark.slow
def test_e2e_C2_full_T25():
    """C2 at full size and T = 25 (bench configuration): K1 at level 1, K11 above."""
    cfg = datagen.CONFIGS[2]
    _e2e(cfg, expect_kernels=["K1-tcgen05-3xtf32", "K11-fused-small-level", "K11-fused-small-level"])


@pytest.mark.slow
def test_e2e_C3_div64_T20():
    cfg = datagen.CONFIGS[3].scaled(64)
    _e2e(cfg)


@pytest.mark.slow
def test_e2e_C4_div4_T15():
    """The sparse config (CSR, d = 10,000) ÷ 4 at T = 15 (250,000 rows, k = 2048 / 64): K3 at
    level 1, dense d = 10,000 above."""
    cfg = datagen.CONFIGS[4].scaled(4)
    _e2e(cfg)


@pytest.mark.slow
def test_e2e_C5_div256_T15():
    cfg = datagen.CONFIGS[5].scaled(256)
    _e2e(cfg)


@pytest.mark.slow
@pytest.mark.parametrize("cid,div", [(5, 64)])
def test_e2e_survey_replicas_long(cid, div):
    """SURVEY §8(c)'s exact C5 replica size (C5 / 64: 1.56M x 128, k = 4096 / 64 / 1, T = 15),
    which takes the FP64 oracle tens of minutes on the host.  Opt-in (MASK_E2E_LONG=1) so the
    default GPU suite stays within minutes; the committed report is profiles/r02_e2e_parity.jsonl
    (all three levels in sync to the last pass, final rel L2 2.5e-8).  Full C4 needs more than
    50 minutes of oracle time on the box's cores; C4 / 4 is in the default suite."""
    if os.environ.get("MASK_E2E_LONG") != "1":
        pytest.skip("set MASK_E2E_LONG=1 (tens of minutes of FP64 oracle time)")
    cfg = datagen.CONFIGS[cid].scaled(div) if div > 1 else datagen.CONFIGS[cid]
    _e2e(cfg, whole_index=False)
