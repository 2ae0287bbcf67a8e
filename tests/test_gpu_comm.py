"""The library's multi-GPU code path on one GPU, and concurrent queries.

* NCCL path (BASELINE north_star: one allreduce of the partial sums and counts per iteration;
  SURVEY §8(e)): ``mask_build`` with a one-rank communicator runs every collective of the
  sharded build (init-row allreduce, per-pass [S | n | J | changed] allreduces, the
  combined-statistics control kernel, the upper-level broadcasts, the end-of-build gathers of
  labels and rows) — each an identity on one rank — so its index must equal the single-GPU
  build's labels and child lists, its prototypes within the parity tolerance, and its queries
  must match the oracle's descent.  (NCCL refuses two ranks on one device, so the 2..8-rank
  decomposition is covered by tests/test_dist_gloo.py on CPU.)
* Concurrent ``mask_query`` calls on one index from several host threads and streams (the
  header allows them) return exactly the sequential answers.
"""
import threading

import numpy as np
import pytest

import datagen
import oracle
from parity import check_prototypes, check_queries

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

import paper_2208_02734_b200 as mk  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cid,div", [(2, 64), (3, 1024)])
def test_one_rank_nccl_build_equals_single_gpu_build(cid, div):
    cfg = datagen.CONFIGS[cid].scaled(div)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    T = 6
    ref = mk.build(t(X), cfg.levels, T, inits)
    comm = mk.Comm.init(mk.Comm.unique_id(), 1, 0)
    c0 = mk.collective_count()
    idx = mk.build(t(X), cfg.levels, T, inits, comm=comm, n_global=X.shape[0], row_offset=0)
    assert mk.collective_count() > c0, "the communicator path issued no NCCL call"
    for lv in range(1, len(cfg.levels) + 1):
        a, b = idx.level_info(lv), ref.level_info(lv)
        assert a["passes"] == b["passes"] and a["n_items"] == b["n_items"]
        np.testing.assert_array_equal(idx.labels(lv), ref.labels(lv))
        oa, ma = idx.children(lv)
        ob, mb = ref.children(lv)
        np.testing.assert_array_equal(oa, ob)
        np.testing.assert_array_equal(ma, mb)
        Pa, Pb = idx.prototypes(lv), ref.prototypes(lv)
        check_prototypes(Pa, Pb.astype(np.float64), what=f"comm vs single level {lv}")
    # queries on the communicator-built index against the oracle's descent over that index
    # (its prototypes may differ from the single-GPU build's in the last bits: FP32 sums are
    # combined in another order, so near-tie descents are exempt as everywhere else)
    Qh = datagen.queries(cfg, count=100)
    ia, da = idx.query(t(Qh), knn=10)
    L = len(cfg.levels)
    ch = [idx.children(lv) for lv in range(1, L + 1)]
    ids_ref, d2_ref, gap = oracle.query([idx.prototypes(lv) for lv in range(1, L + 1)], [c[0] for c in ch],
                                        [c[1] for c in ch], X, Qh, 10, 1)
    check_queries(ia.cpu().numpy(), da.cpu().numpy(), ids_ref, d2_ref, gap, what="comm-built index queries")
    idx.free()
    ref.free()
    comm.free()


def test_concurrent_queries_from_threads_and_streams():
    cfg = datagen.CONFIGS[2].scaled(16)
    X = datagen.data(cfg)
    idx = mk.build(t(X), cfg.levels, 5, datagen.all_init_indices(cfg))
    Qs = [t(datagen.queries(cfg, count=2000 + 37 * i)) for i in range(6)]
    seq = [idx.query(Q, knn=10, beam=1 + i % 3) for i, Q in enumerate(Qs)]
    torch.cuda.synchronize()
    out = [None] * len(Qs)
    errs = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    out[i] = idx.query(Qs[i], knn=10, beam=1 + i % 3, stream=s)
            s.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(Qs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for (a, b), (c, d) in zip(out, seq):
        assert torch.equal(a, c) and torch.equal(b, d)
    idx.free()


def test_injected_allocation_failures_are_reported_and_recovered():
    # failure mapping: a device allocation failing in the middle of a build or a
    # query returns MASK_ERR_OOM with a message, frees what the call had taken, and the
    # library keeps working afterwards (same results as an undisturbed build)
    lib = mk._lib.load()
    cfg = datagen.CONFIGS[2].scaled(256)
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    ref = mk.build(t(X), cfg.levels, 3, inits)
    for nth in (0, 5, 40):
        lib.mask_debug_fail_alloc(nth)
        with pytest.raises(mk.MaskError) as e:
            mk.build(t(X), cfg.levels, 3, inits)
        assert e.value.code == -3 and "injected" in str(e.value)
    lib.mask_debug_fail_alloc(-1)
    Qh = np.ascontiguousarray(datagen.queries(cfg, count=50))
    lib.mask_debug_fail_alloc(0)
    with pytest.raises(mk.MaskError) as e:
        ref.query(Qh, knn=5)  # host queries: the staging buffer allocation fails
    assert e.value.code == -3
    lib.mask_debug_fail_alloc(-1)
    again = mk.build(t(X), cfg.levels, 3, inits)
    for lv in range(1, len(cfg.levels) + 1):  # FP32 atomics: equal up to the summation order
        Pa, Pb = again.prototypes(lv), ref.prototypes(lv)
        assert np.linalg.norm(Pa - Pb) <= 1e-5 * np.linalg.norm(Pb)
    a, _ = ref.query(Qh, knn=5)
    assert a.shape == (50, 5) and (a >= 0).any()
    again.free()
    ref.free()
