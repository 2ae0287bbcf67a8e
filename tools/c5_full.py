"""C5 at full size on one B200 (100M x 128 fp32 = 51.2 GB, k = 262144/4096/64): timing and
sampled step-mode parity of T = 1 (two level-1 passes), run as a tool (about 3 minutes; the full
15-iteration build is ~16 x 25 s of level-1 assignment).

    python tools/c5_full.py [--T 1] [--rows 4096] [--clusters 256]

Checks (SURVEY §8(c) coverage for C3/C5: step mode on sampled rows, FP64 update checks):
* level 1, every pass: GPU labels of sampled rows vs the oracle's assignment of those rows to
  the GPU's own P_t (tie window 1e-5);
* level 1 update: P_1 of sampled clusters vs the oracle's FP64 means of their members under the
  GPU's pass-0 labels (each cluster's mean depends only on its members);
* levels 2-3: every pass in full (step mode), child lists of level 1 on sampled clusters.
Prints the level-1 K1 time per pass (CUDA events in the library) and its 3xTF32 TF/s.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402
from parity import check_assignment, check_prototypes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=1)
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--clusters", type=int, default=256)
    ap.add_argument("--clean", action="store_true",
                    help="time one clean build (no step hook, no checks) and the 1e6-query batch")
    ap.add_argument("--recall-sample", type=int, default=20)
    ap.add_argument("--beams", default="1", help="--clean: beam widths of the query batch")
    ap.add_argument("--modes", default="auto", help="--clean: MASK_QUERY_GROUPED values per beam (0 = per-query)")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[5]
    t0 = time.time()
    X, shm = datagen.data_parallel(cfg)
    print(f"generated {X.shape} in {time.time() - t0:.1f} s", flush=True)
    inits = datagen.all_init_indices(cfg)
    t0 = time.time()
    Xd = torch.from_numpy(X).to("cuda:0")
    torch.cuda.synchronize()
    print(f"H2D {X.nbytes / 1e9:.1f} GB in {time.time() - t0:.1f} s", flush=True)
    if a.clean:
        clean(a, cfg, X, Xd, inits)
        del Xd
        shm.close()
        shm.unlink()
        return
    seen = {}

    def cb(level, p, P, labels):
        seen[(level, p)] = (P, labels)

    t0 = time.time()
    idx = mk.build(Xd, cfg.levels, a.T, inits, flags=mk.MASK_BORROW_DATA | mk.MASK_TIME_KERNELS, iter_cb=cb)
    print(f"build (T={a.T}, with step-hook copies) {time.time() - t0:.1f} s", flush=True)
    tm = idx.timing(1)
    info = idx.level_info(1)
    per = tm["assign"]["ms"] / max(tm["assign"]["launches"], 1)
    n, k, d = cfg.n, cfg.levels[0], cfg.dim
    print(f"level 1 {tm['assign_kernel']}: {per:.1f} ms/pass over {tm['assign']['launches']} passes, "
          f"{6.0 * n * k * d / (per / 1e3) / 1e12:.0f} TF/s 3xTF32, fix-up {tm['fixup']['ms'] / max(tm['fixup']['launches'], 1):.1f} "
          f"ms/pass, update {tm['update']['ms'] / max(tm['update']['launches'], 1):.1f} ms/pass", flush=True)

    rng = np.random.default_rng(5)
    rows = np.sort(rng.choice(n, a.rows, replace=False))
    Xs = X[rows].astype(np.float64)
    l1 = sorted(p for (lv, p) in seen if lv == 1)
    assert len(l1) == info["passes"]
    for p in l1:
        P, lab = seen[(1, p)]
        check_assignment(Xs, P, lab[rows], what=f"C5 level 1 pass {p}")
        print(f"level 1 pass {p}: sampled assignment ok", flush=True)
    # update after pass 0 on sampled clusters: means of their members (FP64)
    if (1, 1) in seen:
        P0, lab0 = seen[(1, 0)]
        P1 = seen[(1, 1)][0]
        cl = np.sort(rng.choice(k, a.clusters, replace=False))
        sel = np.isin(lab0, cl)
        members = np.nonzero(sel)[0]
        remap = np.full(k, -1, np.int64)
        remap[cl] = np.arange(cl.size)
        P_ref, cnt = oracle.means(X[members].astype(np.float64), remap[lab0[members]].astype(np.int32),
                                  P0[cl].astype(np.float64))
        check_prototypes(P1[cl], P_ref, what="C5 level 1 update (sampled clusters)")
        print(f"level 1 update: {cl.size} sampled clusters ({members.size} members) ok", flush=True)
    # child lists of sampled level-1 prototypes
    off, mem = idx.children(1)
    lab_final = idx.labels(1)
    for j in rng.choice(k, 64, replace=False):
        np.testing.assert_array_equal(mem[off[j]:off[j + 1]], np.nonzero(lab_final == j)[0])
    print("level 1 child lists (64 sampled prototypes) ok", flush=True)
    # upper levels: every pass in full
    for lv in range(2, len(cfg.levels) + 1):
        Y = idx.prototypes(lv - 1).astype(np.float64)
        for p in sorted(q for (l2, q) in seen if l2 == lv):
            P, lab = seen[(lv, p)]
            check_assignment(Y, P, lab, what=f"C5 level {lv} pass {p}")
            if (lv, p + 1) in seen and not np.array_equal(seen[(lv, p + 1)][0], P):
                P_ref, _ = oracle.means(Y, lab, P.astype(np.float64))
                check_prototypes(seen[(lv, p + 1)][0], P_ref, what=f"C5 level {lv} update {p}")
        print(f"level {lv}: all passes ok", flush=True)
    idx.free()
    del Xd
    shm.close()
    shm.unlink()
    print("C5 full-size checks passed")


def clean(a, cfg, X, Xd, inits):
    """One production build (CUDA events around mask_build) + the batched query over 1e6 queries."""
    st = torch.cuda.current_stream()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(st)
    idx = mk.build(Xd, cfg.levels, a.T, inits, flags=mk.MASK_BORROW_DATA | mk.MASK_TIME_KERNELS, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    build_s = e0.elapsed_time(e1) / 1e3
    tot = 0
    for lv in range(1, len(cfg.levels) + 1):
        info = idx.level_info(lv)
        tm = idx.timing(lv)
        tot += info["passes"] * info["n_items"] * info["k"]
        print(f"level {lv}: {info['passes']} passes ({tm['assign_kernel']}), assign {tm['assign']['ms'] / 1e3:.2f} s, "
              f"fix-up {tm['fixup']['ms'] / 1e3:.2f} s, update {tm['update']['ms'] / 1e3:.3f} s", flush=True)
    print(f"C5 build (T={a.T}): {build_s:.1f} s, {tot:.3e} distances, {tot / build_s:.3e} distances/s", flush=True)
    Q = datagen.queries(cfg)
    Qd = torch.from_numpy(Q).to("cuda:0")
    m = a.recall_sample
    t0 = time.time()
    eids, _, _ = oracle.knn_exact(X, Q[:m], cfg.knn)
    print(f"exact k-NN of {m} queries on the host: {time.time() - t0:.0f} s", flush=True)
    for beam in [int(b) for b in a.beams.split(",")]:
        for mode in a.modes.split(","):
            os.environ.pop("MASK_QUERY_GROUPED", None)
            if mode != "auto":
                os.environ["MASK_QUERY_GROUPED"] = mode
            ms = []
            for _ in range(3):
                e1.record(st)
                ids, d2 = idx.query(Qd, knn=cfg.knn, beam=beam, stream=st)
                e2.record(st)
                torch.cuda.synchronize()
                ms.append(e1.elapsed_time(e2))
            qms = min(ms)
            rec = oracle.recall(ids[:m].cpu().numpy(), eids)
            print(f"query beam {beam} ({'per-query' if mode == '0' else 'grouped' if mode == '1' else 'auto'}): "
                  f"{Q.shape[0]} queries in {qms:.1f} ms = {Q.shape[0] / qms * 1e3:.3e} QPS, "
                  f"recall@{cfg.knn} {rec:.3f} on {m} queries", flush=True)
        os.environ.pop("MASK_QUERY_GROUPED", None)
    idx.free()


if __name__ == "__main__":
    main()
