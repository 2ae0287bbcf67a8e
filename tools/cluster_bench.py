"""§3.4 distributed mode on one B200: W independent node indexes over
contiguous row ranges of a config (LocalCluster, zero collectives in the builds), then the
batched cluster query for several epsilon: routing (K14), routed per-node descents (K9), merge
(K14).  Reports per-node build time, query time per stage (CUDA events), QPS, the routed
fraction and recall@k against the oracle's exact k-NN on a sample.

    python tools/cluster_bench.py [--config 2] [--nodes 4] [--sample 300]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402
from paper_2208_02734_b200.cluster import LocalCluster  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--nodes", type=int, default=4)
    ap.add_argument("--sample", type=int, default=300)
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.config]
    X = datagen.data(cfg)
    Q = datagen.queries(cfg)
    n, W = X.shape[0], a.nodes
    bounds = [(r * n // W, (r + 1) * n // W) for r in range(W)]
    inits = []
    for r, (lo, hi) in enumerate(bounds):
        m, per = hi - lo, []
        for l, kk in enumerate(cfg.levels, start=1):
            kk = max(1, kk // W) if l == 1 else kk  # each node clusters its own share
            per.append(datagen.init_indices(cfg.cid * 100 + r, l, m, kk))
            m = kk
        inits.append(per)
    levels = [max(1, cfg.levels[0] // W)] + list(cfg.levels[1:])
    parts = [torch.from_numpy(X[lo:hi]).cuda() for lo, hi in bounds]
    torch.cuda.synchronize()
    t0 = time.time()
    cl = LocalCluster.build(parts, levels, cfg.iters, inits, flags=mk.MASK_BORROW_DATA)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    print(json.dumps({"workload": cfg.name, "nodes": W, "levels_per_node": levels, "build_s_all_nodes": build_s,
                      "build_collectives": cl.build_collectives, "registry_rows": int(sum(cl.registry.counts))}),
          flush=True)
    Qd = torch.from_numpy(Q).cuda()
    eids, _, _ = oracle.knn_exact(X, Q[:a.sample], cfg.knn)
    dtop = np.sqrt(((Q[:2000, None, :].astype(np.float64) - cl.registry.protos.cpu().numpy()[None]) ** 2).sum(-1)).min(1)
    for eps in (math.inf, float(np.percentile(dtop, 90)) * 1.5, float(np.percentile(dtop, 50)) * 1.2,
                float(np.percentile(dtop, 50))):
        st = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        best = None
        for _ in range(4):
            ev[0].record(st)
            routed = cl.registry.route(Qd, eps)
            ev[1].record(st)
            ans = [nd.query_routed(Qd, routed, i, cl.registry.id_bases[i], knn=cfg.knn) for i, nd in enumerate(cl.nodes)]
            ev[2].record(st)
            ids, d2 = mk.merge(torch.stack([x[0] for x in ans]), torch.stack([x[1] for x in ans]))
            ev[3].record(st)
            torch.cuda.synchronize()
            t = [ev[0].elapsed_time(ev[i]) for i in (1, 2, 3)]
            best = t if best is None or t[2] < best[2] else best
        rec = oracle.recall(ids[:a.sample].cpu().numpy(), eids)
        frac = float(routed.float().mean())
        print(json.dumps({"epsilon": eps, "route_ms": best[0], "descents_ms": best[1] - best[0],
                          "merge_ms": best[2] - best[1], "total_ms": best[2], "qps": Q.shape[0] / (best[2] / 1e3),
                          "routed_fraction": frac, "recall": rec, "recall_sample": a.sample}), flush=True)
    cl.free()


if __name__ == "__main__":
    main()
