"""A compact pass over every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_workload.py

K1 persistent (d = 16) and tiled (d = 64) tcgen05 kernels with K4 fix-up, K2/K11 SIMT and fused
small levels, K3/K6 CSR, K5/K7/K8/K10, K9 queries (dense + CSR, beam 1 and 3), K12 grouped
build, K13 range search, insertion, and K14 routing / routed queries / merge.  Small sizes
(sanitizers slow kernels down 10-100x)."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402
from paper_2208_02734_b200.cluster import LocalCluster  # noqa: E402


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    for cid, div in ((1, 1), (2, 128), (3, 2048)):
        cfg = datagen.CONFIGS[cid].scaled(div)
        X = datagen.data(cfg)
        idx = mk.build(t(X), cfg.levels, 3, datagen.all_init_indices(cfg))
        Q = t(datagen.queries(cfg, count=64))
        idx.query(Q, knn=10, beam=1)
        idx.query(Q, knn=5, beam=3)
        idx.range_query(Q, 2.0, "cover")
        idx.range_query(Q, 2.0, "paper")
        if cid != 1:
            idx.insert(t(datagen.queries(cfg, count=16)))
        idx.free()
        print(f"{cfg.name}/{div}: build, queries, range, insert ok", flush=True)
    rp, col, val = datagen.random_csr(5, 1500, 400, 8)
    csr = mk.Csr(t(rp), t(col), t(val), 400)
    idx = mk.build(csr, [32, 4], 3, [datagen.init_indices(5, 1, 1500, 32), datagen.init_indices(5, 2, 32, 4)])
    qrp, qcol, qval = datagen.random_csr(6, 40, 400, 8)
    idx.query(mk.Csr(t(qrp), t(qcol), t(qval), 400), knn=10, beam=2)
    idx.free()
    print("CSR build + query ok", flush=True)
    Xg = datagen.gaussian_clouds(7, 200, radius=20.0, sigma=1.0)
    g = mk.build_grouped(t(Xg), 20, 10, 5, perm=datagen.group_perm(7, Xg.shape[0]))
    g.query(t(Xg[:50]), knn=1)
    g.free()
    print("grouped build ok", flush=True)
    parts = [Xg[:700], Xg[700:]]
    inits = [[datagen.init_indices(8 + r, 1, len(p), 8), datagen.init_indices(8 + r, 2, 8, 2)] for r, p in enumerate(parts)]
    cl = LocalCluster.build([t(p) for p in parts], [8, 2], 4, inits)
    for eps in (math.inf, 5.0):
        cl.knn(t(Xg[:30]), knn=5, epsilon=eps)
    cl.free()
    torch.cuda.synchronize()
    print("SANITIZE_WORKLOAD_OK", flush=True)


if __name__ == "__main__":
    main()
