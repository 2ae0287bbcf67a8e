"""Range search timing on C2 (one build, then 10,000 queries, radius = each query's 10th-NN
distance over a sample, cover and paper modes).  python tools/range_bench.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402

cfg = datagen.CONFIGS[2]
X = torch.from_numpy(datagen.data(cfg)).cuda()
idx = mk.build(X, cfg.levels, cfg.iters, datagen.all_init_indices(cfg))
Q = torch.from_numpy(datagen.queries(cfg)).cuda()
d2 = torch.cdist(Q, X[:200000]) ** 2
r = torch.sqrt(torch.kthvalue(d2, 2, dim=1).values).float().contiguous()  # ~10th-NN radius at full size
for mode in ("cover", "paper"):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        off, ids, dd = idx.range_query(Q, r, mode)
        e1.record()
        torch.cuda.synchronize()
    n = int(off[-1])
    print(f"{mode}: {Q.shape[0]} queries, {n} results ({n / Q.shape[0]:.1f}/query) in {e0.elapsed_time(e1):.2f} ms")
