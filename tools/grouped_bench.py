"""The paper's §5.2 parameter sweep on the grouped construction (Algorithm 1, NEXT-1): 8
Gaussian clouds x 10,000 points in R^2, lengthGroup/nCentroids 10/5 ... 110/55 (ratio 2:1):
tree depth, build time, exhaustive point-search time over all 80,000 points (batched k=1
queries), the self-query miss rate (the point itself not returned, G7) and the
wrong-cloud rate (the returned point belongs to another cloud).  Device timings with
CUDA events (one warm-up run first).  Context: the paper's CPU cluster took ~300-340 s to
build and ~2,500-2,900 s to search.

    python tools/grouped_bench.py [--radius 12 --sigma 2] [--T 20]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--radius", type=float, default=12.0)
    ap.add_argument("--sigma", type=float, default=2.0)
    ap.add_argument("--T", type=int, default=20)
    a = ap.parse_args()
    X = datagen.gaussian_clouds(21, 10_000, a.radius, a.sigma)
    perm = datagen.group_perm(22, X.shape[0])
    Xd = torch.from_numpy(X).cuda()
    print(f"80,000 points, 8 clouds (radius {a.radius}, sigma {a.sigma}), T={a.T}")
    cloud = np.repeat(np.arange(8), 10_000)  # generator order: cloud c holds rows [10^4 c, 10^4 (c+1))
    print("lengthGroup nCentroids depth  build_ms  search_ms  self_miss_%  wrong_cloud_%")
    for lg in (10, 30, 50, 70, 90, 110):
        nc = lg // 2
        for rep in range(2):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            e0.record()
            idx = mk.build_grouped(Xd, lg, nc, a.T, perm)
            e1.record()
            ids, _ = idx.query(Xd, knn=1)
            e2.record()
            torch.cuda.synchronize()
            if rep == 1:
                top = ids[:, 0].cpu().numpy()
                err = float((top != np.arange(X.shape[0])).mean()) * 100
                wrong = float((cloud[top] != cloud).mean()) * 100
                print(f"{lg:11d} {nc:10d} {idx.num_levels:5d} {e0.elapsed_time(e1):9.2f} {e1.elapsed_time(e2):10.2f} "
                      f"{err:12.3f} {wrong:14.3f}")
            idx.free()


if __name__ == "__main__":
    main()
