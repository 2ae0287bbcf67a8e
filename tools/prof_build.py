"""Run one mask_build of a config (optionally with CUDA-event kernel timing) for ncu captures.

    python tools/prof_build.py [--cfg 2] [--iters 25] [--times]

Development tool: under `ncu -k regex:k_assign_tc -s S -c 1` it captures the S-th assignment
launch of a real Lloyd loop (later passes see the previous pass's labels).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--times", action="store_true")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--nosort", action="store_true")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    X = datagen.data(cfg, 0, a.n)
    n = X.shape[0]
    inits = [datagen.init_indices(a.cfg, 1, n, cfg.levels[0])]
    levels = [cfg.levels[0]]
    Xd = torch.from_numpy(X).cuda()
    iters = a.iters if a.iters is not None else cfg.iters
    for _ in range(a.reps):
        flags = (mk.MASK_TIME_KERNELS if a.times else 0) | (mk.MASK_NO_SORT if a.nosort else 0)
        idx = mk.build(Xd, levels, iters, inits, flags=flags)
        if a.times:
            print("timing", idx.timing(1))
        print("passes", idx.level_info(1))
        idx.free()


if __name__ == "__main__":
    main()
