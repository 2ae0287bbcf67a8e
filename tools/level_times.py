"""Per-level kernel-class device times of a full C2-style build vs its wall time (development).

    python tools/level_times.py [--cfg 2] [--reps 3]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.cfg]
    X = datagen.data(cfg)
    inits = datagen.all_init_indices(cfg)
    Xd = torch.from_numpy(X).cuda()
    for r in range(a.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = mk.build(Xd, cfg.levels, cfg.iters, inits, flags=mk.MASK_TIME_KERNELS)
        e1.record()
        torch.cuda.synchronize()
        print(f"rep {r}: build {e0.elapsed_time(e1):.2f} ms, launches so far {mk.kernel_launches()}")
        for l in range(1, len(cfg.levels) + 1):
            t = idx.timing(l)
            info = idx.level_info(l)
            tot = sum(v["ms"] for k, v in t.items() if isinstance(v, dict))
            print(f"  level {l} n={info['n_items']} k={info['k']} passes={info['passes']}: kernels {tot:.2f} ms "
                  + " ".join(f"{k}={v['ms']:.2f}/{v['launches']}" for k, v in t.items() if isinstance(v, dict)))
        idx.free()


if __name__ == "__main__":
    main()
