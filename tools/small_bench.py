"""Time one small level (fused K11 vs per-pass kernels) through mask_build (development).

    python tools/small_bench.py [--n 4096 --d 16 --k 256 --T 25]
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
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--d", type=int, default=16)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--T", type=int, default=25)
    a = ap.parse_args()
    X = datagen.blobs(5, a.n, a.d, max(2, a.k // 4))
    inits = [datagen.init_indices(9, 1, a.n, a.k)]
    Xd = torch.from_numpy(X).cuda()
    for flags, name in [(0, "fused"), (mk.MASK_NO_FUSED, "per-pass")]:
        for r in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            idx = mk.build(Xd, [a.k], a.T, inits, flags=flags | mk.MASK_TIME_KERNELS)
            e1.record()
            torch.cuda.synchronize()
            if r == 2:
                t = idx.timing(1)
                print(f"{name:9s} build {e0.elapsed_time(e1):.3f} ms, passes {idx.level_info(1)['passes']}, "
                      f"assign {t['assign']['ms']:.3f} ms ({t['assign_kernel']})")
            idx.free()


if __name__ == "__main__":
    main()
