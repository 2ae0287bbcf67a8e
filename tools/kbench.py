"""Kernel-level micro benchmark of the assignment kernels through the C-ABI (mask_assign).

    python tools/kbench.py [--n 1000000 --d 16 --k 4096] [--simt] [--check 2000]

Reports device time (CUDA events on the launching stream, L2 flushed between launches),
useful TFLOP/s (2nkd) and 3xTF32 tensor TFLOP/s (6nkd), flagged rows, and parity of a row
sample against the FP64 oracle.  Development tool, not the bench contract.
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
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--d", type=int, default=16)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--cfg", type=int, default=0, help="use config generator (2,3,5) instead of blobs")
    ap.add_argument("--simt", action="store_true")
    ap.add_argument("--nofix", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", type=int, default=2000)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    if a.cfg:
        cfg = datagen.CONFIGS[a.cfg]
        X = datagen.data(cfg, 0, a.n)
        a.d = cfg.dim
    else:
        X = datagen.blobs(1, a.n, a.d, max(2, a.k // 16))
    P = X[datagen.init_indices(77, 1, a.n, a.k)] + datagen.random_dense(3, a.k, a.d, scale=0.05)
    Xd = torch.from_numpy(X).to(dev)
    Pd = torch.from_numpy(P).to(dev)
    flags = (mk.MASK_FORCE_SIMT if a.simt else 0) | (mk.MASK_NO_FIXUP if a.nofix else 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    lab, d2, nf = mk.assign(Xd, Pd, flags=flags)
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lab, d2, nf = mk.assign(Xd, Pd, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = min(times)
    useful = 2.0 * a.n * a.k * a.d
    # kernel-only time of the assignment launch (CUDA events inside the library, T = 0 build)
    kt = []
    for _ in range(a.reps):
        flush.zero_()
        idx = mk.build(Xd, [a.k], 0, [datagen.init_indices(77, 1, a.n, a.k)],
                       flags=mk.MASK_TIME_KERNELS | mk.MASK_BORROW_DATA | flags)
        tm = idx.timing(1)
        kt.append((tm["assign"]["ms"], tm["fixup"]["ms"], tm["assign_kernel"]))
        idx.free()
    k_ms, f_ms, kname = min(kt)
    print(f"[{kname}] kernel_ms={k_ms:.3f} fixup_ms={f_ms:.3f} useful_TF={useful / k_ms / 1e9:.1f} "
          f"tensor3x_TF={3 * useful / k_ms / 1e9:.1f} frac_of_808={3 * useful / k_ms / 1e9 / 808.1:.3f}")
    print(f"n={a.n} d={a.d} k={a.k} simt={a.simt} call_ms={ms:.3f} (includes prep/fixup/alloc) "
          f"useful_TF={useful / ms / 1e9:.1f} tensor3x_TF={3 * useful / ms / 1e9:.1f} flagged={nf} "
          f"({100.0 * nf / a.n:.3f}%)")
    if a.check:
        import oracle
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        from parity import check_assignment
        m = min(a.check, a.n)
        rows = np.random.default_rng(0).choice(a.n, m, replace=False)
        labs = lab.cpu().numpy()[rows]
        nd, ne = check_assignment(X[rows], P, labs, d2.cpu().numpy()[rows], what="kbench sample")
        print(f"parity sample {m} rows: ok, label diffs {nd} (all exempt), exempt rows {ne}")


if __name__ == "__main__":
    main()
