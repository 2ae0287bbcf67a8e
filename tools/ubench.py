"""Update-kernel timing: level-1 'update' class time of a T=3 build (CUDA events in libmask)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cid, n = int(sys.argv[1]), int(sys.argv[2])
cfg = datagen.CONFIGS[cid]
X = datagen.data(cfg, 0, n)
k = cfg.levels[0] if n == cfg.n else max(2, cfg.levels[0] * n // cfg.n)
Xd = torch.from_numpy(X).to("cuda:0")
for rep in range(2):
    idx = mk.build(Xd, [k], 3, [datagen.init_indices(cid, 1, n, k)], flags=mk.MASK_TIME_KERNELS | mk.MASK_BORROW_DATA)
    tm = idx.timing(1)["update"]
    ms = tm["ms"] / max(tm["launches"], 1)
    byts = n * cfg.dim * 4 + n * 4 + k * (cfg.dim + 1) * 4
    print(f"{os.environ.get('MASK_UPDATE','sorted')} C{cid} n={n} d={cfg.dim} k={k}: update {ms*1000:.1f} us "
          f"-> {byts / ms / 1e6:.0f} GB/s = {byts / ms / 1e6 / 6541.5:.2f} of HBM", flush=True)
    idx.free()
