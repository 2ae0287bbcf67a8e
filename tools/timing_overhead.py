"""Cost of MASK_TIME_KERNELS (per-kernel-class CUDA events inside the library) on a C2 build:
device time of mask_build with and without it (CUDA events around the call, interleaved)."""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[2]
X = torch.from_numpy(datagen.data(cfg)).cuda()
inits = datagen.all_init_indices(cfg)
flush = torch.empty(128 << 20, dtype=torch.float32, device="cuda")
res = {0: [], 1: []}
for rep in range(12):
    for tk in (0, 1):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        idx = mk.build(X, cfg.levels, cfg.iters, inits, flags=mk.MASK_BORROW_DATA | (mk.MASK_TIME_KERNELS if tk else 0))
        e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            res[tk].append(e0.elapsed_time(e1))
        idx.free()
print({("timed" if k else "plain"): round(statistics.mean(v), 3) for k, v in res.items()})
