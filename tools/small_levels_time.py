"""C2 upper levels (K11 fused small levels): CUDA-event time of the fused launch per level."""
import os, sys, statistics
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[2]
X = torch.from_numpy(datagen.data(cfg)).cuda()
inits = datagen.all_init_indices(cfg)
res = {2: [], 3: []}
for rep in range(6):
    idx = mk.build(X, cfg.levels, cfg.iters, inits, flags=mk.MASK_TIME_KERNELS | mk.MASK_BORROW_DATA)
    for lv in (2, 3):
        t = idx.timing(lv)
        assert t["assign_kernel"] == "K11-fused-small-level", t
        res[lv].append(t["assign"]["ms"])
    idx.free()
print({lv: round(statistics.median(v[1:]), 4) for lv, v in res.items()})
