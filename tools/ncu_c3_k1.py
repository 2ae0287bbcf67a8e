"""One C3 level-1 build with T = 1 (two K1 passes, the second with the pruning bound of the
first) -- the workload for the round's `ncu --set full` capture of K1 at the bench size:

    python tools/ncu_c3_k1.py && \\
    ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 1 -c 1 \\
        -o gpurun_out/r02_k1_c3full python tools/ncu_c3_k1.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402

cfg = datagen.CONFIGS[3]
Xh, shm = datagen.data_parallel(cfg)
X = torch.from_numpy(Xh).cuda()
inits = datagen.all_init_indices(cfg)
idx = mk.build(X, cfg.levels[:1], 1, inits[:1], flags=mk.MASK_BORROW_DATA)
print("passes", idx.level_info(1)["passes"])
idx.free()
del X, Xh
shm.close()
shm.unlink()
