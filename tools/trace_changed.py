"""Per-pass changed-label counts of the C2 level-1 Lloyd loop (mask_get_trace)."""
import sys, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[2]
X = torch.from_numpy(datagen.data(cfg)).cuda()
idx = mk.build(X, cfg.levels, cfg.iters, datagen.all_init_indices(cfg), flags=mk.MASK_BORROW_DATA)
print(idx.trace(1)["changed"].tolist())
