"""C2 near-tie re-check probe: K4 time per build (CUDA events) and, for every level-1 pass of a
build, the number of rows K1 flags when the same prototypes are re-assigned (mask_assign)."""
import sys, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[2]
X = torch.from_numpy(datagen.data(cfg)).cuda()
inits = datagen.all_init_indices(cfg)
Ps = {}
def cb(l, p, P, lab):
    if l == 1: Ps[p] = P
for rep in range(3):
    idx = mk.build(X, cfg.levels, cfg.iters, inits, flags=mk.MASK_TIME_KERNELS | mk.MASK_BORROW_DATA | (mk.MASK_NO_FUSED if rep == 2 else 0))
    t = idx.timing(1); print(rep, {k: v for k, v in t.items()}); idx.free()
idx = mk.build(X, cfg.levels, cfg.iters, inits, flags=mk.MASK_BORROW_DATA, iter_cb=cb)
for p in sorted(Ps):
    lab, d2, nf = mk.assign(X, torch.from_numpy(Ps[p]).cuda())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); lab, d2, nf2 = mk.assign(X, torch.from_numpy(Ps[p]).cuda()); e1.record(); torch.cuda.synchronize()
    print(p, nf, round(e0.elapsed_time(e1), 3))
