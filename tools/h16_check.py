"""K1 3xFP16 (MASK_TC_H16=1) vs 3xTF32 (MASK_TC_TF32 flag) on one C3/C5-shaped assignment:
labels must agree exactly (both are exact after the K4 near-tie decision), times via CUDA events."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
cfg = datagen.CONFIGS[cid]
X = torch.from_numpy(datagen.data(cfg, 0, n)).cuda()
k = cfg.levels[0]
init = datagen.init_indices(cfg.cid, 1, n, k)
P = X[torch.from_numpy(init).cuda().long()].clone()
res = {}
for name, fl in (("tf32", mk.MASK_TC_TF32), ("h16", 0), ("tf32b", mk.MASK_TC_TF32), ("h16b", 0)):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    lab, d2, nf = mk.assign(X, P, flags=fl)
    e1.record(); torch.cuda.synchronize()
    res[name] = (lab.cpu().numpy(), d2.cpu().numpy())
    print(f"C{cid} n={n} d={cfg.dim} k={k} {name}: {e0.elapsed_time(e1):.2f} ms flagged={nf}", flush=True)
a, b = res["tf32b"], res["h16b"]
print("label agreement", float((a[0] == b[0]).mean()), "max |d2 diff|", float(np.abs(a[1] - b[1]).max()))
