"""K1 3xFP16 vs 3xTF32 inside a build (passes after the first use the label-sorted rows and the
pruning bound): level-1 assignment time per pass (MASK_TIME_KERNELS), C3 or C5 rows."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
T = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = datagen.CONFIGS[cid]
X = torch.from_numpy(datagen.data(cfg, 0, n)).cuda()
k = cfg.levels[0]
inits = [datagen.init_indices(cfg.cid, 1, n, k)]
labs = {}
for name, fl in (("tf32", mk.MASK_TC_TF32), ("h16", 0), ("tf32", mk.MASK_TC_TF32), ("h16", 0)):
    idx = mk.build(X, [k], T, inits, flags=mk.MASK_BORROW_DATA | mk.MASK_TIME_KERNELS | fl)
    tm = idx.timing(1)
    a = tm["assign"]
    print(f"C{cid} n={n} k={k} T={T} {name}: assign {a['ms']:.1f} ms / {a['launches']} = {a['ms']/max(a['launches'],1):.2f} ms/pass, "
          f"fixup {tm['fixup']['ms']:.2f} ms", flush=True)
    labs[name] = idx.labels(1) if hasattr(idx, "labels") else idx.prototypes(1)
    idx.free()
print("same level-1 prototypes:", bool(np.array_equal(labs["tf32"], labs["h16"])))
