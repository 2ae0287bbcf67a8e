"""K3T vs K3 (SIMT chunk-major) on one C4-shaped assignment (n = 1e6/div, k = 8192/div): times
both through mask_assign (CUDA events) and serves as the ncu capture workload."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
div = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "both"
cfg = datagen.CONFIGS[4].scaled(div)
rp, col, val = datagen.data(cfg)
dev = "cuda:0"
csr = mk.Csr(torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev), torch.from_numpy(val).to(dev), cfg.dim)
init = datagen.init_indices(cfg.cid, 1, cfg.n, cfg.levels[0])
Y = np.zeros((len(init), cfg.dim), np.float32)
for i, r in enumerate(init):
    Y[i, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
P = torch.from_numpy(Y).to(dev)
modes = [("K3T", mk.MASK_CSR_TC), ("K3", 0)] if mode == "both" else [(mode, mk.MASK_CSR_TC if mode == "K3T" else 0)]
res = {}
for name, fl in modes:
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        lab, d2, _ = mk.assign(csr, P, flags=fl)
        e1.record(); torch.cuda.synchronize()
        print(f"{name} n={cfg.n} k={cfg.levels[0]} rep {rep}: {e0.elapsed_time(e1):.2f} ms (incl. per-call prep)", flush=True)
    res[name] = lab.cpu().numpy()
if len(res) == 2:
    print("label agreement", float((res["K3T"] == res["K3"]).mean()))
