"""C4 (sparse) build timing on the GPU: kernel times of the level-1 sparse assignment/update."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[4]
t0 = time.time(); rp, col, val = datagen.data(cfg); print("gen s", time.time() - t0, flush=True)
inits = datagen.all_init_indices(cfg)
dev = "cuda:0"
csr = mk.Csr(torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev), torch.from_numpy(val).to(dev), cfg.dim)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 3
XF = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # extra build flags (e.g. MASK_CSR_TC = 2048)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    idx = mk.build(csr, cfg.levels, T, inits, flags=mk.MASK_BORROW_DATA | mk.MASK_TIME_KERNELS | XF)
    torch.cuda.synchronize(); dt = time.time() - t0
    info = idx.level_info(1); tm = idx.timing(1); tm2 = idx.timing(2)
    print(f"build {dt*1000:.1f} ms passes={info['passes']} L1 {tm} L2 {tm2}", flush=True)
    idx.free()
