#!/bin/bash
# C5/8 (12.5M x 128) query pipeline at beams 16 / 32: kernel times of the grouped path
mkdir -p gpurun_out
cat > /tmp/c5q.py <<'PY'
import os, sys, time, dataclasses
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, datagen, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[5].scaled(8)
cfg = dataclasses.replace(cfg, n_queries=1_000_000)
X = torch.from_numpy(datagen.data(cfg)).cuda()
idx = mk.build(X, cfg.levels, 2, datagen.all_init_indices(cfg), flags=mk.MASK_BORROW_DATA)
Q = torch.from_numpy(datagen.queries(cfg)).cuda()
for b in [int(x) for x in sys.argv[1].split(",")]:
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.time()
        idx.query(Q, knn=10, beam=b); torch.cuda.synchronize()
        print(f"beam {b}: {1e3 * (time.time() - t0):.1f} ms", flush=True)
PY
MASK_DEBUG_QUERY=1 timeout 900 python /tmp/c5q.py 16,32,64 > gpurun_out/c5q.log 2>&1; echo "plain rc=$?"; cat gpurun_out/c5q.log; nvidia-smi --query-gpu=memory.total,memory.used --format=csv; exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --kernel-name regex:"k_query|k_leaf|k_pair|k_merge|k_cand|k_child|k_select" --log-file gpurun_out/c5q_ncu.csv \
  python /tmp/c5q.py 32 > gpurun_out/c5q_ncu.log 2>&1
echo "ncu rc=$?"
