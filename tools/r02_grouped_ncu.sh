#!/bin/bash
mkdir -p gpurun_out
for b in ${BEAMS:-8 128}; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --kernel-name regex:"k_query|k_leaf|k_pair|k_merge|k_cand|k_child|k_select" --log-file gpurun_out/grp_ncu_b$b.csv \
  python tools/query_sweep.py --config 3 --iters 2 --sample 10 --beams $b --modes auto > gpurun_out/grp_ncu_b$b.log 2>&1
echo "ncu b$b rc=$?"
done
