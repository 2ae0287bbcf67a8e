#!/bin/bash
mkdir -p gpurun_out
MASK_QUERY_GROUPED=${G:-0} timeout 900 ncu --set full --import-source on --clock-control none \
  --kernel-name regex:"${K:-k_query_dense_wide}" -c ${C:-1} -o gpurun_out/grp_full -f \
  python tools/query_sweep.py --config 3 --iters 2 --sample 10 --beams ${B:-128} --modes ${G:-0} > gpurun_out/grp_full.log 2>&1
echo "ncu rc=$?"
