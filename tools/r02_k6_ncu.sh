#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_update_csr_sorted" -c 1 \
  -o gpurun_out/k6_full -f python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep \
  > gpurun_out/k6_ncu.log 2>&1
echo "ncu rc=$?"
