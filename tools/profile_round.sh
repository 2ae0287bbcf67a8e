#!/bin/bash
# Round evidence on the GPU box: bench line, ncu launch list of the bench command (one timed
# step; the per-step slice is the last launches), ncu --set full captures of the dominant kernels.
#   bash tools/profile_round.sh r01
set -x
R=${1:-r01}
O=gpurun_out
python bench.py --steps 5 > $O/${R}_bench_c2.json 2> $O/${R}_bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_bench_c2_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/${R}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 20 -c 1 \
  -o $O/${R}_k1_c2 python tools/prof_build.py --cfg 2 --iters 25 > $O/${R}_ncu_k1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_update_runs -s 10 -c 1 \
  -o $O/${R}_k5_c2 python tools/prof_build.py --cfg 2 --iters 25 > $O/${R}_ncu_k5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 1 -c 1 \
  -o $O/${R}_k1_c3 python tools/prof_build.py --cfg 3 --n 1000000 --iters 1 > $O/${R}_ncu_k1c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_csr_chunked -s 1 -c 1 \
  -o $O/${R}_k3_c4 python tools/c4bench.py 1 > $O/${R}_ncu_k3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_update_csr_sorted -s 1 -c 1 \
  -o $O/${R}_k6_c4 python tools/c4bench.py 1 > $O/${R}_ncu_k6.log 2>&1
ls -la $O/${R}_*
