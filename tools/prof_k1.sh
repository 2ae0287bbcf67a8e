#!/bin/bash
# ncu capture of the K1 assignment kernel on a C2-shaped launch (run on the GPU box).
set -e
OUT=${1:-gpurun_out}
ARGS=${2:-"--n 1000000 --d 16 --k 4096 --reps 2 --check 0"}
python tools/kbench.py $ARGS > $OUT/kbench_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 1 -c 1 -o $OUT/prof_k1 python tools/kbench.py $ARGS > $OUT/ncu_k1.log 2>&1
