#!/bin/bash
# A/B: run kbench ARGS with the in-tree libmask.so and each tools/variants/*.so (GPU box)
ARGS=${1:-"--n 1000000 --d 16 --k 4096 --cfg 2 --check 0 --reps 3"}
cp paper_2208_02734_b200/libmask.so /tmp/base.so
echo -n "base: "; timeout 200 python tools/kbench.py $ARGS 2>&1 | grep kernel_ms
for v in tools/variants/*.so; do
  cp $v paper_2208_02734_b200/libmask.so
  echo -n "$(basename $v): "; timeout 200 python tools/kbench.py $ARGS 2>&1 | grep kernel_ms
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
