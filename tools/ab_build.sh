#!/bin/bash
# A/B on the GPU box: per-kernel CUDA-event times of one level-1 build (tools/prof_build.py)
# with the in-tree libmask.so and each tools/variants/*.so
ARGS=${1:-"--cfg 2 --times --reps 3"}
cp paper_2208_02734_b200/libmask.so /tmp/base.so
echo "base: "; timeout 300 python tools/prof_build.py $ARGS 2>&1 | grep -E "timing|passes" | tail -2
for v in tools/variants/*.so; do
  cp $v paper_2208_02734_b200/libmask.so
  echo "$(basename $v): "; timeout 300 python tools/prof_build.py $ARGS 2>&1 | grep -E "timing|passes" | tail -2
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
