#!/bin/bash
# A/B of compile-time K1 variants (tools/variants/*.so) on the 3xFP16 C3-rows build timing
mkdir -p gpurun_out
cp paper_2208_02734_b200/libmask.so /tmp/base.so
{ for rep in 1 2; do
  echo "== base"; timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -E " h16:"
  for v in tools/variants/*.so; do
    cp $v paper_2208_02734_b200/libmask.so
    echo "== $(basename $v)"; timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -E " h16:|same"
    cp /tmp/base.so paper_2208_02734_b200/libmask.so
  done
done; } > gpurun_out/ab_h16.log 2>&1
