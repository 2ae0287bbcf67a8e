#!/bin/bash
# A/B of the batched query (tools/query_sweep.py) with the in-tree libmask.so and each tools/variants/*.so
cp paper_2208_02734_b200/libmask.so /tmp/base.so
echo "base:"; timeout 600 python tools/query_sweep.py $@ 2>/dev/null
for v in tools/variants/*.so; do
  cp $v paper_2208_02734_b200/libmask.so
  echo "$(basename $v):"; timeout 600 python tools/query_sweep.py $@ 2>/dev/null
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
