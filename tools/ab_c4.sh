#!/bin/bash
# A/B of the C4 (sparse) level-1 kernel times: in-tree libmask.so vs each tools/variants/*.so
cp paper_2208_02734_b200/libmask.so /tmp/base.so
echo "base: $(timeout 300 python tools/c4bench.py ${1:-3} 2>&1 | tail -1 | cut -c1-260)"
for v in tools/variants/*.so; do
  cp $v paper_2208_02734_b200/libmask.so
  echo "$(basename $v): $(timeout 300 python tools/c4bench.py ${1:-3} 2>&1 | tail -1 | cut -c1-260)"
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
