#!/bin/bash
# A/B of the fused small levels: C1 bench step and C2 upper-level K11 times, in-tree vs variants
cp paper_2208_02734_b200/libmask.so /tmp/base.so
for v in base tools/variants/*.so; do
  [ "$v" != base ] && cp $v paper_2208_02734_b200/libmask.so
  echo "$v: C1 $(timeout 300 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["avg_launch_ms"],4))') C2 upper $(timeout 300 python tools/small_levels_time.py)"
done
cp /tmp/base.so paper_2208_02734_b200/libmask.so
