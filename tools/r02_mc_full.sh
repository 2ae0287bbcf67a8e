#!/bin/bash
# C3 full size: K1 3xFP16 default tiling vs the 2-CTA multicast variant, same box, back to back
mkdir -p gpurun_out
for v in 2 5 2 5; do MASK_TC_H16V=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('hv=$v', round(d['ms_per_step'],1), round(r['avg_launch_ms'],2), round(r['frac'],3), d['clocks']['sm_mhz'])"; done > gpurun_out/mc_full.log 2>&1
