#!/bin/bash
mkdir -p gpurun_out
for v in 0 2 4; do echo "== hv=$v"; MASK_TC_H16=1 MASK_TC_H16V=$v timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -v Warn; done > gpurun_out/h16b_c3.log
echo "== hv=0"; MASK_TC_H16=1 timeout 300 python tools/h16_build.py 5 1e6 3 2>&1 | grep -v Warn > gpurun_out/h16b_c5.log
