#!/bin/bash
mkdir -p gpurun_out
for v in 2 6 7 2 6 7; do echo "== hv=$v"; MASK_TC_H16V=$v timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -v Warn | grep -E "h16|same"; done > gpurun_out/h16acc.log 2>&1
