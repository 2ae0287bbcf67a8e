#!/bin/bash
mkdir -p gpurun_out
for v in 0 2 3 4; do echo "== hv=$v"; MASK_TC_H16V=$v timeout 300 python tools/h16_build.py 5 1e6 3 2>&1 | grep -v Warn; done > gpurun_out/h16v128.log
