#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 2 3 4; do echo "== hv=$v"; MASK_TC_H16=1 MASK_TC_H16V=$v timeout 300 python tools/h16_check.py 3 1e6 2>&1 | grep -v Warn; done > gpurun_out/h16v_c3.log
for v in 0 1; do echo "== hv=$v"; MASK_TC_H16=1 MASK_TC_H16V=$v timeout 300 python tools/h16_check.py 5 1e6 2>&1 | grep -v Warn; done > gpurun_out/h16v_c5.log
