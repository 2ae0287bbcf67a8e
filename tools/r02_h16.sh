#!/bin/bash
mkdir -p gpurun_out
MASK_TC_H16=1 timeout 300 python tools/h16_check.py 3 1e6 > gpurun_out/h16_c3.log 2>&1
MASK_TC_H16=1 timeout 300 python tools/h16_check.py 5 1e6 > gpurun_out/h16_c5.log 2>&1
MASK_TC_H16=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_e2e.py -x -q > gpurun_out/h16_tests.log 2>&1; echo rc=$? >> gpurun_out/h16_tests.log
