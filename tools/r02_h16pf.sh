#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -v Warn > gpurun_out/pf_build_c3.log
timeout 300 python tools/h16_build.py 5 1e6 3 2>&1 | grep -v Warn > gpurun_out/pf_build_c5.log
timeout 900 python -m pytest tests/test_gpu_h16.py tests/test_gpu_e2e.py tests/test_gpu_parity.py -x -q > gpurun_out/pf_tests.log 2>&1; echo rc=$? >> gpurun_out/pf_tests.log
