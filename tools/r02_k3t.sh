#!/bin/bash
# K3T: parity tests, then C4 full-size level-1 timings K3T vs the SIMT chunk-major K3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k3t.py -x -q > gpurun_out/k3t_tests.log 2>&1; echo rc=$? >> gpurun_out/k3t_tests.log
timeout 600 python tools/c4bench.py 2 2048 > gpurun_out/k3t_c4.log 2>&1
timeout 600 python tools/c4bench.py 2 > gpurun_out/k3t_c4_simt.log 2>&1
