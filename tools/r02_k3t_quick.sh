#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k3t.py -x -q > gpurun_out/k3t_tests.log 2>&1; echo rc=$? >> gpurun_out/k3t_tests.log
timeout 300 python tools/k3t_ncu.py 4 > gpurun_out/k3t_time.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assign_csr_tc -s 1 -c 1 -o gpurun_out/k3t_full -f python tools/k3t_ncu.py 4 K3T > gpurun_out/k3t_ncu.log 2>&1
