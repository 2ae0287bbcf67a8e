#!/bin/bash
# 3xFP16 default: full GPU suite, default bench (C3), ncu --set full of K1 (3xFP16) at C3 full size
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/hf_tests.log 2>&1; echo rc=$? >> gpurun_out/hf_tests.log
timeout 900 python bench.py > gpurun_out/hf_bench_c3.json 2> gpurun_out/hf_bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 1 -c 1 -o gpurun_out/r02_k1h16_c3full -f python tools/ncu_c3_k1.py > gpurun_out/hf_ncu.log 2>&1
