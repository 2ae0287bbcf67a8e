#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_e2e.py tests/test_gpu_fullsize.py -x -q -m gpu -k "csr or CSR or C4 or farthest or sparse" > gpurun_out/k6_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/k6_tests.log
timeout 900 python bench.py --config 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
