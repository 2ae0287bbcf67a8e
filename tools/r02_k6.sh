#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_insert.py tests/test_gpu_k3t.py -x -q -k "C4 or sparse or csr or CSR or multirank or sharded or insert or split or k3t" > gpurun_out/k6_tests.log 2>&1; echo rc=$? >> gpurun_out/k6_tests.log
timeout 900 python bench.py --config 4 --no-sweep > gpurun_out/k6_bench_c4.json 2> gpurun_out/k6_bench_c4.err
