#!/bin/bash
# session 3 final: full GPU suite, default bench (C3), C2 and C4 bench lines, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/sf_tests.log 2>&1; echo rc=$? >> gpurun_out/sf_tests.log
timeout 900 python bench.py > gpurun_out/sf_bench_c3.json 2> gpurun_out/sf_bench_c3.err
timeout 600 python bench.py --config 2 > gpurun_out/sf_bench_c2.json 2> gpurun_out/sf_bench_c2.err
timeout 900 python bench.py --config 4 > gpurun_out/sf_bench_c4.json 2> gpurun_out/sf_bench_c4.err
