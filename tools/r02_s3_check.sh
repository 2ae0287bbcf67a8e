#!/bin/bash
# session-3 re-entry check: full GPU tests, default bench (C3), C4 bench, C4 kernel timings
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/s3_tests.log 2>&1; echo rc=$? >> gpurun_out/s3_tests.log
timeout 900 python bench.py > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err
timeout 600 python tools/c4bench.py 3 > gpurun_out/s3_c4bench.log 2>&1
timeout 900 python bench.py --config 4 > gpurun_out/s3_bench_c4.json 2> gpurun_out/s3_bench_c4.err
