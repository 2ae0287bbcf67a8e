mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "wide_beam or query or update or replicas" > gpurun_out/bk_tests.log 2>&1; echo rc=$? >> gpurun_out/bk_tests.log
timeout 900 python bench.py > gpurun_out/bk_bench_c3.json 2> gpurun_out/bk_bench_c3.err
timeout 600 python bench.py --config 2 --steps 5 > gpurun_out/bk_bench_c2.json 2> gpurun_out/bk_bench_c2.err
