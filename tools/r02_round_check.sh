mkdir -p gpurun_out
MASK_DEBUG_FIXUP=1 timeout 300 python tools/dbg/near_ties2.py > gpurun_out/rc_near_ties.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=20 > gpurun_out/rc_tests.log 2>&1; echo rc=$? >> gpurun_out/rc_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/rc_bench_c3.json 2> gpurun_out/rc_bench_c3.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/rc_bench_c2.json 2> gpurun_out/rc_bench_c2.err
