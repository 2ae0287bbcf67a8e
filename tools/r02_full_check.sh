mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/fc_tests.log 2>&1; echo rc=$? >> gpurun_out/fc_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29633 bench.py --force-comm --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/fc2_bench_c3.json 2> gpurun_out/fc2_bench_c3.err; echo "torchrun rc=$?" >> gpurun_out/fc2_bench_c3.err
timeout 900 python bench.py > gpurun_out/fc_bench_default.json 2> gpurun_out/fc_bench_default.err
