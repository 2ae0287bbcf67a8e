mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --force-comm --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/fc_bench_c3.json 2> gpurun_out/fc_bench_c3.err
timeout 1500 python tools/c5_full.py --T 15 --clean --beams 1,4,16 > gpurun_out/c5_full_r02.txt 2>&1
