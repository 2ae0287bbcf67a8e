mkdir -p gpurun_out
for v in 0 3 1 4; do echo "d16 variant $v" >> gpurun_out/mc.log; MASK_TC_D16=$v timeout 300 python tools/kbench.py --n 1000000 --d 16 --k 4096 --cfg 2 --reps 5 --check 1000 >> gpurun_out/mc.log 2>&1; done
for v in 0 3; do echo "d64 variant $v" >> gpurun_out/mc.log; MASK_TC_D64=$v timeout 300 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 3 --check 500 >> gpurun_out/mc.log 2>&1; done
MASK_TC_D16=3 MASK_TC_D64=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "assign or near_ties or replicas" > gpurun_out/mc_tests.log 2>&1; echo rc=$? >> gpurun_out/mc_tests.log
for v in 3 4; do MASK_TC_D16=$v timeout 300 python bench.py --config 2 --steps 5 --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/mc_bench_c2_v$v.json 2>> gpurun_out/mc.err; done
timeout 900 python bench.py --no-e2e --no-sweep --no-cpu-baseline > gpurun_out/mc_bench_c3.json 2>> gpurun_out/mc.err
