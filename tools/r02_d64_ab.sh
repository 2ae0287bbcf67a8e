mkdir -p gpurun_out
for v in 0 1 2 0; do
  echo "variant $v" >> gpurun_out/ab_d64.log
  MASK_TC_D64=$v timeout 300 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 3 --check 500 >> gpurun_out/ab_d64.log 2>&1
done
for v in 1 2; do
  MASK_TC_D64=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline --no-e2e > gpurun_out/ab_d64_bench_$v.json 2>> gpurun_out/ab_d64.log
done
timeout 900 python -m pytest tests/test_gpu_insert.py -x -q -m gpu > gpurun_out/ab_insert.log 2>&1; echo rc=$? >> gpurun_out/ab_insert.log
