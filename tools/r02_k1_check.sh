set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "assign or replicas or fused or edge" > gpurun_out/k1_parity.log 2>&1; echo rc=$? >> gpurun_out/k1_parity.log
timeout 300 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 3 > gpurun_out/k1_kbench.log 2>&1
MASK_TC_LEGACY=1 timeout 300 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 3 >> gpurun_out/k1_kbench.log 2>&1
timeout 300 python tools/kbench.py --n 500000 --d 128 --k 65536 --cfg 5 --reps 3 >> gpurun_out/k1_kbench.log 2>&1
MASK_TC_LEGACY=1 timeout 300 python tools/kbench.py --n 500000 --d 128 --k 65536 --cfg 5 --reps 3 >> gpurun_out/k1_kbench.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep > gpurun_out/bench_c3_p.json 2> gpurun_out/bench_c3_p.err
MASK_E2E_REPORT=gpurun_out/e2e_p.jsonl timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_multirank.py -x -q -m gpu -k "C3 or C5 or C2_div64 or sharded" > gpurun_out/k1_e2e.log 2>&1; echo rc=$? >> gpurun_out/k1_e2e.log
