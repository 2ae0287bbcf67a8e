mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_comm.py -x -q -m gpu > gpurun_out/k4_parity.log 2>&1; echo rc=$? >> gpurun_out/k4_parity.log
MASK_E2E_REPORT=gpurun_out/e2e_k4.jsonl timeout 1200 python -m pytest tests/test_gpu_e2e.py -x -q -m gpu > gpurun_out/k4_e2e.log 2>&1; echo rc=$? >> gpurun_out/k4_e2e.log
timeout 300 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 3 > gpurun_out/k4_kbench.log 2>&1
timeout 300 python tools/kbench.py --n 500000 --d 128 --k 65536 --cfg 5 --reps 3 >> gpurun_out/k4_kbench.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep > gpurun_out/bench_c3_k4.json 2> gpurun_out/bench_c3_k4.err
