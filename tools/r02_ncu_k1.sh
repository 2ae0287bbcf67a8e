mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_insert.py tests/test_gpu_parity.py -x -q -m gpu -k "insert or split or near_ties or assign" > gpurun_out/nk_tests.log 2>&1; echo rc=$? >> gpurun_out/nk_tests.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/nk_bench_c2.json 2> gpurun_out/nk_bench_c2.err
python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 1 --check 0 > gpurun_out/nk_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -c 1 -o gpurun_out/r02_k1_c3 python tools/kbench.py --n 1000000 --d 64 --k 65536 --cfg 3 --reps 1 --check 0 > gpurun_out/nk_ncu.log 2>&1
echo ncu_rc=$?
