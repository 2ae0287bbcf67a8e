mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/c2_tests.log 2>&1; echo rc=$? >> gpurun_out/c2_tests.log
timeout 900 python bench.py > gpurun_out/c2_bench_c3.json 2> gpurun_out/c2_bench_c3.err
for v in 0 1 2; do MASK_TC_D16=$v timeout 300 python bench.py --config 2 --steps 5 --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/c2_bench_c2_v$v.json 2>> gpurun_out/c2_d16.err; done
python tools/ncu_c3_k1.py > gpurun_out/ncu_c3_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 1 -c 1 -o gpurun_out/r02_k1_c3full_hint python tools/ncu_c3_k1.py > gpurun_out/ncu_c3_hint.log 2>&1
echo done
