mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err
timeout 600 python bench.py --config 2 --steps 5 > gpurun_out/final_bench_c2.json 2> gpurun_out/final_bench_c2.err
timeout 900 python bench.py --config 4 --steps 3 > gpurun_out/final_bench_c4.json 2> gpurun_out/final_bench_c4.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python tools/ncu_c3_k1.py > gpurun_out/ncu_c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 1 -c 1 -o gpurun_out/r02_k1_c3full python tools/ncu_c3_k1.py > gpurun_out/ncu_c3.log 2>&1
python bench.py --steps 1 --warmup 1 --no-e2e --no-sweep --no-cpu-baseline > gpurun_out/ll_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-sweep --no-cpu-baseline > gpurun_out/ll_ncu.log 2>&1
echo done
