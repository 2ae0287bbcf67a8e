#!/bin/bash
# session 3, final code: full GPU suite, smoke, bench C3 (default) / C2 / C4, C3 launch list
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/sg_tests.log 2>&1; echo rc=$? >> gpurun_out/sg_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/sg_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/sg_bench_c3.json 2> gpurun_out/sg_bench_c3.err
timeout 600 python bench.py --config 2 > gpurun_out/sg_bench_c2.json 2> gpurun_out/sg_bench_c2.err
timeout 900 python bench.py --config 4 > gpurun_out/sg_bench_c4.json 2> gpurun_out/sg_bench_c4.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sg_launches_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/sg_ncu_bench.log 2>&1; echo ncu_rc=$? >> gpurun_out/sg_ncu_bench.log
