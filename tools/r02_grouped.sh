#!/bin/bash
# query path: parity tests, then the A/B sweep on C3 (per-query vs leaf-grouped variants)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_insert.py tests/test_gpu_range.py -x -q -m gpu ${TK:+-k "$TK"} > gpurun_out/grp_tests.log 2>&1
echo "tests rc=$?"
tail -3 gpurun_out/grp_tests.log
timeout 900 python tools/query_sweep.py --config ${CFG:-3} --iters 5 --sample 200 --beams ${BEAMS:-1,2,4,8,16,32,64,128,256} --modes ${MODES:-0,1} > gpurun_out/grp_c3.jsonl 2> gpurun_out/grp_c3.err
echo "sweep rc=$?"
