#!/bin/bash
# end of session: multicast A/B for 3xFP16 at d = 64, smoke(), C3 launch list (ncu, one step)
mkdir -p gpurun_out
for v in 2 5; do echo "== hv=$v"; MASK_TC_H16V=$v timeout 300 python tools/h16_build.py 3 2e6 4 2>&1 | grep -v Warn; done > gpurun_out/fin_mc.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv \
  python bench.py --steps 1 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/fin_ncu_bench.log 2>&1; echo ncu_rc=$? >> gpurun_out/fin_ncu_bench.log
