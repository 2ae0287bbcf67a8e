#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc_persist -s 1 -c 1 -o gpurun_out/r02_k1h16b_c3full -f python tools/ncu_c3_k1.py > gpurun_out/k1h16b_ncu.log 2>&1; echo rc=$? >> gpurun_out/k1h16b_ncu.log
