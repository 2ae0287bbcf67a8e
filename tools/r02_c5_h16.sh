#!/bin/bash
# C5 at full size (100M x 128, 51 GB) with K1 3xFP16: clean timed build T = 15 + 1e6 queries
mkdir -p gpurun_out
timeout 1700 python tools/c5_full.py --T 15 --clean --beams 1,16 > gpurun_out/c5_full_h16.txt 2>&1; echo rc=$? >> gpurun_out/c5_full_h16.txt
