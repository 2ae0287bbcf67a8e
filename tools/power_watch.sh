#!/bin/bash
# Sample SM clock, power and throttle reasons every 20 ms while running a command (GPU box).
#   bash tools/power_watch.sh <command...>
OUT=${POWER_OUT:-/tmp/power.csv}
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,temperature.gpu --format=csv,noheader -lms 20 > $OUT &
P=$!
"$@"
kill $P
python - "$OUT" <<'PY'
import sys, statistics
rows = [l.strip().split(", ") for l in open(sys.argv[1]) if l.strip()]
busy = [r for r in rows if float(r[2].split()[0]) > 300]
print(f"samples {len(rows)}, busy(>300W) {len(busy)}")
if busy:
    clk = [float(r[1].split()[0]) for r in busy]; pw = [float(r[2].split()[0]) for r in busy]
    print(f"busy: sm clock median {statistics.median(clk):.0f} MHz (min {min(clk):.0f}), power median {statistics.median(pw):.0f} W (max {max(pw):.0f})")
    from collections import Counter
    print("reasons", Counter((r[3], r[4], r[5]) for r in busy).most_common(4))
PY
