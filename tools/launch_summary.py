"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: time share per kernel.

usage: python tools/launch_summary.py launches.csv [last_n_launches] [title]
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main():
    path = sys.argv[1]
    last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    title = sys.argv[3] if len(sys.argv) > 3 else path
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
    if last:
        data = data[-last:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        ms = float(r[iv].replace(",", "")) * SCALE[r[iu]]
        name = r[ik].split("(")[0].replace("void ", "")[:64]
        agg[name][0] += 1
        agg[name][1] += ms
        tot += ms
    print(title)
    print("ncu gpu__time_duration.sum, --clock-control none (cold-cache, serialised launches)")
    print(f"total kernel time {tot:.3f} ms over {len(data)} launches")
    for name, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        print(f"{ms:9.3f} ms {c:5d}x {100 * ms / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main()
