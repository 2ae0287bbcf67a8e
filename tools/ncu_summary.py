"""Summarise an ncu --set full report (one kernel launch) into a few lines of text."""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("smsp__cycles_active.avg", "SMSP active cycles"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (realtime, % of peak elapsed)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe (% of peak active)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (% of peak active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput (% of peak)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def traffic(path):
    """DRAM bytes (read + write) of the first kernel in a --set full report."""
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(key)
        tot += float(vals[i].replace(",", "")) * SCALE[units[i]]
    return vals[hdr.index("Kernel Name")], tot


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        print(f"kernel: {name[:140]}")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {label:52s} {vals[i]} {units[i]}")


if __name__ == "__main__":
    # usage: ncu_summary.py REPORT...   |   ncu_summary.py --traffic WORKLOAD KERNEL_CLASS REPORT OUT.json
    if sys.argv[1] == "--traffic":
        import json, os
        workload, kclass, rep, outp = sys.argv[2:6]
        name, tot = traffic(rep)
        db = json.load(open(outp)) if os.path.exists(outp) else {}
        db[workload] = {"kernel_class": kclass, "kernel": name[:120], "dram_bytes_per_launch": tot,
                        "capture": os.path.basename(rep)}
        json.dump(db, open(outp, "w"), indent=1)
        print(workload, kclass, tot)
    else:
        for p in sys.argv[1:]:
            print(f"== {p}")
            main(p)
