"""The bench.py contract pieces that run without a GPU: the reference arm (the FP64 oracle on
the host cores) prints one JSON line with the contract's keys, and the C4 (CSR) helpers slice
rows consistently."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "C1"


def test_csr_row_slices():
    sys.path.insert(0, ROOT)
    import bench
    import datagen
    rp, col, val = datagen.random_csr(3, 50, 40, 5)
    a, b, c = bench._csr_rows((rp, col, val), 10, 20)
    assert a[0] == 0 and a.size == 11 and b.size == a[-1] == rp[20] - rp[10]
    np.testing.assert_array_equal(b, col[rp[10]:rp[20]])
    dense = bench._densify((a, b, c), 40)
    for i in range(10):
        row = np.zeros(40)
        row[col[rp[10 + i]:rp[11 + i]]] = val[rp[10 + i]:rp[11 + i]]
        np.testing.assert_array_equal(dense[i], row)
