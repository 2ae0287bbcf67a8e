#!/usr/bin/env python
"""Benchmark of the MASK hot path on B200: one step = one full multilevel index build
(all levels, T Lloyd iterations + final assignment per level) + one batched k-NN query
over the config's query set, on seeded synthetic data resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl mask|reference]

N > 1 is launched with torch.distributed.run (one rank per GPU, NCCL): the config's rows are
sharded (strong scaling: rank r owns rows shard.row_range(n, N, r) of the same block-seeded
generator, so every N builds the identical index) and mask_build combines each Lloyd
iteration's partial sums, counts and statistics with ONE NCCL allreduce; the query batch is
sharded by rank.  Default workload: C3 (BASELINE configs[2], listed at 1/2/4/8 GPUs).

Prints ONE JSON line on rank 0 (contract in DESIGN.md "Measurement").  Metric: Lloyd
point·prototype distances/s = (sum over levels and assignment passes of n_items * k_l)
/ step time; the step time includes the query batch.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "Lloyd point·prototype distances/s"
UNIT = "distances/s"
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="mask", choices=["mask", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-simt", action="store_true")
    ap.add_argument("--beam", type=int, default=1, help="prototypes kept per level in the query (1 = Algorithm 2)")
    ap.add_argument("--knn", type=int, default=None, help="neighbours per query (default: the config's)")
    ap.add_argument("--iters", type=int, default=None, help="Lloyd iterations T (default: the config's)")
    ap.add_argument("--force-comm", action="store_true",
                    help="build through an NCCL communicator even on one rank (exercises the multi-GPU path)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the QPS@recall beam sweep")
    ap.add_argument("--seed", type=int, default=0, help="data / query / init streams (0 = the documented ones)")
    ap.add_argument("--tol", type=float, default=0.0, help="Lloyd tolerance stop on max displacement (D3; 0 = off)")
    ap.add_argument("--empty", default="keep", choices=["keep", "farthest"],
                    help="empty-cluster policy (D5 keep / D5b farthest, single GPU)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def wait_rows(self, n, timeout):
        """Block until ``n`` samples exist (nvidia-smi needs ~0.1-0.5 s to start): short timed
        regions (C1: a few ms) are then bracketed by a sample right before and right after."""
        t0 = time.time()
        while self.proc and len(self.rows) < n and time.time() - t0 < timeout:
            time.sleep(0.01)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        smax = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- helpers
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return {"hbm_gbs": p.get("hbm_gbs", 6650.0), "bf16_tflops": p.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": p.get("bf16_tflops_sustained", 1400.0),
                "sm_max_mhz": p.get("sm_max_mhz", 1965.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
            "source": "fallback"}


def ncu_traffic(workload, kernel):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_traffic.json, written by tools/ncu_summary.py --traffic),
    or None when no capture of this workload / kernel class is recorded."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        rec = json.load(open(path)).get(workload)
    except (OSError, ValueError):
        return None
    if not rec or not kernel.startswith(rec.get("kernel_class", "")):
        return None
    return rec["dram_bytes_per_launch"]


def _csr_rows(trip, lo, hi):
    rp, col, val = trip
    return (rp[lo:hi + 1] - rp[lo], col[rp[lo]:rp[hi]], val[rp[lo]:rp[hi]])


def _nbytes(a):
    return sum(x.nbytes for x in a) if isinstance(a, tuple) else a.nbytes


def _densify(trip, dim):
    rp, col, val = trip
    Y = np.zeros((rp.size - 1, dim))
    for i in range(rp.size - 1):
        Y[i, col[rp[i]:rp[i + 1]]] = val[rp[i]:rp[i + 1]]
    return Y


def _oracle_pass(cfg, X_all, rows, P):
    """One FP64 oracle Lloyd pass (assignment + update) over the first ``rows`` rows of X_all."""
    import oracle

    if cfg.sparse:
        Y = _csr_rows(X_all, 0, rows)
        lab, _, _ = oracle.assign_csr(Y, cfg.dim, P)
        S, cnt = oracle.cluster_sums_csr(Y, cfg.dim, lab, P.shape[0])
        oracle.means_from_sums(S, cnt, P)
        return
    Y = X_all[:rows].astype(np.float64)
    lab, _, _ = oracle.assign(Y, P)
    oracle.means(Y, lab, P)


def _init_protos(cfg, X_all, init):
    if cfg.sparse:
        return np.stack([_densify(_csr_rows(X_all, int(i), int(i) + 1), cfg.dim)[0] for i in init])
    return X_all[init].astype(np.float64)


def lloyd_distances(idx, n_levels):
    tot = 0
    per = []
    for l in range(1, n_levels + 1):
        info = idx.level_info(l)
        dist = info["passes"] * info["n_items"] * info["k"]
        per.append(dist)
        tot += dist
    return tot, per


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The oracle (FP64 CPU, as it stands) on a bounded sample of the same workload."""
    if rank != 0:
        return
    import oracle

    cfg = datagen.CONFIGS[args.config]
    if args.seed:
        import dataclasses
        cfg = dataclasses.replace(cfg, seed=args.seed)
    k = cfg.levels[0]
    X_all = datagen.data(cfg) if cfg.sparse else datagen.data(cfg, 0, cfg.n)
    P = _init_protos(cfg, X_all, datagen.init_indices(cfg.cid, 1, cfg.n, k, cfg.seed))
    cores = oracle.num_threads()
    # rows per step: ~3 s of one oracle Lloyd pass (assignment + update) on the box's cores
    rows = min(cfg.n, 4096)
    for _ in range(4):
        t0 = time.perf_counter()
        _oracle_pass(cfg, X_all, rows, P)
        dt = time.perf_counter() - t0
        if dt >= 2.0 or rows >= cfg.n:
            break
        rows = int(min(cfg.n, rows * 3.0 / max(dt, 1e-3)))
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _oracle_pass(cfg, X_all, rows, P)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = rows * k / (ms / 1000.0)
    sample = f"one Lloyd pass (assign + update) of the first {rows} rows of {cfg.name} level 1 against k={k}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "dim": cfg.dim, "levels": list(cfg.levels), "iters": cfg.iters},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline(cfg, X_all, init):
    """Oracle timed on the host cores on a bounded sample (~10 s): level-1 Lloyd passes."""
    import oracle

    Pd = _init_protos(cfg, X_all, init)
    k = Pd.shape[0]
    rows = min(cfg.n, 2048)
    for _ in range(5):  # re-size until the sample is ~10 s (a small probe under-estimates the rate)
        t0 = time.perf_counter()
        _oracle_pass(cfg, X_all, rows, Pd)
        dt = time.perf_counter() - t0
        if dt >= 7.0 or rows >= cfg.n:
            break
        rows = int(min(cfg.n, rows * 10.0 / max(dt, 1e-3)))
    reps = 1
    while dt < 7.0:  # the whole level-1 pass is short: repeat it (the oracle as it stands, re-run)
        t0 = time.perf_counter()
        _oracle_pass(cfg, X_all, rows, Pd)
        dt += time.perf_counter() - t0
        reps += 1
    cores = oracle.num_threads()
    value = reps * rows * k / dt
    # single-core rate on a smaller sample of the same pass (~3 s)
    single = None
    try:
        oracle.set_num_threads(1)
        r1 = max(64, int(rows * reps * min(1.0, 3.0 / max(dt * cores, 1e-3))))
        r1 = min(r1, cfg.n)
        t0 = time.perf_counter()
        _oracle_pass(cfg, X_all, r1, Pd)
        single = {"value": r1 * k / (time.perf_counter() - t0), "rows": r1}
    finally:
        oracle.set_num_threads(cores)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "single_core": single,
            "sample": f"{reps} x one FP64 Lloyd pass (assign + update) over the first {rows} rows of {cfg.name} "
                      f"level 1 against its k={k} seeded init prototypes ({dt:.1f} s)"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# --------------------------------------------------------------------------- main arm
def main():
    # NCCL prints a version banner on stdout unless told otherwise: the contract is one JSON line
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing contract", file=sys.stderr)

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2208_02734_b200 as mk
    from paper_2208_02734_b200 import buildlib

    if rank == 0:
        buildlib.build()
    comm = None
    if world > 1 or args.force_comm:  # --force-comm: the NCCL build path on one rank (testing)
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        if rank != 0:
            dist.barrier()
        else:
            dist.barrier()
        comm = mk.Comm.from_process_group()

    cfg = datagen.CONFIGS[args.config]
    if args.knn is not None or args.iters is not None or args.seed:  # overrides, reported in `config`
        import dataclasses
        cfg = dataclasses.replace(cfg, knn=args.knn if args.knn is not None else cfg.knn,
                                  iters=args.iters if args.iters is not None else cfg.iters, seed=args.seed)
    beam = args.beam
    bkw = {"tol": args.tol, "empty": args.empty}  # harness flags (defaults = the configs' runs)
    # strong scaling: rank r owns rows [lo, hi) of the config's block-seeded generator
    lo, hi = mk.row_range(cfg.n, world, rank)
    n_local = hi - lo
    n_global = cfg.n
    X_host = datagen.data(cfg, lo, n_local)
    inits = datagen.all_init_indices(cfg)
    qlo, qhi = mk.query_range(cfg.n_queries, world, rank)
    Q_host = datagen.queries(cfg)
    if not cfg.sparse:
        Q_host = Q_host[qlo:qhi]
    csr = cfg.sparse
    if csr:  # C4: CSR rows and CSR queries (row_ptr int64, col int32, val fp32)
        def to_dev(trip):
            rp, col, val = trip
            return mk.Csr(torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev), torch.from_numpy(val).to(dev),
                          cfg.dim)

        X = to_dev(X_host)
        Q_host = _csr_rows(Q_host, qlo, qhi)
        Q = to_dev(Q_host)
    else:
        X = torch.from_numpy(X_host).to(dev)
        Q = torch.from_numpy(np.ascontiguousarray(Q_host)).to(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    # live timing of the assignment kernel only inside the timed region (one event pair per
    # pass; timing every kernel class costs ~5 % of a C2 step); the update kernel is timed in
    # two extra builds after the timed region
    flags = mk.MASK_TIME_ASSIGN | (mk.MASK_FORCE_SIMT if args.force_simt else 0)
    if world == 1:
        flags |= mk.MASK_BORROW_DATA
    stream = torch.cuda.current_stream(dev)
    nq_local = (Q.rows if csr else int(Q.shape[0]))
    qout = (torch.empty((nq_local, cfg.knn), dtype=torch.int64, device=dev),
            torch.empty((nq_local, cfg.knn), dtype=torch.float32, device=dev))  # result buffers, reused

    def step():
        idx = mk.build(X, cfg.levels, cfg.iters, inits, **bkw, flags=flags, comm=comm, n_global=n_global,
                       row_offset=lo, stream=stream)
        ids, d2 = idx.query(Q, knn=cfg.knn, beam=beam, stream=stream, out=qout)
        return idx, ids, d2

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        idx, _, _ = step()
        idx.free()
    barrier()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        sampler.wait_rows(1, 5.0)
    launches0 = mk.kernel_launches()
    step_ms = []
    kt = {"assign": 0.0, "assign_n": 0, "update": 0.0, "update_n": 0}
    dist_total = 0
    per_level = None
    build_ms = []
    query_ms = []
    for s in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (inputs are smaller than L2)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx = mk.build(X, cfg.levels, cfg.iters, inits, **bkw, flags=flags, comm=comm, n_global=n_global,
                       row_offset=lo, stream=stream)
        e1.record(stream)
        ids, d2 = idx.query(Q, knn=cfg.knn, beam=beam, stream=stream, out=qout)
        e2.record(stream)
        barrier()
        step_ms.append(e0.elapsed_time(e2))
        build_ms.append(e0.elapsed_time(e1))
        query_ms.append(e1.elapsed_time(e2))
        dt, per_level = lloyd_distances(idx, len(cfg.levels))
        dist_total += dt
        tm = idx.timing(1)
        kt["assign"] += tm["assign"]["ms"]
        kt["assign_n"] += tm["assign"]["launches"]
        if s < args.steps - 1:
            idx.free()
    launches = mk.kernel_launches() - launches0
    if sampler:
        sampler.wait_rows(len(sampler.rows) + 1, 1.0)
        sampler.stop()
    # update kernel (K5/K6) times: two extra builds with every kernel class timed (untimed region)
    for _ in range(2):
        idx_u = mk.build(X, cfg.levels, cfg.iters, inits, **bkw, flags=(flags & ~mk.MASK_TIME_ASSIGN) | mk.MASK_TIME_KERNELS,
                         comm=comm, n_global=n_global, row_offset=lo, stream=stream)
        tu = idx_u.timing(1)
        kt["update"] += tu["update"]["ms"]
        kt["update_n"] += tu["update"]["launches"]
        idx_u.free()

    total_ms = sum(step_ms)

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t[0])

    # every rank's index covers all n_global rows (level 1 n_items = n_global after the gather),
    # so dist_total already counts the whole job's work; the time is the slowest rank's
    total_ms = max_over_ranks(total_ms)
    build_mean = max_over_ranks(statistics.mean(build_ms))
    query_mean = max_over_ranks(statistics.mean(query_ms))
    value = dist_total / (total_ms / 1000.0)

    # ---- roofline of the dominant kernel (level-1 assignment), measured live above
    pk = peaks()
    lvl1 = idx.level_info(1)
    n1, k1, d = n_local, lvl1["k"], cfg.dim
    n1g = n_local  # rows this rank's level-1 assignment launches process
    assign_avg_ms = kt["assign"] / max(kt["assign_n"], 1)
    akern = idx.timing(1)["assign_kernel"]
    use_tc = akern in ("K1-tcgen05-3xtf32", "K1-tcgen05-3xfp16")
    h16 = akern == "K1-tcgen05-3xfp16"
    if akern == "K11-fused-small-level":  # one launch runs the whole level: all its passes
        flops = 3.0 * n1 * k1 * d * lvl1["passes"]
        peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "K11 fused small level (level 1, all passes in one launch)",
                "unit": "TFLOP/s", "peak_basis": "FP32 SIMT = 148 SMs x 128 lanes x 2 flop x sm_max_mhz; "
                "latency-bound (grid barriers between passes), DESIGN.md K11"}
    elif akern == "K3-csr":
        flops = 2.0 * X_host[0][-1] * k1  # one FMA per (non-zero, prototype): the sparse contraction
        peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "K3 CSR assignment (level 1)", "unit": "TFLOP/s",
                "peak_basis": "FP32 FMA = 148 SMs x 128 lanes x 2 flop x sm_max_mhz (DESIGN.md K3)"}
    elif use_tc:
        flops = 6.0 * n1g * k1 * d  # 3xTF32 / 3xFP16: three MMA products per useful multiply-add
        # a kernel timed inside a long step runs at the sustained clock (B200_PROFILING.md):
        # steps over 1 s take the sustained bf16 figure, shorter ones the burst figure
        sustained = total_ms / args.steps > 1000.0
        bf = pk["bf16_tflops_sustained"] if sustained else pk["bf16_tflops"]
        if h16:  # kind::f16 runs at the bf16 rate
            peak = bf
            roof = {"bound": "tensor", "kernel": "K1 tcgen05 3xFP16 assignment (level 1)", "unit": "TFLOP/s",
                    "peak_basis": f"FP16 dense = {pk['source']} bf16 {'sustained' if sustained else 'burst'} "
                                  f"{bf} TFLOP/s (same rate)"}
        else:
            peak = 0.5 * bf
            roof = {"bound": "tensor", "kernel": "K1 tcgen05 3xTF32 assignment (level 1)", "unit": "TFLOP/s",
                    "peak_basis": f"TF32 dense = 0.5 x {pk['source']} bf16 {'sustained' if sustained else 'burst'} "
                                  f"{bf} TFLOP/s (nominal ratio)"}
    else:
        flops = 3.0 * n1 * k1 * d  # sub + fma per coordinate
        peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "K2 FP32 SIMT assignment (level 1)", "unit": "TFLOP/s",
                "peak_basis": "FP32 SIMT = 148 SMs x 128 lanes x 2 flop x sm_max_mhz"}
    achieved = flops / (assign_avg_ms / 1000.0) / 1e12 if assign_avg_ms > 0 else 0.0
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak if peak else None,
                 "traffic": ncu_traffic(cfg.name, roof["kernel"]), "avg_launch_ms": assign_avg_ms,
                 "timing": "CUDA events around every launch of this kernel inside the timed region (MASK_TIME_ASSIGN)",
                 "share_of_step": kt["assign"] / total_ms if total_ms else None})
    upd_avg = kt["update"] / max(kt["update_n"], 1)
    if csr:  # K6: CSR rows + labels read, k x d sums + counts written
        upd_bytes = int(X_host[0][-1]) * 8 + (n1 + 1) * 8 + n1 * 4 + k1 * (d + 1) * 4
    else:
        upd_bytes = n1 * d * 4 + n1 * 4 + k1 * (d + 1) * 4
    upd = {"kernel": "K6 CSR update (sums+counts)" if csr else "K5 update (sums+counts)", "avg_launch_ms": upd_avg,
           "timing": "CUDA events in 2 builds after the timed region (MASK_TIME_KERNELS)",
           "achieved_gbs": upd_bytes / (upd_avg / 1000.0) / 1e9 if upd_avg > 0 else None,
           "peak_gbs": pk["hbm_gbs"]}
    if upd["achieved_gbs"]:
        upd["frac"] = upd["achieved_gbs"] / pk["hbm_gbs"]

    # ---- recall of the query batch on a sample (oracle exact k-NN is the definition), and the
    #      QPS @ recall sweep: the whole local query batch at beams 1..32 (CUDA events), recall@k
    #      of each on the same sample; qps_at_recall = the fastest beam reaching recall >= 0.9
    recall = None
    sweep = None
    if rank == 0 and world == 1:
        try:
            import oracle

            m = 100 if cfg.n >= 5_000_000 else 200
            Qs = _csr_rows(Q_host, 0, m) if csr else Q_host[:m]
            eids, _, gap = oracle.knn_exact(X_host, Qs, cfg.knn, csr=csr)
            recall = oracle.recall(ids[:m].cpu().numpy(), eids)
            if not args.no_sweep:
                sweep = []
                for b in (1, 2, 4, 8, 16, 32) + (() if csr else (64, 128, 256)):  # (CSR queries: beam <= 32)
                    idx.query(Q, knn=cfg.knn, beam=b, stream=stream, out=qout)  # warm-up
                    q0 = torch.cuda.Event(enable_timing=True)
                    q1 = torch.cuda.Event(enable_timing=True)
                    q0.record(stream)
                    ib, _ = idx.query(Q, knn=cfg.knn, beam=b, stream=stream, out=qout)
                    q1.record(stream)
                    torch.cuda.synchronize(dev)
                    qms = q0.elapsed_time(q1)
                    sweep.append({"beam": b, "recall": oracle.recall(ib[:m].cpu().numpy(), eids),
                                  "qps": nq_local / (qms / 1000.0), "ms": qms})
                    if sweep[-1]["recall"] >= 0.9:  # the smallest beam at the target: done
                        break
        except Exception as e:  # the recall sample is a report, not the timed value
            recall = f"unavailable: {e}"
    qps_at_recall = None
    if sweep:
        hit = [r for r in sweep if r["recall"] >= 0.9]
        best = hit[0] if hit else max(sweep, key=lambda r: r["recall"])
        qps_at_recall = {"target_recall": 0.9, "reached": bool(hit), "beam": best["beam"], "recall": best["recall"],
                         "qps": best["qps"], "sample_queries": m, "sweep": sweep}

    # ---- e2e through the C-ABI with HOST buffers (H2D/D2H copies inside the call): every
    #      rank passes its pinned host shard and query slice; max over ranks of the wall time
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        if csr:
            Xp = mk.Csr(*[pin(a) for a in X_host], cfg.dim)
            Qp = mk.Csr(*[pin(a) for a in Q_host], cfg.dim)
        else:
            Xp, Qp = pin(X_host), pin(Q_host)
        h_ms, dh_tot = [], 0
        for s in range(4):  # one untimed warm-up of the host path, then the mean of three
            flush.zero_()
            barrier()
            t0 = time.perf_counter()
            idx_h = mk.build(Xp, cfg.levels, cfg.iters, inits, **bkw, comm=comm, n_global=n_global, row_offset=lo,
                             stream=stream)
            ids_h, d2_h = idx_h.query(Qp, knn=cfg.knn, beam=beam, stream=stream)
            torch.cuda.synchronize(dev)
            dt_ms = (time.perf_counter() - t0) * 1000.0
            barrier()
            if s > 0:
                h_ms.append(max_over_ranks(dt_ms))
                dh_tot += lloyd_distances(idx_h, len(cfg.levels))[0]
            idx_h.free()
        e2e = {"value": dh_tot / (sum(h_ms) / 1000.0), "unit": UNIT, "ms_per_step": statistics.mean(h_ms),
               "h2d_bytes_per_step": int(_nbytes(X_host) + _nbytes(Q_host)) * world,
               "d2h_bytes_per_step": int(ids_h.nbytes + d2_h.nbytes) * world,
               "timing": "host wall clock around mask_build + mask_query with pinned host inputs/outputs, "
                         "max over ranks, L2 flushed before each step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, X_host, inits[0])
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {e}"}

    if rank == 0:
        clocks = sampler.summary() if sampler else None
        if use_tc and clocks and clocks.get("sm_mhz"):
            # context for `frac`: the MMA rate measured on this GPU (tools/mma_ubench.cu: TF32 4096, FP16 twice that
            # flop/clk/SM, K1) at the median SM clock of the timed region, and the burst peak
            hw = (8192.0 if h16 else 4096.0) * 148 * clocks["sm_mhz"] * 1e6 / 1e12
            roof["tensor_util_at_clock"] = achieved / hw
            roof["hw_tf32_at_clock_tflops" if not h16 else "hw_f16_at_clock_tflops"] = hw
            roof["frac_of_burst_peak"] = achieved / ((1.0 if h16 else 0.5) * pk["bf16_tflops"])
        if akern == "K3-csr" and clocks and clocks.get("sm_mhz") and assign_avg_ms > 0:
            # the binding unit of K3 (DESIGN.md §6 K3/K3T): every FMA consumes one 4-byte prototype
            # operand through the L1/shared-memory data path (128 B/clk/SM); operand bytes/s
            # against that path at the timed region's median clock
            opb = 4.0 * X_host[0][-1] * k1 / (assign_avg_ms / 1000.0)
            l1 = 148 * 128.0 * clocks["sm_mhz"] * 1e6
            roof["l1_datapath"] = {"operand_gbs": opb / 1e9, "peak_gbs": l1 / 1e9, "frac": opb / l1}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "n_per_gpu": n_local, "n_global": n_global, "dim": cfg.dim,
                       "levels": list(cfg.levels), "iters": cfg.iters, "queries": cfg.n_queries,
                       "knn": cfg.knn, "beam": beam, "parallelism": f"dp{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (512 MiB write)",
                       "seed": args.seed, "tol": args.tol, "empty": args.empty},
            "per_level_distances": per_level, "build_ms": build_mean,
            # SURVEY §8(d) variant (i): level-1 distances over the level-1 assignment kernels'
            # own time (live CUDA events); `value` is variant (ii), the whole step
            "level1_distances_per_s_assign_only": (per_level[0] * args.steps / (kt["assign"] / 1000.0)
                                                   if kt["assign"] > 0 and akern != "K11-fused-small-level" else None),
            "query_ms": query_mean, "query_qps": cfg.n_queries / (query_mean / 1000.0),
            "recall_at_k_sample": recall, "qps_at_recall": qps_at_recall, "roofline": roof, "update_roofline": upd,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches // max(args.steps, 1)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    idx.free()
    if comm:
        comm.free()
    if world > 1 or args.force_comm:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
