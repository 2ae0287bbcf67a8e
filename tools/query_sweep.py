"""QPS @ recall of the batched k-NN descent (K9) over the beam width b (SURVEY §8(d) "query QPS
@ recall"; b = 1 is Algorithm 2, b > 1 the multi-probe descent of NEXT-2) on a full-size
config built once on one B200.  QPS = Q / (device time of one mask_query over the config's
whole query batch, resident in HBM; CUDA events, median of 5); recall@k on the first
``--sample`` queries against the oracle's exact k-NN (brute force, FP64, host cores).

    python tools/query_sweep.py [--config 2] [--sample 500] [--beams 1,2,4,8,16,32]
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--sample", type=int, default=500)
    ap.add_argument("--beams", default="1,2,4,8,16,32")
    ap.add_argument("--iters", type=int, default=0, help="Lloyd iterations (0: the config's)")
    ap.add_argument("--modes", default="auto", help="MASK_QUERY_GROUPED values to compare, e.g. 0,1")
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.config]
    X = datagen.data(cfg)
    Q = datagen.queries(cfg)
    dev = torch.device("cuda", 0)
    Xd = torch.from_numpy(X).to(dev)
    Qd = torch.from_numpy(Q).to(dev)
    t0 = time.time()
    idx = mk.build(Xd, cfg.levels, a.iters or cfg.iters, datagen.all_init_indices(cfg), flags=mk.MASK_BORROW_DATA)
    torch.cuda.synchronize()
    print(f"{cfg.name}: build {time.time() - t0:.2f} s", file=sys.stderr, flush=True)
    t0 = time.time()
    eids, _, _ = oracle.knn_exact(X, Q[:a.sample], cfg.knn)
    print(f"exact k-NN of {a.sample} queries on the host: {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    st = torch.cuda.current_stream(dev)
    for b in [int(x) for x in a.beams.split(",")]:
        first = None
        for mode in a.modes.split(","):
            os.environ.pop("MASK_QUERY_GROUPED", None)
            os.environ.pop("MASK_GROUPED_LEVEL", None)
            os.environ.pop("MASK_GROUPED_FROM_TOP", None)
            if mode.startswith("g"):  # g0 / g1 / g2: grouped leaf scan; + level-1 step; + steps from the top
                os.environ["MASK_QUERY_GROUPED"] = "1"
                os.environ["MASK_GROUPED_LEVEL"] = "0" if mode == "g0" else "1"
                if mode == "g2":
                    os.environ["MASK_GROUPED_FROM_TOP"] = "1"
            elif mode != "auto":
                os.environ["MASK_QUERY_GROUPED"] = mode
            ms = []
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                ids, d2 = idx.query(Qd, knn=cfg.knn, beam=b, stream=st)
                e1.record(st)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            t = statistics.median(ms[1:])
            rec = oracle.recall(ids[:a.sample].cpu().numpy(), eids)
            h = ids.cpu().numpy()
            agree = None if first is None else float((h == first).all(1).mean())
            first = h if first is None else first
            print(json.dumps({"workload": cfg.name, "queries": int(Q.shape[0]), "knn": cfg.knn, "beam": b,
                              "grouped": mode, "query_ms": t, "qps": Q.shape[0] / (t / 1e3), "recall": rec,
                              "recall_sample": a.sample, "ids_agree_with_first_mode": agree}), flush=True)
        os.environ.pop("MASK_QUERY_GROUPED", None)
        os.environ.pop("MASK_GROUPED_LEVEL", None)
    idx.free()


if __name__ == "__main__":
    main()
