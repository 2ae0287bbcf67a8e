"""Run by test_gpu_cluster.py under torch.distributed.run (NCCL): DistCluster end to end, each
rank's node built independently, against LocalCluster over the same partitions in rank 0."""
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2208_02734_b200 as mk  # noqa: E402
from paper_2208_02734_b200.cluster import DistCluster, LocalCluster  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    X = datagen.gaussian_clouds(71, 400, radius=20.0, sigma=1.0)
    n = X.shape[0]
    bounds = [(r * n // world, (r + 1) * n // world) for r in range(world)]
    inits = [[datagen.init_indices(700 + r, 1, hi - lo, 16), datagen.init_indices(700 + r, 2, 16, 4)]
             for r, (lo, hi) in enumerate(bounds)]
    lo, hi = bounds[rank]
    Xl = torch.from_numpy(X[lo:hi]).to(dev)
    c0 = mk.collective_count()
    cl = DistCluster.build(Xl, [16, 4], 8, inits[rank])
    assert cl.build_collectives == 0 and mk.collective_count() == c0
    Q = datagen.gaussian_clouds(72, 13, radius=20.0, sigma=1.0)  # 104 queries
    qlo, qhi = mk.query_range(len(Q), world, rank)
    for eps in (math.inf, 3.0):
        ids, d2, stats = cl.knn(torch.from_numpy(Q[qlo:qhi]).to(dev), knn=10, epsilon=eps)
        parts = [None] * world
        dist.all_gather_object(parts, (qlo, ids.cpu().numpy(), d2.cpu().numpy()))
        if rank == 0:
            got_i = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])])
            got_d = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            loc = LocalCluster.build([torch.from_numpy(X[a:b]).to(dev) for a, b in bounds], [16, 4], 8, inits)
            ri, rd, _, _ = loc.knn(torch.from_numpy(Q).to(dev), knn=10, epsilon=eps)
            assert np.array_equal(got_i, ri.cpu().numpy()) and np.array_equal(got_d, rd.cpu().numpy())
            loc.free()
    cl.free()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("DIST_CLUSTER_OK")


if __name__ == "__main__":
    main()
