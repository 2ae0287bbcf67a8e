"""Host-side sharding arithmetic for one-process-per-GPU runs (no method arithmetic).

Rows: rank r owns global rows [floor(r*N/W), floor((r+1)*N/W)); prototypes
are replicated and the per-iteration partial sums/counts are combined by one allreduce
inside mask_build.  Queries are sharded by batch the same way; results concatenate in rank
order.
"""
from __future__ import annotations

from typing import Tuple


def row_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return (rank * n) // world, ((rank + 1) * n) // world


def query_range(nq: int, world: int, rank: int) -> Tuple[int, int]:
    return row_range(nq, world, rank)
