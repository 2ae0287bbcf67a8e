"""Seeded synthetic inputs for the MASK hot path (BASELINE.json configs C1-C5).

This module is shared by the oracle side (``oracle/``) and the CUDA side
(``paper_2208_02734_b200``) and deliberately holds NONE of the method's
arithmetic: it draws data points, queries and the random initial-prototype
indices (the only random numbers the method consumes, passed to both sides as
inputs).  Nothing here computes a distance, an assignment, a mean or a
neighbour list.

Recipe:

* seeds: data = 1000+c, queries = 2000+c, init = 3000+c (c = config number), each plus
  100,000 s for the harness's ``--seed s`` (s = 0: the documented streams);
* rows are generated in whole blocks of 2**14; block b draws from
  ``SeedSequence([seed, b])`` so any GPU count / shard sees identical rows;
* mixture parameters (centres, scales, covariances, weights, the C4 column
  permutation) come from ``SeedSequence([seed, 0xFFFFFFFF])``;
* initial prototypes of level l are ``Generator(PCG64(SeedSequence([3000+c, l])))
  .choice(n_{l-1}, k_l, replace=False)`` (D2: seeded random-point init).

The paper's own synthetic data are 8 Gaussian clouds in R^2 (PAPER.md
§4 "Performance evaluation", lines 1146-1191); its high-dimensional sparse
workload is Reuters-21578 TF-IDF (§4.3), which is
NOT reproduced here — C4's generator only imitates its shape (non-negative,
sparse, Zipfian column popularity, L2-normalised rows).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import os

import numpy as np

BLOCK_ROWS = 1 << 14
PARAM_BLOCK = 0xFFFFFFFF


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (configs[c-1])."""

    cid: int
    name: str
    n: int
    dim: int
    levels: Tuple[int, ...]  # k per level, bottom first
    iters: int  # Lloyd (assign, update) pairs T; one final assignment follows
    n_queries: int
    knn: int
    sparse: bool = False
    seed: int = 0  # harness --seed: 0 = the documented streams; s > 0 offsets every base seed by 100,000 s

    @property
    def seed_base(self) -> int:
        return 100_000 * self.seed

    def scaled(self, div: int, min_k: int = 2) -> "Config":
        """Scaled-down replica: same generator and d, N and every k_l divided by ``div``."""
        n = max(self.n // div, 1)
        ks = []
        prev = n
        for k in self.levels:
            kk = max(min(k // div, prev), min(min_k, prev))
            ks.append(kk)
            prev = kk
        return dataclasses.replace(
            self,
            name=f"{self.name}/{div}",
            n=n,
            levels=tuple(ks),
            n_queries=max(self.n_queries // div, 16),
        )


CONFIGS = {
    1: Config(1, "C1", 10_000, 2, (100, 10), 20, 100, 10),
    2: Config(2, "C2", 1_000_000, 16, (4096, 256, 16), 25, 10_000, 10),
    3: Config(3, "C3", 10_000_000, 64, (65536, 1024, 32), 20, 100_000, 10),
    4: Config(4, "C4", 1_000_000, 10_000, (8192, 256), 15, 10_000, 10, sparse=True),
    5: Config(5, "C5", 100_000_000, 128, (262144, 4096, 64), 15, 1_000_000, 10),
}

C4_NNZ_PER_ROW = 50  # 0.5% of d = 10,000 (BASELINE.json configs[3]); fixed (flagged reading)


def _rng(*words: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(words))))


# --------------------------------------------------------------------------- mixtures
def _mixture_params(cfg: Config, seed: int):
    """Per-config mixture parameters from the reserved parameter stream."""
    g = _rng(seed, PARAM_BLOCK)
    d = cfg.dim
    if cfg.cid == 1:
        m = 10
        centers = g.uniform(-10.0, 10.0, size=(m, d))
        return dict(kind="iso", centers=centers, sigma=np.ones(m), weights=np.full(m, 1.0 / m))
    if cfg.cid == 2:
        m = 256
        centers = g.uniform(-10.0, 10.0, size=(m, d))  # unspecified by BJ -> flagged reading
        lam = g.uniform(0.1, 2.0, size=(m, d))  # covariance eigenvalues (variances)
        qs = np.empty((m, d, d))
        for i in range(m):
            a = g.standard_normal((d, d))
            q, r = np.linalg.qr(a)
            q = q * np.sign(np.diag(r))[None, :]  # Haar sign fix
            qs[i] = q
        w = np.arange(1, m + 1, dtype=np.float64) ** -1.1
        return dict(kind="aniso", centers=centers, lam=lam, q=qs, weights=w / w.sum())
    if cfg.cid == 3:
        m = 1024
        centers = g.standard_normal((m, d)) * 5.0  # N(0, 25 I)
        sigma = g.uniform(0.5, 2.0, size=m)
        return dict(kind="iso", centers=centers, sigma=sigma, weights=np.full(m, 1.0 / m))
    if cfg.cid == 5:
        m = 16384
        centers = g.standard_normal((m, d)) * 4.0  # N(0, 16 I)
        return dict(kind="iso", centers=centers, sigma=np.ones(m), weights=np.full(m, 1.0 / m))
    if cfg.cid == 4:
        perm = g.permutation(cfg.dim)  # rank -> column, so hot terms are not adjacent
        return dict(kind="sparse", perm=perm)
    raise ValueError(cfg.cid)


def _dense_block(cfg: Config, params, seed: int, block: int, rows: int) -> np.ndarray:
    g = _rng(seed, block)
    comp = g.choice(len(params["weights"]), size=rows, p=params["weights"])
    z = g.standard_normal((rows, cfg.dim))
    if params["kind"] == "iso":
        x = params["centers"][comp] + params["sigma"][comp][:, None] * z
    else:
        lam = params["lam"][comp]  # rows x d
        q = params["q"][comp]  # rows x d x d
        x = params["centers"][comp] + np.einsum("rij,rj->ri", q, np.sqrt(lam) * z)
    return x.astype(np.float32)


def _zipf_ranks(g: np.random.Generator, count: int, s: float, nmax: int) -> np.ndarray:
    """``count`` draws from Zipf(s) truncated to 1..nmax (inverse-CDF on the exact pmf)."""
    pmf = np.arange(1, nmax + 1, dtype=np.float64) ** -s
    cdf = np.cumsum(pmf)
    cdf /= cdf[-1]
    u = g.random(count)
    return np.minimum(np.searchsorted(cdf, u, side="right"), nmax - 1)  # 0-based rank


def _sparse_block(cfg: Config, params, seed: int, block: int, rows: int):
    g = _rng(seed, block)
    nnz = C4_NNZ_PER_ROW
    # repeated truncated-Zipf(1.2) rank draws, duplicates rejected, first nnz distinct kept
    # in draw order (flagged reading).  Draw in rounds of 4*nnz per row until every row has nnz.
    draws = _zipf_ranks(g, rows * 4 * nnz, 1.2, cfg.dim).reshape(rows, 4 * nnz)
    while True:
        m = draws.shape[1]
        order = np.argsort(draws, axis=1, kind="stable")
        srt = np.take_along_axis(draws, order, axis=1)
        first = np.ones_like(srt, dtype=bool)
        first[:, 1:] = srt[:, 1:] != srt[:, :-1]
        uniq = np.zeros_like(first)
        np.put_along_axis(uniq, order, first, axis=1)
        short = uniq.sum(axis=1) < nnz
        if not short.any():
            break
        extra = _zipf_ranks(g, rows * nnz, 1.2, cfg.dim).reshape(rows, nnz)
        draws = np.concatenate([draws, extra], axis=1)
    rank = np.cumsum(uniq, axis=1)
    keep = uniq & (rank <= nnz)
    cols = draws[keep].reshape(rows, nnz)
    cols = params["perm"][cols]
    cols.sort(axis=1)
    vals = g.lognormal(0.0, 1.0, size=(rows, nnz))
    vals /= np.sqrt((vals * vals).sum(axis=1, keepdims=True))  # rows L2-normalised (BJ configs[3])
    row_ptr = np.arange(rows + 1, dtype=np.int64) * nnz
    return row_ptr, cols.reshape(-1).astype(np.int32), vals.reshape(-1).astype(np.float32)


def _rows(cfg: Config, seed: int, n: int, start: int = 0):
    params = _mixture_params(cfg, seed)
    out = []
    row = start
    end = start + n
    while row < end:
        b = row // BLOCK_ROWS
        b_start = b * BLOCK_ROWS
        lo = row - b_start
        hi = min(end - b_start, BLOCK_ROWS)
        # always draw the whole block so that any slice of the dataset is prefix/shard stable
        if cfg.sparse:
            rp, c, v = _sparse_block(cfg, params, seed, b, BLOCK_ROWS)
            out.append((rp[lo:hi + 1] - rp[lo], c[rp[lo]:rp[hi]], v[rp[lo]:rp[hi]]))
        else:
            out.append(_dense_block(cfg, params, seed, b, BLOCK_ROWS)[lo:hi])
        row = b_start + hi
    if cfg.sparse:
        rps, cs, vs = [], [], []
        off = 0
        for rp, c, v in out:
            rps.append(rp[:-1] + off)
            off += rp[-1]
            cs.append(c)
            vs.append(v)
        rps.append(np.array([off], dtype=np.int64))
        return np.concatenate(rps), np.concatenate(cs), np.concatenate(vs)
    return np.concatenate(out, axis=0) if out else np.zeros((0, cfg.dim), np.float32)


def _fill_blocks(args):
    """Worker of data_parallel: whole blocks [b0, b1) into the shared output array."""
    name, shape, cid, b0, b1, n, seed = args
    from multiprocessing import shared_memory

    cfg = dataclasses.replace(CONFIGS[cid], seed=seed)
    shm = shared_memory.SharedMemory(name=name)
    try:
        out = np.ndarray(shape, dtype=np.float32, buffer=shm.buf)
        params = _mixture_params(cfg, 1000 + cid + cfg.seed_base)
        for b in range(b0, b1):
            lo, hi = b * BLOCK_ROWS, min((b + 1) * BLOCK_ROWS, n)
            out[lo:hi] = _dense_block(cfg, params, 1000 + cid + cfg.seed_base, b, BLOCK_ROWS)[: hi - lo]
    finally:
        shm.close()
    return b1 - b0


def data_parallel(cfg: Config, workers: Optional[int] = None):
    """All rows of a dense config, blocks generated by a process pool into shared memory.

    Identical to ``data(cfg)`` (same per-block streams); for the 51 GB C5 set.  Returns
    (array, shm): keep ``shm`` alive while the array is used, then ``shm.close(); shm.unlink()``."""
    import multiprocessing as mp
    from multiprocessing import shared_memory

    assert not cfg.sparse
    n = cfg.n
    shape = (n, cfg.dim)
    shm = shared_memory.SharedMemory(create=True, size=n * cfg.dim * 4)
    nb = (n + BLOCK_ROWS - 1) // BLOCK_ROWS
    workers = workers or os.cpu_count() or 1
    step = max(1, (nb + 4 * workers - 1) // (4 * workers))
    jobs = [(shm.name, shape, cfg.cid, b, min(b + step, nb), n, cfg.seed) for b in range(0, nb, step)]
    with mp.get_context("fork").Pool(workers) as pool:
        done = sum(pool.map(_fill_blocks, jobs))
    assert done == nb
    return np.ndarray(shape, dtype=np.float32, buffer=shm.buf), shm


def group_perm(seed: int, n: int) -> np.ndarray:
    """The seeded random split order of the grouped construction's data layer (points
    "randomly assigned" to groups): a permutation of range(n)."""
    return _rng(seed, 0).permutation(n).astype(np.int64)


def relocation_keys(base_seed: int, iteration: int, n: int) -> np.ndarray:
    """Random order keys of relocation iteration ``iteration`` (the rebuild seed policy
    seed = base_seed + iteration, SPEC DESIGN DECISIONS): a permutation rank per point, used to
    order the points inside each target group before the rebuild (no method arithmetic)."""
    return _rng(base_seed + iteration, 7).permutation(n).astype(np.int64)


def gaussian_clouds(seed: int, per_cloud: int, radius: float, sigma: float = 1.0, clouds: int = 8) -> np.ndarray:
    """``clouds`` isotropic Gaussian clouds in R^2 (the paper's synthetic benchmark),
    centres evenly spaced on a circle of ``radius``; radius >> sigma gives the no-overlap version
    (centres and sigma are unspecified in the paper: flagged reading G6)."""
    g = _rng(seed, 0)
    ang = np.arange(clouds) * (2.0 * np.pi / clouds)
    centres = radius * np.stack([np.cos(ang), np.sin(ang)], axis=1)
    comp = np.repeat(np.arange(clouds), per_cloud)
    return (centres[comp] + sigma * g.standard_normal((clouds * per_cloud, 2))).astype(np.float32)


def data(cfg: Config, start: int = 0, count: Optional[int] = None):
    """Rows [start, start+count) of config ``cfg``'s dataset (dense fp32 n x d, or CSR triple)."""
    count = cfg.n - start if count is None else count
    return _rows(cfg, 1000 + cfg.cid + cfg.seed_base, count, start)


def queries(cfg: Config, count: Optional[int] = None):
    """Queries drawn from an independent stream of the same generator."""
    count = cfg.n_queries if count is None else count
    return _rows(cfg, 2000 + cfg.cid + cfg.seed_base, count, 0)


def init_indices(cfg_id: int, level: int, n_items: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct indices in [0, n_items) for level ``level`` (1-based), seeded (D2)."""
    if not (1 <= k <= n_items):
        raise ValueError("need 1 <= k <= n_items")
    g = _rng(3000 + cfg_id + 100_000 * seed, level)
    return g.choice(n_items, size=k, replace=False).astype(np.int64)


def all_init_indices(cfg: Config) -> List[np.ndarray]:
    out = []
    prev = cfg.n
    for l, k in enumerate(cfg.levels, start=1):
        out.append(init_indices(cfg.cid, l, prev, k, cfg.seed))
        prev = k
    return out


def random_dense(seed: int, n: int, d: int, scale: float = 1.0, offset: float = 0.0) -> np.ndarray:
    """Plain seeded Gaussian matrix for unit/edge tests."""
    g = _rng(seed, 7)
    return (offset + scale * g.standard_normal((n, d))).astype(np.float32)


def blobs(seed: int, n: int, d: int, m: int, spread: float = 10.0, sigma: float = 1.0) -> np.ndarray:
    """Isotropic Gaussian mixture with m components (test helper, C1-like)."""
    g = _rng(seed, 11)
    centers = g.uniform(-spread, spread, size=(m, d))
    comp = g.integers(0, m, size=n)
    return (centers[comp] + sigma * g.standard_normal((n, d))).astype(np.float32)


def ragged_csr(seed: int, n: int, d: int, max_nnz: int, zipf: float = 1.2):
    """Random CSR rows of 0..max_nnz distinct sorted columns (Zipf(``zipf``) column popularity,
    so a hot set exists), non-negative L2-normalised values; row 0 is empty, row 1 (if any) has
    min(max_nnz, d) non-zeros."""
    g = _rng(seed, 17)
    lens = g.integers(0, max_nnz + 1, size=n)
    if n:
        lens[0] = 0
    if n > 1:
        lens[1] = min(max_nnz, d)
    cols, vals, rp = [], [], [0]
    for i in range(n):
        m = int(min(lens[i], d))
        c = np.unique(_zipf_ranks(g, 8 * m + 8, zipf, d))[:m] if m else np.zeros(0, np.int64)
        while c.size < m:
            c = np.unique(np.concatenate([c, g.choice(d, size=m, replace=False)]))[:m]
        v = g.lognormal(0.0, 1.0, size=c.size)
        if c.size:
            v /= np.sqrt((v * v).sum())
        cols.append(np.sort(c))
        vals.append(v)
        rp.append(rp[-1] + c.size)
    col = np.concatenate(cols).astype(np.int32) if n else np.zeros(0, np.int32)
    val = np.concatenate(vals).astype(np.float32) if n else np.zeros(0, np.float32)
    return np.asarray(rp, np.int64), col, val


def random_csr(seed: int, n: int, d: int, nnz_row: int):
    """Random CSR rows with ``nnz_row`` distinct sorted columns, non-negative L2-normalised values."""
    g = _rng(seed, 13)
    nnz_row = min(nnz_row, d)
    cols = np.stack([np.sort(g.choice(d, size=nnz_row, replace=False)) for _ in range(n)]) if n else np.zeros((0, nnz_row), np.int64)
    vals = g.lognormal(0.0, 1.0, size=(n, nnz_row))
    if n:
        vals /= np.sqrt((vals * vals).sum(axis=1, keepdims=True))
    row_ptr = np.arange(n + 1, dtype=np.int64) * nnz_row
    return row_ptr, cols.reshape(-1).astype(np.int32), vals.reshape(-1).astype(np.float32)
