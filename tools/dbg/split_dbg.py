import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import datagen, oracle, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[2].scaled(64)
X = datagen.data(cfg)
idx = mk.build(torch.from_numpy(X).cuda(), cfg.levels, 6, datagen.all_init_indices(cfg))
L = idx.num_levels
P0 = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
L0 = [idx.labels(l).astype(np.int64) for l in range(1, L + 1)]
thr = 300
ns = idx.split(thr, iters=8, seed=11)
Pr, Lr, split = oracle.split_partitions(P0, L0, X, threshold=thr, T=8, seed=11)
P1 = idx.prototypes(1).astype(np.float64); L1 = idx.labels(1)
print("split", ns, split, "k", P1.shape, Pr[0].shape)
k1 = P0[0].shape[0]
nxt = k1
X64 = X.astype(np.float64)
counts = np.bincount(L0[0], minlength=k1)
for j in split:
    s = -(-int(counts[j]) // thr)
    ids = [j] + list(range(nxt, nxt + s - 1)); nxt += s - 1
    e = np.linalg.norm(P1[ids] - Pr[0][ids]) / np.linalg.norm(Pr[0][ids])
    rows = np.nonzero(L0[0] == j)[0]
    nd = int((L1[rows] != Lr[0][rows]).sum())
    # oracle trajectory and the tie windows along it
    init = oracle.seeded_init((11 + j) & ((1 << 64) - 1), 1, len(rows), s)
    res = oracle.lloyd(X64[rows], init, 8, trace=True)
    gaps = []
    for (P, lab) in res.passes:
        _, b1, b2 = oracle.assign(X64[rows], P)
        gaps.append(float(((b2 - b1) / b2).min()))
    print(f"j={j} n={len(rows)} s={s} relL2={e:.2e} label diffs={nd} passes={len(res.passes)} min rel gap per pass={['%.1e'%g for g in gaps]}")
