import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2208_02734_b200 as mk
for d in (16, 64):
    rng = np.random.default_rng(d)
    k, n = 300, 4096
    P = (rng.standard_normal((k, d)) * 4.0).astype(np.float32)
    a = rng.integers(0, k, n)
    b = (a + 1 + rng.integers(0, k - 1, n)) % k
    diff = P[a].astype(np.float64) - P[b]
    z = rng.standard_normal((n, d))
    z -= (z * diff).sum(1, keepdims=True) / (diff * diff).sum(1, keepdims=True) * diff
    X = ((P[a].astype(np.float64) + P[b]) / 2 + 0.05 * z).astype(np.float32)
    lab0, _, _ = mk.assign(torch.from_numpy(X).cuda(), torch.from_numpy(P).cuda(), flags=mk.MASK_NO_FIXUP)
    lab, d2, nf = mk.assign(torch.from_numpy(X).cuda(), torch.from_numpy(P).cuda())
    ref, b1, b2 = oracle.assign(X.astype(np.float64), P.astype(np.float64))
    got = lab.cpu().numpy(); g0 = lab0.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    print(f"d={d} bad={bad.size}; among bad: K1 label == final {np.sum(g0[bad]==got[bad])}; K1 label in (a,b): {np.sum((g0[bad]==a[bad])|(g0[bad]==b[bad]))}")
    print("  bad rows:", bad[:10].tolist(), "a:", a[bad[:10]].tolist(), "b:", b[bad[:10]].tolist(), "chunk a/32:", (a[bad[:10]]//32).tolist(), "chunk b/32:", (b[bad[:10]]//32).tolist())
