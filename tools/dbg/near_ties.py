import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, paper_2208_02734_b200 as mk
for d in (16, 32, 64, 128):
    rng = np.random.default_rng(d)
    k, n = 300, 4096
    P = (rng.standard_normal((k, d)) * 4.0).astype(np.float32)
    a = rng.integers(0, k, n)
    b = (a + 1 + rng.integers(0, k - 1, n)) % k
    diff = P[a].astype(np.float64) - P[b]
    z = rng.standard_normal((n, d))
    z -= (z * diff).sum(1, keepdims=True) / (diff * diff).sum(1, keepdims=True) * diff
    X = ((P[a].astype(np.float64) + P[b]) / 2 + 0.05 * z).astype(np.float32)
    for flags in (0, mk.MASK_NO_FIXUP):
        lab, d2, nf = mk.assign(torch.from_numpy(X).cuda(), torch.from_numpy(P).cuda(), flags=flags)
        ref, b1, b2 = oracle.assign(X.astype(np.float64), P.astype(np.float64))
        got = lab.cpu().numpy()
        bad = np.nonzero(got != ref)[0]
        D = ((X[bad, None, :].astype(np.float64) - P[None].astype(np.float64)) ** 2).sum(-1)
        srt = np.sort(D, axis=1)
        print(f"d={d} flags={flags} flagged={nf} bad={bad.size}")
        for r in bad[:6]:
            print("   row", r, "gpu", got[r], "ref", ref[r], "a,b", a[r], b[r], "d(gpu)", D[list(bad).index(r), got[r]], "b1", b1[r], "b2", b2[r], "3rd", srt[list(bad).index(r), 2])
