import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..', 'tests'))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..', '..'))
import numpy as np, torch
import datagen, oracle
import paper_2208_02734_b200 as mk
rp, col, val = datagen.random_csr(720, 4000, 300, 12)
rows = [(col[rp[i]:rp[i + 1]], val[rp[i]:rp[i + 1]]) for i in range(20)]
rows = [rows[i // 8] for i in range(160)] + [(col[rp[i]:rp[i + 1]], val[rp[i]:rp[i + 1]]) for i in range(160, 4000)]
rp2 = np.concatenate([[0], np.cumsum([len(c) for c, _ in rows])]).astype(np.int64)
col2 = np.concatenate([c for c, _ in rows]).astype(np.int32)
val2 = np.concatenate([v for _, v in rows]).astype(np.float32)
k = 48
init = [np.arange(k, dtype=np.int64)]
dev = "cuda"
data = mk.Csr(torch.from_numpy(rp2).to(dev), torch.from_numpy(col2).to(dev), torch.from_numpy(val2).to(dev), 300)
idx = mk.build(data, [k], 1, init, flags=mk.MASK_TRACE_PASSES, empty="farthest")
ref = oracle.lloyd((rp2, col2, val2), init[0], 1, csr_dim=300, trace=True, empty="farthest")
g = idx.passes(1)
print("npass", len(g), len(ref.passes))
print("labels0 equal", np.array_equal(g[0][1], ref.passes[0][1]))
P1g, P1o = g[1][0], ref.passes[1][0]
cnt = np.bincount(ref.passes[0][1], minlength=k)
D = np.zeros((4000, 300))
for i in range(4000):
    D[i, col2[rp2[i]:rp2[i + 1]]] = val2[rp2[i]:rp2[i + 1]]
for j in range(k):
    e = np.abs(P1g[j] - P1o[j]).max()
    if e > 1e-5:
        mg = np.nonzero((np.abs(D - P1g[j]).max(1) < 1e-6))[0][:3]
        mo = np.nonzero((np.abs(D - P1o[j]).max(1) < 1e-6))[0][:3]
        print(j, "count", cnt[j], "err", e, "gpu row", mg, "oracle row", mo, "gpu nnz", (P1g[j] != 0).sum())
lab = ref.passes[0][1]
P0 = ref.passes[0][0]
best = ((D - P0[lab]) ** 2).sum(1)
o = np.lexsort((np.arange(4000), -best))
print("oracle farthest", o[:10], best[o[:10]])
