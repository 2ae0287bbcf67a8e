import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import datagen, oracle, paper_2208_02734_b200 as mk
cfg = datagen.CONFIGS[4] if len(sys.argv) < 2 else datagen.CONFIGS[4].scaled(int(sys.argv[1]))
rp, col, val = datagen.data(cfg)
inits = datagen.all_init_indices(cfg)
dev = "cuda:0"
T = lambda a: torch.from_numpy(a).to(dev)
idx = mk.build(mk.Csr(T(rp), T(col), T(val), cfg.dim), cfg.levels, 8, inits)
qrp, qcol, qval = datagen.queries(cfg, count=200)
ids, d2 = idx.query(mk.Csr(T(qrp), T(qcol), T(qval), cfg.dim), knn=10)
ids = ids.cpu().numpy(); d2 = d2.cpu().numpy()
L = len(cfg.levels)
P = [idx.prototypes(l).astype(np.float64) for l in range(1, L + 1)]
ch = [idx.children(l) for l in range(1, L + 1)]
rids, rd2, gap = oracle.query(P, [c[0] for c in ch], [c[1] for c in ch], (rp, col, val), (qrp, qcol, qval), 10, 1, dim=cfg.dim, x_csr=True, q_csr=True)
bad = np.nonzero(~np.all(ids == rids, axis=1) & (gap >= 1e-5))[0]
print("levels", cfg.levels, "bad", bad[:10], len(bad))
lab1 = idx.labels(1)
for q in bad[:3]:
    qd = np.zeros(cfg.dim); qd[qcol[qrp[q]:qrp[q+1]]] = qval[qrp[q]:qrp[q+1]]
    dtop = ((P[1] - qd) ** 2).sum(1)
    print("q", q, "gpu ids", ids[q][:4], "ref", rids[q][:4], "gpu d2", d2[q][:3], "ref d2", rd2[q][:3])
    print("  gpu leaf protos", set(lab1[ids[q][ids[q]>=0]].tolist()), "ref leaf protos", set(lab1[rids[q][rids[q]>=0]].tolist()))
    o = np.argsort(dtop)[:3]; print("  top-level best", o, dtop[o])
for q in bad[:2]:
    print("q", q)
    print(" gpu", list(zip(ids[q].tolist(), np.round(d2[q], 7).tolist())))
    print(" ref", list(zip(rids[q].tolist(), np.round(rd2[q], 7).tolist())))
    print(" gap", gap[q])
    qd = np.zeros(cfg.dim); qd[qcol[qrp[q]:qrp[q+1]]] = qval[qrp[q]:qrp[q+1]]
    for i in set(ids[q].tolist()) ^ set(rids[q].tolist()):
        xd = np.zeros(cfg.dim); xd[col[rp[i]:rp[i+1]]] = val[rp[i]:rp[i+1]]
        print("  id", i, "exact d2", ((xd - qd) ** 2).sum(), "nnz", rp[i+1]-rp[i], "label1", lab1[i])
