"""Parity criteria of BASELINE.json north_star, made operational.

* Assignments: identical except rows whose oracle best and second-best squared distances
  differ by less than 1e-5 relative (D10: (d2 - d1) < 1e-5 * d2 on FP64 squared distances);
  for those exempt rows the oracle distance of the GPU's label must be <= d1 * (1 + 1e-5).
* Prototypes: within 1e-4 relative L2 (Frobenius) error per level.
* Queries: identical (d^2, id)-ordered result sets except queries whose oracle selections
  had a competing candidate within 1e-5 relative (counted, not silently passed).
"""
from __future__ import annotations

import numpy as np

import oracle

TIE_REL = 1e-5
PROTO_REL = 1e-4


def check_assignment(Y, P, labels_gpu, d2_gpu=None, what=""):
    """Compare GPU labels with the oracle's assignment of the same rows to the same P."""
    Y = np.asarray(Y, np.float64)
    P = np.asarray(P, np.float64)
    lab, b1, b2 = oracle.assign(Y, P)
    labels_gpu = np.asarray(labels_gpu).astype(np.int64)
    assert labels_gpu.min() >= 0 and labels_gpu.max() < P.shape[0], f"{what}: label out of range"
    exempt = (b2 - b1) < TIE_REL * b2
    bad = (labels_gpu != lab) & ~exempt
    assert not bad.any(), (f"{what}: {int(bad.sum())} non-exempt label mismatches of {len(lab)} "
                           f"(first rows {np.nonzero(bad)[0][:5].tolist()})")
    diff = labels_gpu != lab
    if diff.any():
        rows = np.nonzero(diff)[0]
        dg = ((Y[rows] - P[labels_gpu[rows]]) ** 2).sum(axis=1)
        assert np.all(dg <= b1[rows] * (1 + TIE_REL) + 1e-300), f"{what}: exempt row label not within window"
    if d2_gpu is not None:
        d2_gpu = np.asarray(d2_gpu, np.float64)
        ref = ((Y - P[labels_gpu]) ** 2).sum(axis=1)
        err = np.abs(d2_gpu - ref)
        # FP32 value of a squared distance: 1e-5 of itself, plus (expanded form, tensor path)
        # the worst-case 3xTF32 error of ||c||^2 - 2 x.c relative to the magnitudes that
        # cancel in it: (2^-20 + 3 ceil(d/8) 2^-24 + 2^-23) (||x||^2 + ||c||^2)  (K1)
        d = Y.shape[1]
        coef = 2.0 ** -20 + 3 * np.ceil(d / 8) * 2.0 ** -24 + 2.0 ** -23
        allow = 1e-5 * ref + coef * ((Y ** 2).sum(axis=1) + (P[labels_gpu] ** 2).sum(axis=1)) + 1e-30
        assert np.all(err <= allow), f"{what}: d2 max err/allow {float((err / allow).max())}"
    return int(diff.sum()), int(exempt.sum())


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def check_prototypes(P_gpu, P_ref, what=""):
    e = rel_l2(P_gpu, P_ref)
    assert e <= PROTO_REL, f"{what}: prototype rel L2 error {e:.3e} > {PROTO_REL}"
    return e


def check_queries(ids_gpu, d2_gpu, ids_ref, d2_ref, gap_ref, what=""):
    """Identical result lists except queries exempt by the oracle's tie window."""
    ids_gpu = np.asarray(ids_gpu)
    exempt = gap_ref < TIE_REL
    same = np.all(ids_gpu == ids_ref, axis=1)
    # the same result set whose order differs only inside groups of (near-)equal distances
    # (adjacent oracle d^2 within 1e-5 relative: the (d^2, id) order of a tie is not decided by
    # FP32 vs FP64 rounding) counts as identical
    for q in np.nonzero(~same)[0]:
        a, b = ids_gpu[q], ids_ref[q]
        if set(a.tolist()) != set(b.tolist()):
            continue
        dref = {int(i): float(v) for i, v in zip(b, d2_ref[q]) if i >= 0}
        da = np.array([dref[int(i)] for i in a if i >= 0])
        pad_ok = np.all(a[len(da):] < 0)  # padding only at the tail
        order_ok = pad_ok and np.all(np.diff(da) >= -TIE_REL * np.maximum(np.abs(da[1:]), 1e-30))
        if order_ok:
            same[q] = True
    bad = ~same & ~exempt
    assert not bad.any(), (f"{what}: {int(bad.sum())} non-exempt query mismatches of {len(same)} "
                           f"(first {np.nonzero(bad)[0][:5].tolist()})")
    ok = same
    fin = np.isfinite(d2_ref[ok])
    if fin.any():
        a = np.asarray(d2_gpu, np.float64)[ok][fin]
        b = d2_ref[ok][fin]
        assert np.all(np.abs(a - b) <= 1e-4 * np.maximum(b, 1e-6) + 1e-6), f"{what}: d2 mismatch"
    pad_gpu = ids_gpu < 0
    assert np.all(np.isinf(np.asarray(d2_gpu)[pad_gpu])), f"{what}: padding must carry +inf"
    return int((~same).sum()), int(exempt.sum())


def _rows_d2(Y, P, rows, labels, csr_dim):
    """FP64 ||y_i - P[labels_i]||^2 for the given rows (dense, or CSR (rp, col, val) through
    ||c||^2 + sum_nz (y^2 - 2 y c), the oracle's D12 form)."""
    P = np.asarray(P, np.float64)
    rows = np.asarray(rows, np.int64)
    lab = np.asarray(labels, np.int64)
    if csr_dim is None:
        Y = np.asarray(Y, np.float64)
        return ((Y[rows] - P[lab]) ** 2).sum(axis=1)
    rp, col, val = Y
    cnt = rp[rows + 1] - rp[rows]
    pos = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows]) if rows.size else np.zeros(0, np.int64)
    owner = np.repeat(np.arange(rows.size), cnt)
    v = np.asarray(val, np.float64)[pos]
    c = P[lab[owner], np.asarray(col)[pos]]
    part = np.zeros(rows.size)
    np.add.at(part, owner, v * v - 2.0 * v * c)
    return (P[lab] ** 2).sum(axis=1) + part


def _assign_any(Y, P, csr_dim):
    if csr_dim is None:
        return oracle.assign(Y, P)
    return oracle.assign_csr(Y, csr_dim, P)


def _means_any(Y, labels, P_old, csr_dim):
    if csr_dim is None:
        return oracle.means(np.asarray(Y, np.float64), labels, P_old)[0]
    S, cnt = oracle.cluster_sums_csr(Y, csr_dim, labels, P_old.shape[0])
    return oracle.means_from_sums(S, cnt, P_old)[0]


def check_assignment_any(Y, P, labels, csr_dim=None, what=""):
    """check_assignment for dense or CSR (rp, col, val) level inputs."""
    lab, b1, b2 = _assign_any(Y, np.asarray(P, np.float64), csr_dim)
    labels = np.asarray(labels).astype(np.int64)
    exempt = (b2 - b1) < TIE_REL * b2
    bad = (labels != lab) & ~exempt
    assert not bad.any(), (f"{what}: {int(bad.sum())} non-exempt label mismatches of {len(lab)} "
                           f"(first rows {np.nonzero(bad)[0][:5].tolist()})")
    diff = np.nonzero(labels != lab)[0]
    if diff.size:
        # the oracle distance of the GPU's label is within the window of the best one
        dg = _rows_d2(Y, P, diff, labels[diff], csr_dim)
        assert np.all(dg <= b1[diff] * (1 + TIE_REL) + 1e-300), f"{what}: exempt row label not within window"
    return int(diff.size), int(exempt.sum())


def check_trajectory(Y, gpu, ref, csr_dim=None, what=""):
    """End-to-end parity of one level's Lloyd run (BASELINE north_star; D15).

    gpu / ref: the per-pass sequences [(P_t, labels_t), ...] (P_t = the prototypes assignment
    pass t used; the last entry is the final assignment) of the production GPU build
    (MASK_TRACE_PASSES, no iteration callback, so every kernel choice is the bench's) and of the
    FP64 oracle (oracle.lloyd(trace=True)) from the same level input and init rows.

    * While the two label sequences agree pass for pass, the prototypes each pass used agree
      within PROTO_REL (1e-4 relative L2).  If they agree to the end, the final prototypes agree
      within 1e-4: plain end-to-end parity.
    * At the first pass t where they differ, every differing row must be inside the oracle's own
      tie window at the oracle's P_t ((d2 - d1) < 1e-5 d2, the GPU's label within the window of
      the best distance): the trajectories part at a legitimate near-tie decision, after which
      each is a valid Lloyd run of its own.  From t on every GPU pass is checked in step mode
      against its own P_t (assignment in the tie window; the next P = FP64 member means).

    Returns a report dict (diverged_at, flipped rows, final errors and objectives)."""
    assert len(gpu) >= 1 and len(ref) >= 1
    t_div = None
    flipped = 0
    for t in range(min(len(gpu), len(ref))):
        Pg, lg = gpu[t]
        Po, lo = ref[t]
        e = rel_l2(Pg, Po)
        assert e <= PROTO_REL, f"{what}: pass {t} (labels in sync so far) prototype rel L2 error {e:.3e}"
        if np.array_equal(np.asarray(lg), np.asarray(lo)):
            continue
        t_div = t
        flipped, _ = check_assignment_any(Y, Po, lg, csr_dim, what=f"{what}: first differing pass {t} vs the oracle's P_t")
        break
    if t_div is None:
        # in sync through the shorter run: the no-change stop rule then ends both identically
        assert len(gpu) == len(ref), f"{what}: labels in sync but pass counts differ ({len(gpu)} vs {len(ref)})"
    else:
        for t in range(t_div, len(gpu)):
            Pg, lg = gpu[t]
            check_assignment_any(Y, Pg, lg, csr_dim, what=f"{what}: step pass {t}")
            if t + 1 < len(gpu) and not np.array_equal(gpu[t + 1][0], Pg):
                P_ref = _means_any(Y, np.asarray(lg, np.int32), np.asarray(Pg, np.float64), csr_dim)
                check_prototypes(gpu[t + 1][0], P_ref, what=f"{what}: step update after pass {t}")
    final_err = rel_l2(gpu[-1][0], ref[-1][0])
    if t_div is None:
        assert final_err <= PROTO_REL, f"{what}: final prototype rel L2 error {final_err:.3e}"
    n = len(gpu[-1][1])
    allrows = np.arange(n)
    Jg = float(_rows_d2(Y, gpu[-1][0], allrows, gpu[-1][1], csr_dim).sum())
    Jo = float(_rows_d2(Y, ref[-1][0], allrows, ref[-1][1], csr_dim).sum())
    return dict(what=what, passes_gpu=len(gpu), passes_oracle=len(ref), diverged_at=t_div,
                flipped_rows=flipped, final_rel_l2=final_err, J_gpu=Jg, J_oracle=Jo)
