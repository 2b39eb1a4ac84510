"""The column-sharded LUPP pivot search, emulated on one host (TEST INFRASTRUCTURE ONLY).

SURVEY.md 8(e): with A (hence X = Gamma A, hence the LUPP panel M = X(0:k, :)^T) split by
column blocks over P ranks, step t of column-wise LUPP (eq:def_LUPP) becomes
  1. every rank proposes its best active row: (|M_r(i, t)|, global index i);
  2. the merge rule picks max |value|, ties -> lowest GLOBAL index (R6);
  3. the winning row (the pivot row U(t, t:)) is broadcast; every rank eliminates its own
     active rows with it (the Schur update of P:278).
This module runs that protocol over a list of per-rank panels with plain loops, so the merge
rule can be checked against single-process LUPP (oracle.lupp): with the lowest-original-index
tie rule the two are the same algorithm, step for step and bit for bit.
"""
import numpy as np

from .lupp import RANK_TOL, RankError


def select_cols_sharded(X_blocks, k):
    """X_blocks: list of (l x n_r) sketch blocks in rank order.  Returns (piv, Lf, U)."""
    panels = [np.array(Xr[:k, :].T, dtype=np.float64) for Xr in X_blocks]   # n_r x k, rows of M
    offs = np.cumsum([0] + [p.shape[0] for p in panels])
    n = int(offs[-1])
    scale = max((float(np.max(np.abs(p))) for p in panels if p.size), default=0.0)
    active = [np.ones(p.shape[0], dtype=bool) for p in panels]
    Lf = [np.zeros((p.shape[0], k)) for p in panels]
    U = np.zeros((k, k))
    piv = np.empty(k, dtype=np.int64)
    for t in range(k):
        # 1. per-rank proposals (first maximum within a rank = its lowest index)
        props = []
        for r, p in enumerate(panels):
            a = np.where(active[r], np.abs(p[:, t]), -1.0)
            if a.size and a.max() >= 0.0:
                i = int(np.argmax(a))
                props.append((float(a[i]), int(offs[r] + i), r, i))
        # 2. merge: max |value|, ties -> lowest global index
        best = None
        for prop in props:
            if best is None or prop[0] > best[0] or (prop[0] == best[0] and prop[1] < best[1]):
                best = prop
        if best is None or not (best[0] > RANK_TOL * scale):
            raise RankError(t + 1)
        _, g, rw, iw = best
        piv[t] = g
        urow = panels[rw][iw, t:].copy()                                   # 3. broadcast pivot row
        U[t, t:] = urow
        active[rw][iw] = False
        Lf[rw][iw, t] = 1.0
        for r, p in enumerate(panels):
            rows = np.nonzero(active[r])[0]
            mult = p[rows, t] / urow[0]
            Lf[r][rows, t] = mult
            p[rows, t + 1:] -= np.outer(mult, urow[1:])
    if n < k:
        raise ValueError("k <= n required")
    return piv, np.vstack(Lf), U
