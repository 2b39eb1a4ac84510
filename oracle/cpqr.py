"""Column-pivoted Householder QR on the sketch (TEST INFRASTRUCTURE ONLY).

Paper: eq:def_QRCP:  X Pi_n = Q_l [R1 R2];  at step t+1 the pivot is
    j_{t+1} = argmax_j || X^{(t)}(t+1:l, j) ||_2
over the ENTIRE active submatrix (all remaining rows of the sketch), followed by
a Householder (rank-1) orthogonal update (Trefethen-Bau Alg. 10.1).
This is the "Rand-CPQR" comparison of Section 5 (Voronin-Martinsson).

Readings: R6 ties -> lowest original index; R9 the remaining
column norms are recomputed exactly each step (no downdating); a maximal
remaining norm <= 1e-14 ||X||_F is a rank failure.

Returns (piv, R) with R (k x n): R[t, j] is row t of the triangular factor for
original column j (R[t, piv[t']] = 0 for t' < t).
"""
import numpy as np

from .lupp import RankError

RANK_TOL = 1e-14


def select_cols_cpqr(X, k):
    W = np.array(X, dtype=np.float64, copy=True)
    l, n = W.shape
    if k > min(l, n):
        raise ValueError("k <= min(l, n) required")
    fro = np.sqrt(np.sum(W * W))
    active = np.ones(n, dtype=bool)
    piv = np.empty(k, dtype=np.int64)
    R = np.zeros((k, n))
    for t in range(k):
        norms = np.sqrt(np.sum(W[t:, :] ** 2, axis=0))
        cand = np.where(active, norms, -1.0)
        p = int(np.argmax(cand))
        if not (cand[p] > RANK_TOL * fro):
            raise RankError(t + 1)
        x = W[t:, p].copy()
        nx = np.sqrt(np.sum(x * x))
        alpha = -nx if x[0] >= 0 else nx
        v = x.copy()
        v[0] -= alpha
        vv = np.sum(v * v)
        cols = np.nonzero(active)[0]
        if vv > 0:
            W[t:, cols] -= np.outer(v, (2.0 / vv) * (v @ W[t:, cols]))
        W[t:, p] = 0.0
        W[t, p] = alpha
        R[t, cols] = W[t, cols]
        piv[t] = p
        active[p] = False
    return piv, R
