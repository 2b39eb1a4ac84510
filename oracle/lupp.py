"""Column-wise / row-wise LU with partial pivoting for skeleton selection (TEST INFRASTRUCTURE ONLY).

Paper: eq:def_LUPP and the pivot rule, P:270-284:
    X Pi_n = L_l [R1 R2], R1 unit upper, |R(i,j)| <= 1;
    step t+1 searches only row t+1 of the active submatrix,
        j_{t+1} = argmax_j |X^{(t)}(t+1, j)|,
    and updates the active submatrix by the Schur complement
        X^{(t+1)} = X^{(t)} - X^{(t)}(:, t) X^{(t)}(t, :) / X^{(t)}(t, t).
Algorithm 2 lines 3-4: column LUPP on X picks J_s; row LUPP on
C = A(:, J_s) picks I_s.  The introduction's "partially pivoted LU of Y^*"
 is the same computation stated on the transpose, which is the form used
here: M = X^T (n x k), pivot over rows of M, step t scans column t.

Readings: R5 -- J_s is the first k pivots; only rows 0..k-1 of X
enter (the first k LUPP steps never look at rows >= k).  R6 -- ties go to the
lowest ORIGINAL index (no physical swaps).  R7 -- a pivot with
|a| <= 1e-14 * max|panel| is a rank failure (SK_E_RANK, 1-based step).
R8 -- row LUPP on C scans column t of C at step t, with C's columns in J_s pivot
order (MATLAB lu(...,'vector') semantics).

Outputs follow include/skel.h: Lf (n x k) with Lf[i, t] the multiplier of row i
at step t, Lf[p_t, t] = 1 and Lf[p_t, t'] = 0 for t' > t; U (k x k) upper with
U[t, t:] the pivot row at step t; gaps[t] = (a1 - a2) / a1 for the two largest
candidate magnitudes at step t.
"""
import ctypes
import os
import subprocess

import numpy as np

RANK_TOL = 1e-14
_HERE = os.path.dirname(os.path.abspath(__file__))
_CLIB = None


class RankError(Exception):
    def __init__(self, step):
        super().__init__(f"LUPP: zero pivot at step {step} (1-based)")
        self.step = step


def lupp_panel(M, k, forced=None):
    """k-step swap-free LUPP on the rows of M (n x >=k).  Returns (piv, Lf, U, gaps).

    forced: optional {step: row} overriding the argmax at that step (used by the
    parity harness to follow the GPU through a documented near-tie).
    """
    M = np.array(M, dtype=np.float64, copy=True)
    n = M.shape[0]
    if k > M.shape[1] or k > n:
        raise ValueError("LUPP needs k <= min(n, panel width)")
    W = M[:, :k].copy()
    scale = np.max(np.abs(W)) if W.size else 0.0
    active = np.ones(n, dtype=bool)
    Lf = np.zeros((n, k))
    U = np.zeros((k, k))
    piv = np.empty(k, dtype=np.int64)
    gaps = np.zeros(k)
    for t in range(k):
        a = np.where(active, np.abs(W[:, t]), -1.0)
        p = int(np.argmax(a))                       # first maximum = lowest original index
        a1 = a[p]
        a_rest = np.where(np.arange(n) == p, -1.0, a)
        a2 = max(float(np.max(a_rest)), 0.0) if n > 1 else 0.0
        gaps[t] = (a1 - a2) / a1 if a1 > 0 else 0.0
        if forced is not None and t in forced:
            p = int(forced[t])
            assert active[p], "forced pivot must be active"
            a1 = abs(W[p, t])
        if not (a1 > RANK_TOL * scale):
            raise RankError(t + 1)
        piv[t] = p
        U[t, t:] = W[p, t:]
        active[p] = False
        Lf[p, t] = 1.0
        rows = np.nonzero(active)[0]
        mult = W[rows, t] / W[p, t]
        Lf[rows, t] = mult
        W[rows, t + 1:] -= np.outer(mult, U[t, t + 1:])
    return piv, Lf, U, gaps


def build_c(force=False):
    """Compile oracle/c/lupp.c (plain C + OpenMP, -ffp-contract=off) to oracle/c/liboracle_lupp.so."""
    src = os.path.join(_HERE, "c", "lupp.c")
    so = os.path.join(_HERE, "c", "liboracle_lupp.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared", src, "-o", so + ".tmp"],
                       check=True)
        os.replace(so + ".tmp", so)
    return so


def _clib():
    global _CLIB
    if _CLIB is None:
        lib = ctypes.CDLL(build_c())
        lib.or_lupp_panel.restype = ctypes.c_int64
        P = ctypes.c_void_p
        lib.or_lupp_panel.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, P, P, P, P, P]
        _CLIB = lib
    return _CLIB


def lupp_panel_c(M, k, forced=None):
    """lupp_panel in plain C (oracle/c/lupp.c): the same steps and the same rounding, for panels
    too large for the numpy loop (tests/test_oracle_path.py checks the two agree bit for bit)."""
    n = M.shape[0]
    if k > M.shape[1] or k > n:
        raise ValueError("LUPP needs k <= min(n, panel width)")
    W = np.ascontiguousarray(np.asarray(M, dtype=np.float64)[:, :k]).copy()
    piv = np.zeros(k, dtype=np.int64)
    Lf = np.zeros((n, k))
    U = np.zeros((k, k))
    gaps = np.zeros(k)
    act = np.zeros(n, dtype=np.uint8)
    fz = None
    if forced:
        fz = np.full(k, -1, dtype=np.int64)
        for t, p in forced.items():
            fz[t] = p
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p) if a is not None else None  # noqa: E731
    st = _clib().or_lupp_panel(ptr(W), n, k, ptr(fz), ptr(piv), ptr(Lf), ptr(U), ptr(gaps), ptr(act))
    if st:
        raise RankError(int(st))
    return piv, Lf, U, gaps


def _panel(M, k, forced, fast):
    return lupp_panel_c(M, k, forced) if fast else lupp_panel(M, k, forced)


def select_cols(X, k, forced=None, fast=False):
    """J_s by column-wise LUPP on the sketch X (l x n), Algorithm 2 line 3.
    fast=True runs the same algorithm in plain C (lupp_panel_c)."""
    X = np.asarray(X, dtype=np.float64)
    if k > X.shape[0]:
        raise ValueError("k <= l required")
    return _panel(X[:k, :].T, k, forced, fast)


def select_rows(C, k, forced=None, fast=False):
    """I_s by row-wise LUPP on C = A(:, J_s) (m x k), Algorithm 2 line 4."""
    return _panel(np.asarray(C, dtype=np.float64), k, forced, fast)


def growth(Lf, piv):
    """max |(R1^{-1} R2)_{ij}| of Lemma 2, via a library solve (test helper)."""
    n, k = Lf.shape
    rest = np.setdiff1d(np.arange(n), piv)
    L1 = Lf[piv, :]
    L2 = Lf[rest, :]
    T = np.linalg.solve(L1.T, L2.T)
    return np.max(np.abs(T), axis=1) if T.size else np.zeros(k)
