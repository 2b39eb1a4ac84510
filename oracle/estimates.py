"""Sketch-only ID / CUR estimates of Algorithm 3 (TEST INFRASTRUCTURE ONLY).

Paper, after Algorithm 3: without revisiting A beyond the skeletons,
    C^+ A  ~  X_1^+ X,      A R^+  ~  Y Y_1^+,
with X_1 = X(:, J_s) and Y_1 = Y(I_s, :) the column / row pivots of the row sketch X = Gamma A
and the column sketch Y = A Omega^T; and the CUR C S^{-1} R with S = A(I_s, J_s), C = A(:, J_s),
R = A(I_s, :).  Each is the definition written out, with a library least-squares / linear solve
as the one step.
"""
import numpy as np


def id_estimate_cols(X, Js):
    """Z = X_1^+ X (k x n)."""
    X = np.asarray(X, dtype=np.float64)
    return np.linalg.lstsq(X[:, Js], X, rcond=None)[0]


def id_estimate_rows(Y, Is):
    """W = Y Y_1^+ (m x k):  Y_1^+ = pinv(Y(I_s, :)), via the least-squares problem Y_1^T W^T = Y^T."""
    Y = np.asarray(Y, dtype=np.float64)
    return np.linalg.lstsq(Y[Is, :].T, Y.T, rcond=None)[0].T


def cur_css(A, Is, Js):
    """C S^{-1} R."""
    A = np.asarray(A, dtype=np.float64)
    S = A[np.ix_(Is, Js)]
    return A[:, Js] @ np.linalg.solve(S, A[Is, :])
