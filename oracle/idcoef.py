"""Interpolative-decomposition coefficients and the Theorem 4.1 certificate (TEST INFRASTRUCTURE ONLY).

Paper:
  * eq:colID: A ~ C Z, C = A(:, J_s), Z in R^{k x n}.
  * classical ID form A Pi ~ (A Pi_1) [I_k, R11^{-1} R12].
  * Theorem 4.1: with X Pi = [X1, X2] (first k pivots),
    eta <= sqrt(1 + ||X1^+ X2||_2^2), computable a posteriori in O(l^2 (n - l)).
Reading (R10): Z is the sketch interpolation matrix
    Z(:, J_s) = I_k,  Z(:, rest) = T = X1^{-1} X2 = L1^{-T} L2^T
from the LUPP factors of X^T (rows 0..k-1 of X, R5): X^T(rest) = L2 U and
X^T(J_s) = L1 U give X1 = U^T L1^T, X2 = U^T L2^T, hence X1^{-1} X2 = L1^{-T} L2^T.
T is obtained by plain back substitution with the unit upper L1^T; the identity
block is assigned, not computed.
"""
import numpy as np


def id_coeffs(Lf, piv):
    """Return (Z, T, eta) from the LUPP factor Lf (n x k) and pivots."""
    Lf = np.asarray(Lf, dtype=np.float64)
    n, k = Lf.shape
    piv = np.asarray(piv, dtype=np.int64)
    rest = np.setdiff1d(np.arange(n), piv)          # ascending original order
    L1 = Lf[piv, :]                                   # k x k, unit lower triangular
    L2 = Lf[rest, :]                                  # (n - k) x k
    # Solve L1^T T = L2^T by back substitution (L1^T is unit upper triangular).
    B = L2.T.copy()                                   # k x (n - k)
    T = np.zeros_like(B)
    for t in range(k - 1, -1, -1):
        T[t] = B[t] - L1[t + 1:, t] @ T[t + 1:]
    Z = np.zeros((k, n))
    Z[:, piv] = np.eye(k)
    Z[:, rest] = T
    eta = float(np.sqrt(1.0 + np.linalg.norm(T, 2) ** 2)) if T.size else 1.0
    return Z, T, eta
