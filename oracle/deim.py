"""RSVD-DEIM column skeletons, the paper's pivoting comparator (TEST INFRASTRUCTURE ONLY).

Paper: eq:rsvd_procedures: with Q_X an orthonormal basis of the row space of the
sketch X (n x l), svd(A Q_X, 'econ') = U^ S^ V~^T and V^ = Q_X V~; DEIM (Sorensen-Embree,
P:241-243, Sec. 5 item 3 P:529) selects the column skeletons by LU with partial pivoting on the
leading k right singular vectors V^(:, 0:k)^T -- the same swap-free LUPP as oracle.lupp, here on
the rows of the n x k panel V^(:, 0:k).  Library QR / SVD are the steps' primitives.
"""
import numpy as np

from .lupp import lupp_panel


def rsvd_vectors(A, X):
    """V^ (n x l) of eq:rsvd_procedures."""
    A = np.asarray(A, dtype=np.float64)
    Q, _ = np.linalg.qr(np.asarray(X, dtype=np.float64).T, mode="reduced")
    _, _, Vt = np.linalg.svd(A @ Q, full_matrices=False)
    return Q @ Vt.T


def select_cols_deim(A, X, k):
    """J_s (pivot order) by DEIM on the leading k right singular vectors of the RSVD."""
    V = rsvd_vectors(A, X)
    piv, _, _, _ = lupp_panel(V[:, :k], k)
    return piv
