"""Frobenius residuals of the skeleton approximations (TEST INFRASTRUCTURE ONLY).

Paper:
  * column ID  CC^+A            eq:def_column_id
  * row ID     AR^+R            eq:def_row_id
  * CUR        C(C^+AR^+)R      eq:def_cur, formed stably as
               Q_C (Q_C^T A Q_R) Q_R^T with Q_C = ortho(C), Q_R = ortho(R^T)
               (Remark 2.3, eq:cur_stable; protocol P:554)
  * ID coeffs  C Z              eq:colID
ortho(M) is taken from the library Householder QR (numpy.linalg.qr), the
one library step; the residual A - (approximation) is then formed explicitly and
its Frobenius norm taken -- never the Pythagorean shortcut (R11).
Norm: Frobenius only (R12).
"""
import numpy as np


def ortho(M):
    """An orthonormal basis of range(M)."""
    q, _ = np.linalg.qr(np.asarray(M, dtype=np.float64), mode="reduced")
    return q


def residual(A, Js=None, Is=None, kind="col_id", Z=None):
    """Return (||A - approx||_F, ||A||_F)."""
    A = np.asarray(A, dtype=np.float64)
    nA = float(np.linalg.norm(A))
    if kind == "col_id":
        Qc = ortho(A[:, Js])
        E = A - Qc @ (Qc.T @ A)
    elif kind == "row_id":
        Qr = ortho(A[Is, :].T)
        E = A - (A @ Qr) @ Qr.T
    elif kind == "cur":
        Qc = ortho(A[:, Js])
        Qr = ortho(A[Is, :].T)
        Mid = Qc.T @ A @ Qr
        E = A - Qc @ Mid @ Qr.T
    elif kind == "id_coeffs":
        E = A - A[:, Js] @ Z
    else:
        raise ValueError(kind)
    return float(np.linalg.norm(E)), nA


def optimal_error(sigma, k):
    """||A - A_k||_F = sqrt(sum_{i>k} sigma_i^2) (Eckart-Young)."""
    s = np.sort(np.asarray(sigma, dtype=np.float64))[::-1]
    return float(np.sqrt(np.sum(s[k:] ** 2)))
