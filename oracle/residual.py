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


def residual_col_id_streamed(get_cols, m, n, Js, block=4096):
    """(||A - Q_C Q_C^T A||_F, ||A||_F) of the column ID (eq:def_column_id) for an A taken
    in column blocks from get_cols(j0, j1): C = A(:, J_s) is gathered first, Q_C = ortho(C) (the one
    library step), then for every column block the residual block A_b - Q_C (Q_C^T A_b) is formed
    explicitly and squared.  ||E||_F^2 is the sum over columns, so the result is the definition's
    (BASELINE C5, which does not fit in host memory at once)."""
    Js = np.asarray(Js, dtype=np.int64)
    C = np.empty((m, Js.size))
    for t, j in enumerate(Js):
        C[:, t] = np.asarray(get_cols(int(j), int(j) + 1), dtype=np.float64)[:, 0]
    Qc = ortho(C)
    del C
    r2 = a2 = 0.0
    for j0 in range(0, n, block):
        j1 = min(n, j0 + block)
        Ab = np.asarray(get_cols(j0, j1), dtype=np.float64)
        E = Ab - Qc @ (Qc.T @ Ab)
        r2 += float(np.sum(E * E))
        a2 += float(np.sum(Ab * Ab))
    return float(np.sqrt(r2)), float(np.sqrt(a2))
