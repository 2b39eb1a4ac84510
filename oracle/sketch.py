"""Row sketch X = Gamma A (TEST INFRASTRUCTURE ONLY).

Paper: Algorithm 2 line 2 "Construct a row sketch X = Gamma A";
Table 1 for the cost model.  The oracle forms Gamma explicitly
(oracle.omega) and multiplies -- the definition written out, with the library
matmul as the one step (no blocking or reordering of the method).

Layout: A is an (m, n) float64 array; X is returned as an (l, n) array.
"""
import numpy as np

from . import omega


def sketch(A, l, kind="gaussian", seed=0, zeta=8):
    """X = Gamma A with Gamma from oracle.omega (P:176 / P:182)."""
    A = np.asarray(A, dtype=np.float64)
    m = A.shape[0]
    G = omega.embedding(kind, seed, l, m, zeta)
    return G @ A


def sketch_srtt_fft(A, l, seed=0):
    """SRTT sketch for larger m with the library FFT as the transform step (DHT = Re F - Im F of
    the DFT F, F(k) = sum_i y_i e^{-2 pi i ik/m}); otherwise the same formula as omega.srtt."""
    A = np.asarray(A, dtype=np.float64)
    m = A.shape[0]
    perm, signs, sel = omega.srtt_parts(seed, l, m)
    Y = signs[:, None] * A[perm]
    F = np.fft.fft(Y, axis=0)
    H = (F.real - F.imag) / np.sqrt(m)
    return np.sqrt(m / l) * H[sel]


def sketch_columns(A_cols, l, kind="gaussian", seed=0, zeta=8):
    """X[:, J] for a sample of columns A[:, J] (same Gamma; used for full-size spot checks)."""
    return sketch(A_cols, l, kind, seed, zeta)


def sketch_power(A, l, kind="gaussian", seed=0, q=1, zeta=8):
    """Row-space approximator with q plain power iterations, eq:def_power_iter:

        X = Omega (A^T A)^q,   Omega l x n drawn like Gamma (oracle.omega) over the n index.

    q = 0 is the row sketch X = Gamma A (Gamma l x m).  Written out literally: form the
    Gram matrix A^T A and apply it q times (the paper's O(T_s + (2q-1) nnz(A) l) evaluation
    order is the GPU's business; the value is the same)."""
    A = np.asarray(A, dtype=np.float64)
    if q == 0:
        return sketch(A, l, kind, seed, zeta)
    n = A.shape[1]
    X = omega.embedding(kind, seed, l, n, zeta)
    G = A.T @ A
    for _ in range(q):
        X = X @ G
    return X


def sketch_cols(A, l, kind="gaussian", seed=0, zeta=8):
    """Column sketch Y = A Omega^T of Algorithm 3 line 2, Omega l x n drawn like Gamma
    (oracle.omega) over the column index of A."""
    A = np.asarray(A, dtype=np.float64)
    Om = omega.embedding(kind, seed, l, A.shape[1], zeta)
    return A @ Om.T


def sketch_streamed(get_cols, m, n, l, kind="gaussian", seed=0, zeta=8, block=4096):
    """X = Gamma A for an A too large to hold at once (BASELINE C5, 68.7 GB): X = Gamma A is
    column-separable, X(:, J) = Gamma A(:, J), so A is taken in column blocks from
    get_cols(j0, j1) (an m x (j1 - j0) array) and each block is multiplied by the same explicit
    Gamma (oracle.omega).  The value is the definition's; only the column order of the work differs."""
    G = omega.embedding(kind, seed, l, m, zeta)
    X = np.empty((l, n))
    for j0 in range(0, n, block):
        j1 = min(n, j0 + block)
        X[:, j0:j1] = G @ np.asarray(get_cols(j0, j1), dtype=np.float64)
    return X


def ortho_pos(M):
    """ortho(M) as the Q factor of the thin QR with diag(R) > 0 -- the unique orthonormal basis
    whose Gram-Schmidt order matches M's columns (reading R21: the paper leaves the basis free)."""
    q, r = np.linalg.qr(np.asarray(M, dtype=np.float64), mode="reduced")
    d = np.sign(np.diag(r))
    d[d == 0] = 1.0
    return q * d


def sketch_power_ortho(A, l, kind="gaussian", seed=0, q=1, zeta=8):
    """Row-space approximator with q orthogonalised power iterations, eq:ortho_power_iter:

        Y(1) = A Omega^T;  Y(i) = ortho(A ortho(A^T Y(i-1))), i = 2..q;  X = ortho(Y(q))^T A,

    Omega l x n drawn like Gamma over the column index of A (as sketch_power), ortho = ortho_pos."""
    A = np.asarray(A, dtype=np.float64)
    n = A.shape[1]
    Om = omega.embedding(kind, seed, l, n, zeta)
    Y = A @ Om.T
    for _ in range(2, q + 1):
        Y = ortho_pos(A @ ortho_pos(A.T @ Y))
    return ortho_pos(Y).T @ A
