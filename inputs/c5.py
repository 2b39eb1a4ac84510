"""C5 (BASELINE.json configs[4]): A = U diag(sigma) V^T, 131072 x 65536 FP64 (68.7 GB),
sigma_i = i^-1.5, U and V products of b = 64 Householder reflectors (R17).

    U = H_1 H_2 ... H_b,  H_a = I - 2 y_a y_a^T (unit y_a, Gaussian from the seed);  V likewise (y'_a).

Nothing here implements the method: this module only produces the synthetic input, two ways.
* ``build_on_device`` (the path the GPU runs on): compact WY, U = I - Y T Y^T with T upper
  triangular (Schreiber-Van Loan), so A = E - Y W - Z Y'^T with E = diag(sigma) (m x n),
  W = T (Y^T E) - (T (Y^T E Y') T'^T) Y'^T (b x n) and Z = (E Y') T'^T (m x b): one rank-2b
  product per column block, built with torch matmuls (input generation, not the hot path).
* ``column_by_reflectors`` (the check): A(:, j) = H_1(H_2(...H_b(E (H'_b(...H'_1 e_j))))), the
  definition applied reflector by reflector in numpy -- independent of the WY algebra.
"""
import numpy as np

M5, N5, B5 = 131072, 65536, 64


def factors(seed=1005, m=M5, n=N5, b=B5):
    """(Y m x b, Yp n x b) unit Gaussian reflector vectors and sigma (length n)."""
    rng = np.random.default_rng(seed)
    Y = rng.standard_normal((m, b))
    Y /= np.linalg.norm(Y, axis=0)
    Yp = rng.standard_normal((n, b))
    Yp /= np.linalg.norm(Yp, axis=0)
    sigma = np.arange(1, n + 1, dtype=np.float64) ** -1.5
    return Y, Yp, sigma


def wy_t(Y):
    """T (b x b upper) with H_1 ... H_b = I - Y T Y^T for H_a = I - 2 y_a y_a^T (unit y_a)."""
    b = Y.shape[1]
    G = Y.T @ Y
    T = np.zeros((b, b))
    for a in range(b):
        T[a, a] = 2.0
        if a:
            T[:a, a] = -2.0 * (T[:a, :a] @ G[:a, a])
    return T


def wy_operands(Y, Yp, sigma):
    """(W b x n, Z m x b) of A = E - Y W - Z Y'^T."""
    m, b = Y.shape
    n = Yp.shape[0]
    T, Tp = wy_t(Y), wy_t(Yp)
    P = (Y[:n] * sigma[:, None]).T                      # Y^T E     (b x n)
    S = P @ Yp                                           # Y^T E Y'  (b x b)
    W = T @ P - (T @ S @ Tp.T) @ Yp.T                    # b x n
    Q = np.zeros((m, b))
    Q[:n] = Yp * sigma[:, None]                          # E Y'      (m x b)
    Z = Q @ Tp.T
    return W, Z


def build_on_device(device, seed=1005, m=M5, n=N5, b=B5, col_block=4096, factors_out=None, col0=0, ncols=None):
    """A(:, col0 : col0 + ncols) (default: all n columns) as a column-major float64 CUDA tensor
    (A.t() contiguous), plus sigma (all n).  The column block is what one rank of the column-sharded
    multi-GPU path holds.  factors_out: optional list that receives (Y, Yp) for checks."""
    import torch
    ncols = n - col0 if ncols is None else ncols
    Y, Yp, sigma = factors(seed, m, n, b)
    if factors_out is not None:
        factors_out.extend([Y, Yp])
    W, Z = wy_operands(Y, Yp, sigma)
    Yd = torch.from_numpy(Y).to(device)
    Zd = torch.from_numpy(Z).to(device)
    Wd = torch.from_numpy(W).to(device)
    Ypd = torch.from_numpy(Yp).to(device)
    sd = torch.from_numpy(sigma).to(device)
    At = torch.empty((ncols, m), dtype=torch.float64, device=device)   # rows of At = columns of A
    for j0 in range(col0, col0 + ncols, col_block):
        j1 = min(col0 + ncols, j0 + col_block)
        blk = -(Yd @ Wd[:, j0:j1]) - Zd @ Ypd[j0:j1].T                # m x (j1 - j0)
        idx = torch.arange(j0, j1, device=device)
        blk[idx, idx - j0] += sd[j0:j1]
        At[j0 - col0:j1 - col0] = blk.t()
        del blk
    return At.t(), sigma


def build_block_host(j0, j1, seed=1005, m=M5, n=N5, b=B5, cache={}):
    """A(:, j0:j1) in host memory (numpy), the same compact-WY formula as build_on_device: for the
    CPU-only reference arm, which must not touch the GPU."""
    key = (seed, m, n, b)
    if key not in cache:
        Y, Yp, sigma = factors(seed, m, n, b)
        W, Z = wy_operands(Y, Yp, sigma)
        cache.clear()
        cache[key] = (Y, Yp, sigma, W, Z)
    Y, Yp, sigma, W, Z = cache[key]
    blk = -(Y @ W[:, j0:j1]) - Z @ Yp[j0:j1].T
    idx = np.arange(j0, j1)
    blk[idx, idx - j0] += sigma[j0:j1]
    return blk


def column_by_reflectors(j, Y, Yp, sigma):
    """A(:, j) by applying the reflectors one at a time (the definition)."""
    m, b = Y.shape
    n = Yp.shape[0]
    v = np.zeros(n)
    v[j] = 1.0
    for a in range(b):                    # V^T e_j = H'_b ... H'_1 e_j
        v -= 2.0 * Yp[:, a] * (Yp[:, a] @ v)
    x = np.zeros(m)
    x[:n] = sigma * v                     # E V^T e_j
    for a in range(b - 1, -1, -1):        # U x = H_1 ... H_b x
        x -= 2.0 * Y[:, a] * (Y[:, a] @ x)
    return x
