"""Seeded synthetic matrices for BASELINE.json configs C1-C5 (recipes: DESIGN.md §6).

All matrices are float64, returned column-major (numpy order='F') because the
C-ABI stores A column-major.  Nothing here implements the method.
"""
import numpy as np

# name -> (m, n, spectrum/recipe, embedding, ks, l(k), input seed, sketch seed base)
CONFIGS = {
    "C1": dict(m=256, n=256, emb="gaussian", ks=(20,), l=lambda k: 40, seed=1001, sk_seed=2001),
    "C2": dict(m=4096, n=4096, emb="gaussian", ks=(16, 64, 256, 512), l=lambda k: k + 10,
               seed=1002, sk_seed=2002),
    "C3": dict(m=16384, n=16384, emb="sparse_sign", ks=(500,), l=lambda k: k + 10, seed=1003,
               sk_seed=2003, zeta=8),
    "C4": dict(m=65536, n=784, emb="gaussian", ks=(50, 100, 200), l=lambda k: 2 * k, seed=1004,
               sk_seed=2004),
    "C5": dict(m=131072, n=65536, emb="gaussian", ks=(1000,), l=lambda k: 1100, seed=1005,
               sk_seed=2005),
}


def haar(n, r, rng):
    """n x r matrix with orthonormal columns, Haar (Stiefel) distributed.

    Q of a Gaussian matrix with the sign fix diag(sign(R_ii)) (Mezzadri 2007)."""
    g = rng.standard_normal((n, r))
    q, rr = np.linalg.qr(g, mode="reduced")
    d = np.sign(np.diag(rr))
    d[d == 0] = 1.0
    return q * d


def make_lowrank(m, n, sigma, rng):
    """U diag(sigma) V^T with Haar U (m x r), V (n x r); returns Fortran-ordered A."""
    r = len(sigma)
    U = haar(m, r, rng)
    V = haar(n, r, rng)
    return np.asfortranarray((U * sigma) @ V.T)


def make_c1(seed=1001, m=256, n=256):
    """C1: A = U diag(i^-2) V^T, Haar U, V (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    r = min(m, n)
    sigma = np.arange(1, r + 1, dtype=np.float64) ** -2.0
    return make_lowrank(m, n, sigma, rng), sigma


def make_c2(seed=1002, m=4096, n=4096):
    """C2: A = U diag(10^(-i/50)) V^T, Haar U, V (configs[1])."""
    rng = np.random.default_rng(seed)
    r = min(m, n)
    sigma = 10.0 ** (-np.arange(1, r + 1, dtype=np.float64) / 50.0)
    return make_lowrank(m, n, sigma, rng), sigma


def make_c3(seed=1003, m=16384, n=16384, rank=1000, noise=1e-6):
    """C3: rank-1000 U diag(1/i) V^T + i.i.d. N(0,1) * 1e-6 noise (configs[2]; reading R13: std 1e-6)."""
    rng = np.random.default_rng(seed)
    rank = min(rank, m, n)
    sigma = 1.0 / np.arange(1, rank + 1, dtype=np.float64)
    A = make_lowrank(m, n, sigma, rng)
    A += noise * np.asfortranarray(rng.standard_normal((m, n)))
    return A, sigma


def make_c4(seed=1004, m=65536, n=784, clusters=10, proto_rank=20, noise=0.05):
    """C4: nonnegative image-like rows (configs[3]; reading R14).

    Each cluster c owns B_c ~ U[0,1]^{proto_rank x n}; row = sum_c w_c h_c^T B_c with
    w ~ Dir(1_clusters), h_c ~ Dir(1_proto_rank); + U[0, noise] noise; clipped to [0,1]."""
    rng = np.random.default_rng(seed)
    B = rng.random((clusters, proto_rank, n))
    w = rng.dirichlet(np.ones(clusters), size=m)                    # m x clusters
    h = rng.dirichlet(np.ones(proto_rank), size=(m, clusters))      # m x clusters x proto_rank
    coef = (w[:, :, None] * h).reshape(m, clusters * proto_rank)
    A = coef @ B.reshape(clusters * proto_rank, n)
    A += noise * rng.random((m, n))
    np.clip(A, 0.0, 1.0, out=A)
    return np.asfortranarray(A), None


def make_config(name, **kw):
    return {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4}[name](**kw)


def kahan_witness(l, n):
    """Lemma 2's tight case: X = [R1 R2] with R1 unit upper, R1(i,j) = -1 above the
    diagonal, R2 = 1.  Every LUPP step is an all-ties step."""
    X = np.ones((l, n))
    X[:, :l] = np.triu(-np.ones((l, l)), 1) + np.eye(l)
    return X
