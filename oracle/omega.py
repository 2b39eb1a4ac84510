"""The oblivious embeddings Gamma in R^{l x m}, explicit and dense (TEST INFRASTRUCTURE ONLY).

Paper: Section 2.2 "Randomized linear embeddings".
  * Gaussian:    i.i.d. entries S_ij ~ N(mu, 1/l)
  * sparse sign: i.i.d. zeta-sparse columns, zeta Rademacher variables at
                 uniformly random coordinates, zeta = min(l, 8)

Readings: mu = 0 (R3); the sparse-sign entries are +-1/sqrt(zeta)
(R4: BASELINE.json's "+-1/sqrt(8)"; the printed sqrt(m/zeta) is not norm
preserving); the i.i.d. draws come from Philox4x32-10 with the counter layout
R1/R2 below, which the CUDA path implements independently.

Counter layout (R1):
  Gaussian   Philox(ctr = (i mod 2^32, i div 2^32, p, 0x47415553), key = seed)
             -> u1 = U53(w0, w1), u2 = U53(w2, w3) -> Box-Muller
             z_{2p}   = sqrt(-2 ln u1) cos(2 pi u2),
             z_{2p+1} = sqrt(-2 ln u1) sin(2 pi u2),   Gamma[r, i] = z_r / sqrt(l).
  sparse     column i, call c: Philox(ctr = (i mod 2^32, i div 2^32, c, 0x53504152), key = seed);
             row word j (j < zeta) = word (j mod 4) of call (j div 4); the rows are
             drawn by Floyd's subset algorithm: for j = 0..zeta-1,
             N = l - zeta + j + 1, t = floor(w_j * N / 2^32), and t is replaced by
             N - 1 if already chosen; sign bit of entry j = bit (j mod 32) of word
             ((j div 32) mod 4) of call ceil(zeta/4) + (j div 128); bit 1 -> negative.
"""
import math

import numpy as np

from .philox import philox4x32_10, uniform53

TAG_GAUSS = 0x47415553
TAG_SPARSE = 0x53504152


def _seed_key(seed):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def gaussian_z(seed, l, rows_i):
    """Standard normals z[r, i] (before the 1/sqrt(l) scale) for r < l and i in rows_i."""
    k0, k1 = _seed_key(seed)
    i = np.asarray(rows_i, dtype=np.uint64)
    npair = (l + 1) // 2
    z = np.empty((2 * npair, i.size), dtype=np.float64)
    for p in range(npair):
        w = philox4x32_10(i & np.uint64(0xFFFFFFFF), i >> np.uint64(32), p, TAG_GAUSS, k0, k1)
        u1 = uniform53(w[0], w[1])
        u2 = uniform53(w[2], w[3])
        rad = np.sqrt(-2.0 * np.log(u1))
        z[2 * p] = rad * np.cos(2.0 * np.pi * u2)
        z[2 * p + 1] = rad * np.sin(2.0 * np.pi * u2)
    return z[:l]


def gaussian(seed, l, m):
    """Dense Gaussian embedding Gamma (l x m), entries N(0, 1/l)."""
    return gaussian_z(seed, l, np.arange(m)) / math.sqrt(l)


def sparse_sign_structure(seed, l, m, zeta):
    """For each column i of Gamma: the zeta distinct rows and their signs (+1/-1).

    Returns (rows int64 [m, zeta], signs float64 [m, zeta]), entry order = draw order j.
    """
    if not (2 <= zeta <= l):
        raise ValueError("sparse sign needs 2 <= zeta <= l (P:182)")
    k0, k1 = _seed_key(seed)
    i = np.arange(m, dtype=np.uint64)
    ilo, ihi = i & np.uint64(0xFFFFFFFF), i >> np.uint64(32)
    n_row_calls = (zeta + 3) // 4
    words = []
    for c in range(n_row_calls):
        words.extend(philox4x32_10(ilo, ihi, c, TAG_SPARSE, k0, k1))
    n_sign_calls = (zeta + 127) // 128
    sign_words = []
    for c in range(n_sign_calls):
        sign_words.extend(philox4x32_10(ilo, ihi, n_row_calls + c, TAG_SPARSE, k0, k1))
    rows = np.empty((m, zeta), dtype=np.int64)
    signs = np.empty((m, zeta), dtype=np.float64)
    for col in range(m):
        chosen = []
        for j in range(zeta):
            n_range = l - zeta + j + 1
            t = (int(words[j][col]) * n_range) >> 32
            if t in chosen:
                t = n_range - 1
            chosen.append(t)
            bit = (int(sign_words[j >> 5][col]) >> (j & 31)) & 1
            signs[col, j] = -1.0 if bit else 1.0
        rows[col] = chosen
    return rows, signs


def sparse_sign(seed, l, m, zeta):
    """Dense copy of the sparse-sign embedding Gamma (l x m), entries +-1/sqrt(zeta)."""
    rows, signs = sparse_sign_structure(seed, l, m, zeta)
    g = np.zeros((l, m), dtype=np.float64)
    scale = 1.0 / math.sqrt(zeta)
    for col in range(m):
        g[rows[col], col] = signs[col] * scale
    return g


def embedding(kind, seed, l, m, zeta=8):
    if kind in ("gaussian", 0):
        return gaussian(seed, l, m)
    if kind in ("sparse_sign", 1):
        return sparse_sign(seed, l, m, zeta)
    if kind in ("srtt", 2):
        return srtt(seed, l, m)
    raise ValueError(kind)


# ----------------------------------------------------------------------------------- SRTT
# Subsampled randomized trigonometric transform (Table 1):
#     Gamma = sqrt(m/l) Pi_{m->l} T Phi Pi_{m->m},
# T the unitary discrete Hartley transform T(k, i) = cas(2 pi i k / m) / sqrt(m), cas = cos + sin.
# Readings (R18): the random choices are counter-based so both sides can draw them
# independently -- Pi_{m->m} and Pi_{m->l} are keyed 4-round Feistel bijections on the b = log2(m)
# bit indices (XOR of each half with a Philox word of the other half), Phi(i) = -1 iff bit 0 of a
# Philox word of i is 1.  R19: m must be a power of two (the fast transform's radix-2 length).
TAG_PERM, TAG_SUBS, TAG_SIGN = 0x5045524D, 0x53554253, 0x5349474E


def feistel(x, b, tag, seed):
    """Keyed bijection of [0, 2^b) (4 rounds; round r XORs one half with a Philox word of the other)."""
    k0, k1 = _seed_key(seed)
    x = np.asarray(x, dtype=np.uint64)
    hb = b // 2
    lb = b - hb
    lo = x & np.uint64((1 << lb) - 1)
    hi = x >> np.uint64(lb)
    for r in range(4):
        if r % 2 == 0:
            w = philox4x32_10(lo, r, 0, tag, k0, k1)[0]
            hi = hi ^ (w & np.uint64((1 << hb) - 1))
        else:
            w = philox4x32_10(hi, r, 0, tag, k0, k1)[0]
            lo = lo ^ (w & np.uint64((1 << lb) - 1))
    return ((hi << np.uint64(lb)) | lo).astype(np.int64)


def srtt_parts(seed, l, m):
    """(perm, signs, sel): y_i = signs_i x_{perm_i}; output row r takes transform index sel_r."""
    b = int(m).bit_length() - 1
    if m < 2 or (1 << b) != m:
        raise ValueError("SRTT needs m a power of two (R19)")
    if not (1 <= l <= m):
        raise ValueError("1 <= l <= m")
    idx = np.arange(m, dtype=np.uint64)
    perm = feistel(idx, b, TAG_PERM, seed)
    k0, k1 = _seed_key(seed)
    w = philox4x32_10(idx, 0, 0, TAG_SIGN, k0, k1)[0]
    signs = np.where((w & np.uint64(1)) == 1, -1.0, 1.0)
    sel = feistel(np.arange(l, dtype=np.uint64), b, TAG_SUBS, seed)
    return perm, signs, sel


def hartley(m):
    """The unitary DHT matrix, by definition."""
    i = np.arange(m)
    th = 2.0 * np.pi * (np.outer(i, i) % m) / m       # reduce i k mod m first (exact integers)
    return (np.cos(th) + np.sin(th)) / math.sqrt(m)


def srtt(seed, l, m):
    """Dense SRTT embedding Gamma (l x m), formed literally: sqrt(m/l) Pi_{m->l} T Phi Pi_{m->m}."""
    perm, signs, sel = srtt_parts(seed, l, m)
    Pmm = np.zeros((m, m))
    Pmm[np.arange(m), perm] = 1.0                    # (Pi x)_i = x_{perm_i}
    Pml = np.zeros((l, m))
    Pml[np.arange(l), sel] = 1.0
    return math.sqrt(m / l) * Pml @ hartley(m) @ np.diag(signs) @ Pmm
