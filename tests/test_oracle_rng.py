"""Oracle pins: Philox KAT and the distribution of the embeddings."""
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import omega
from oracle.philox import philox4x32_10, uniform53

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def test_philox_known_answers():
    n = 0
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        out = philox4x32_10(*v[:6])
        assert [int(o) for o in out] == v[6:]
        n += 1
    assert n == 3


def test_uniform53_range_and_exactness():
    # extremes of the word range: smallest 2^-54 (> 0), largest rounds to exactly 1.0
    lo = uniform53(np.array([0]), np.array([0]))[0]
    hi = uniform53(np.array([0xFFFFFFFF]), np.array([0xFFFFFFFF]))[0]
    assert lo == 0.5 * 2.0 ** -53 and 0 < lo
    assert hi == 1.0
    # 53 significant bits: consecutive low words differ by exactly 2^-53
    a = uniform53(np.array([123]), np.array([64]))[0]
    b = uniform53(np.array([123]), np.array([128]))[0]
    assert b - a == 2.0 ** -53


def test_gaussian_moments_and_ks():
    # 1e6 draws: mean 0, variance 1/l, kurtosis 3, KS against N(0, 1/l)  (reading R3: mu = 0)
    l, m = 20, 50000
    g = omega.gaussian(seed=7, l=l, m=m).ravel()
    assert abs(g.mean()) < 5 * math.sqrt(1.0 / l / g.size)
    assert abs(g.var() * l - 1.0) < 0.01
    assert abs(stats.kurtosis(g * math.sqrt(l), fisher=False) - 3.0) < 0.03
    p = stats.kstest(g * math.sqrt(l), "norm").pvalue
    assert p > 1e-3


def test_gaussian_norm_preservation():
    # E ||Gamma e_1||^2 = 1; here over 2000 independent seeds, l = 20
    vals = [np.sum(omega.gaussian_z(s, 20, [0])[:, 0] ** 2) / 20 for s in range(2000)]
    assert abs(np.mean(vals) - 1.0) < 0.1


def test_gaussian_rows_independent_of_l():
    # prefix consistency: rows r < k of an l-row Gamma equal sqrt(k/l) x the k-row Gamma
    g40 = omega.gaussian(3, 40, 64)
    g20 = omega.gaussian(3, 20, 64)
    np.testing.assert_allclose(g40[:20] * math.sqrt(40), g20 * math.sqrt(20), rtol=0, atol=1e-15)


def test_gaussian_pairs_are_independent_draws():
    # the two normals of one Box-Muller pair are uncorrelated across columns
    z = omega.gaussian_z(11, 2, np.arange(200000))
    assert abs(np.corrcoef(z[0], z[1])[0, 1]) < 0.01


@pytest.mark.parametrize("l,zeta", [(16, 8), (510, 8), (9, 2), (40, 33)])
def test_sparse_sign_structure(l, zeta):
    m = 3000
    rows, signs = omega.sparse_sign_structure(5, l, m, zeta)
    # exactly zeta distinct rows per column, all in range
    assert rows.min() >= 0 and rows.max() < l
    for c in range(m):
        assert len(set(rows[c].tolist())) == zeta
    g = omega.sparse_sign(5, l, m, zeta)
    nnz = np.count_nonzero(g, axis=0)
    assert np.all(nnz == zeta)
    assert np.allclose(np.abs(g[g != 0]), 1 / math.sqrt(zeta))
    # unit column norms (reading R4) -> E||Gamma x||^2 = ||x||^2
    assert np.allclose(np.sum(g * g, axis=0), 1.0)
    # sign balance
    frac_neg = np.mean(signs < 0)
    assert abs(frac_neg - 0.5) < 5 * math.sqrt(0.25 / signs.size)


def test_sparse_sign_rows_uniform():
    # each row is hit with probability zeta/l: chi-square on the row frequencies
    l, m, zeta = 64, 40000, 8
    rows, _ = omega.sparse_sign_structure(9, l, m, zeta)
    counts = np.bincount(rows.ravel(), minlength=l)
    p = stats.chisquare(counts).pvalue
    assert p > 1e-3


def test_sparse_sign_subsets_uniform():
    # Floyd's algorithm gives uniformly random zeta-subsets: all C(5,2) = 10 subsets equally likely
    l, zeta, m = 5, 2, 50000
    rows, _ = omega.sparse_sign_structure(13, l, m, zeta)
    keys = np.sort(rows, axis=1) @ np.array([l, 1])
    _, counts = np.unique(keys, return_counts=True)
    assert counts.size == 10
    assert stats.chisquare(counts).pvalue > 1e-3


def test_sparse_sign_norm_preservation():
    vals = []
    for s in range(2000):
        g = omega.sparse_sign(s, 16, 4, 8)
        vals.append(np.sum(g[:, 0] ** 2))
    assert abs(np.mean(vals) - 1.0) < 0.1


# ------------------------------------------------------------------ SRTT (R18, R19)
@pytest.mark.parametrize("b", [3, 8, 12, 17])
def test_srtt_feistel_is_a_bijection(b):
    x = np.arange(2 ** b, dtype=np.uint64)
    for tag in (omega.TAG_PERM, omega.TAG_SUBS):
        y = omega.feistel(x, b, tag, 99)
        assert np.array_equal(np.sort(y), np.arange(2 ** b))


def test_srtt_closed_forms():
    m, l = 64, 20
    T = omega.hartley(m)
    np.testing.assert_allclose(T @ T, np.eye(m), atol=1e-13)          # the unitary DHT is an involution
    np.testing.assert_allclose(T, T.T, atol=0)                         # and symmetric
    G = omega.srtt(5, l, m)
    np.testing.assert_allclose(G @ G.T, (m / l) * np.eye(l), atol=1e-12)   # rows of a scaled unitary
    perm, signs, sel = omega.srtt_parts(5, l, m)
    assert set(np.unique(signs)) <= {-1.0, 1.0} and len(set(sel.tolist())) == l


def test_srtt_fft_route_equals_definition_and_preserves_norms():
    from oracle import sketch as o_sketch
    rng = np.random.default_rng(1)
    A = rng.standard_normal((128, 9))
    np.testing.assert_allclose(o_sketch.sketch(A, 30, "srtt", 7), o_sketch.sketch_srtt_fft(A, 30, 7), atol=1e-12)
    x = rng.standard_normal(256)
    ratios = [np.sum(o_sketch.sketch_srtt_fft(x[:, None], 64, s) ** 2) / np.sum(x * x) for s in range(200)]
    assert abs(np.mean(ratios) - 1.0) < 0.05                          # E ||Gamma x||^2 = ||x||^2
