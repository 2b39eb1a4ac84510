"""Oracle pins for sketch, LUPP, CPQR, ID coefficients and residuals.

Each test pins an oracle function to something other than itself: a closed form,
a worked example (SPEC S:170, S:185, S:369 -- derived by hand in the test),
a paper statement (Lemma 2, Theorem 4.1, Remark 2.1), an independent
library routine (LAPACK getrf/geqp3/lstsq/solve via scipy/numpy) on tie-free
inputs, or brute force on tiny inputs.
"""
import itertools
import math

import numpy as np
import pytest
import scipy.linalg as sla

from inputs import haar, kahan_witness, make_c1, make_lowrank
from oracle import cpqr, idcoef, lupp, omega, residual, sketch

U_RND = 2.0 ** -53


# ----------------------------------------------------------------------------- sketch
def test_sketch_closed_forms():
    l, m, n = 12, 30, 7
    G = omega.gaussian(4, l, m)
    assert np.array_equal(sketch.sketch(np.zeros((m, n)), l, "gaussian", 4), np.zeros((l, n)))
    np.testing.assert_allclose(sketch.sketch(np.eye(m), l, "gaussian", 4), G, rtol=0, atol=0)
    E = np.zeros((m, n)); E[5, 3] = 1.0            # A = e_i e_j^T  =>  X(:, j) = Gamma(:, i)
    X = sketch.sketch(E, l, "gaussian", 4)
    np.testing.assert_array_equal(X[:, 3], G[:, 5])
    assert np.count_nonzero(X[:, [0, 1, 2, 4, 5, 6]]) == 0


def test_sketch_linearity_and_rank():
    rng = np.random.default_rng(0)
    m, n, l = 60, 40, 10
    A, B = rng.standard_normal((m, n)), rng.standard_normal((m, n))
    for kind in ("gaussian", "sparse_sign"):
        XA = sketch.sketch(A, l, kind, 9)
        XB = sketch.sketch(B, l, kind, 9)
        XAB = sketch.sketch(2 * A - 3 * B, l, kind, 9)
        np.testing.assert_allclose(XAB, 2 * XA - 3 * XB, atol=1e-12)
    # Lemma 1: rank-r A, l <= r  =>  X full row rank; rank-r A, l > r => rank r
    Ar = make_lowrank(m, n, np.array([3.0, 2.0, 1.0, 0.5]), rng)
    X = sketch.sketch(Ar, 3, "gaussian", 1)
    s = np.linalg.svd(X, compute_uv=False)
    assert s[-1] > 1e-10 * s[0]
    X = sketch.sketch(Ar, 8, "gaussian", 1)
    s = np.linalg.svd(X, compute_uv=False)
    assert s[4] < 1e-12 * s[0]


def test_sparse_sketch_is_signed_row_sums():
    rng = np.random.default_rng(2)
    m, n, l, z = 50, 6, 16, 8
    A = rng.standard_normal((m, n))
    rows, signs = omega.sparse_sign_structure(3, l, m, z)
    X = np.zeros((l, n))
    for i in range(m):                                  # scatter form, independent of the matmul
        for j in range(z):
            X[rows[i, j]] += signs[i, j] * A[i] / math.sqrt(z)
    np.testing.assert_allclose(sketch.sketch(A, l, "sparse_sign", 3, z), X, atol=1e-13)


def test_power_sketch_closed_forms():
    # eq:def_power_iter: X = Omega (A^T A)^q.  (a) A with orthonormal columns scaled by s:
    # A^T A = diag(s^2) exactly -> X = Omega diag(s^(2q)) column-wise; (b) A = I -> X = Omega;
    # (c) q = 0 is the row sketch; (d) rank-r A -> rank-r X.
    rng = np.random.default_rng(11)
    m, n, l = 40, 12, 5
    Q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    s = np.linspace(0.5, 2.0, n)
    A = Q * s
    Om = omega.gaussian(7, l, n)
    for q in (1, 2):
        np.testing.assert_allclose(sketch.sketch_power(A, l, "gaussian", 7, q), Om * s ** (2 * q), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(sketch.sketch_power(np.eye(n), l, "gaussian", 7, 1), Om, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(sketch.sketch_power(A, l, "gaussian", 7, 0), sketch.sketch(A, l, "gaussian", 7))
    Ar = make_lowrank(m, n, np.array([3.0, 1.0, 0.2]), rng)
    sv = np.linalg.svd(sketch.sketch_power(Ar, 6, "gaussian", 3, 1), compute_uv=False)
    assert sv[3] < 1e-12 * sv[0] and sv[2] > 1e-6 * sv[0]


def test_streaming_alg3_closed_forms_and_exact_rank_cur():
    # Alg. 3: Y = A Omega^T.  A = I -> Y = Omega^T.  On an exact rank-k A, column LUPP on
    # X = Gamma A and row LUPP on Y = A Omega^T (independent draws, one pass) give skeletons whose
    # stable CUR reproduces A (residual at rounding level): both sketches capture range and co-range.
    Om = omega.gaussian(5, 6, 9)
    np.testing.assert_array_equal(sketch.sketch_cols(np.eye(9), 6, "gaussian", 5), Om.T)
    rng = np.random.default_rng(3)
    A = make_lowrank(120, 90, np.array([4.0, 2.0, 1.0, 0.5, 0.1]), rng)
    k, l = 5, 9
    X = sketch.sketch(A, l, "gaussian", 11)
    Y = sketch.sketch_cols(A, l, "gaussian", 12)
    piv, _, _, _ = lupp.select_cols(X, k)
    ipiv, _, _, _ = lupp.select_rows(Y, k)
    r, nA = residual.residual(A, piv, ipiv, kind="cur")
    assert r <= 1e-12 * nA


def test_rsvd_deim_exact_rank_recovers_true_singular_vectors():
    # eq:rsvd_procedures: when rank(A) = l the sketch's row space is row(A), so V^ equals A's right
    # singular vectors up to sign (closed form from the construction), and DEIM on V^ equals LUPP
    # on those true vectors.
    from oracle import deim
    rng = np.random.default_rng(8)
    m, n, l = 60, 40, 6
    U, _ = np.linalg.qr(rng.standard_normal((m, l)))
    V, _ = np.linalg.qr(rng.standard_normal((n, l)))
    s = np.array([6.0, 4.0, 3.0, 2.0, 1.5, 1.0])
    A = (U * s) @ V.T
    X = sketch.sketch(A, l, "gaussian", 4)
    Vh = deim.rsvd_vectors(A, X)
    np.testing.assert_allclose(np.abs(np.sum(Vh * V, axis=0)), np.ones(l), atol=1e-10)
    piv = deim.select_cols_deim(A, X, 4)
    piv_true, _, _, _ = lupp.lupp_panel(V[:, :4], 4)
    assert piv.tolist() == piv_true.tolist()


# ----------------------------------------------------------------------------- LUPP
@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_spec_2x2_case(fast):
    # X = [[4,2],[1,3]] -> pivots [1,2] (1-based), L_l = [[4,0],[1,2.5]], R = [[1,.5],[0,1]].
    X = np.array([[4.0, 2.0], [1.0, 3.0]])
    piv, Lf, U, _ = lupp.select_cols(X, 2, fast=fast)
    assert piv.tolist() == [0, 1]
    np.testing.assert_array_equal(U.T, [[4.0, 0.0], [1.0, 2.5]])          # L_l = U^T
    np.testing.assert_array_equal(Lf.T, [[1.0, 0.5], [0.0, 1.0]])         # R^{LU} = Lf^T


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_identity_and_ties_lowest_original_index(fast):
    piv, _, _, _ = lupp.select_cols(np.eye(6), 6, fast=fast)
    assert piv.tolist() == list(range(6))
    # tie demo: lowest ORIGINAL index wins -> [2, 0]; LAPACK's swapped order gives [2, 1]
    X = np.array([[1.0, 1.0, 3.0], [5.0, -5.0, 0.0]])
    piv, _, _, _ = lupp.select_cols(X, 2, fast=fast)
    assert piv.tolist() == [2, 0]


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_factorization_and_bounds(fast):
    rng = np.random.default_rng(5)
    for (n, k) in [(50, 8), (200, 30), (31, 31)]:
        X = rng.standard_normal((k + 3, n))
        piv, Lf, U, gaps = lupp.select_cols(X, k, fast=fast)
        assert len(set(piv.tolist())) == k
        assert np.max(np.abs(Lf)) <= 1.0 + 1e-15                        # |R^{LU}| <= 1
        np.testing.assert_array_equal(Lf[piv, np.arange(k)], 1.0)
        L1 = Lf[piv]
        assert np.all(np.triu(L1, 1) == 0)                              # unit lower in pivot order
        M = X[:k].T
        err = np.max(np.abs(M - Lf @ U))
        assert err <= 8 * k * U_RND * np.max(np.abs(M)) * 10
        assert np.all(np.tril(U, -1) == 0)
        assert np.all((gaps >= 0) & (gaps <= 1))


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_matches_lapack_getrf_tie_free(fast):
    # scipy's getrf on X^T (partial pivoting) picks the same k pivots on tie-free random input
    rng = np.random.default_rng(6)
    for trial in range(20):
        n, k = 120, 25
        X = rng.standard_normal((k, n))
        piv, _, _, _ = lupp.select_cols(X, k, fast=fast)
        lu, ipiv = sla.lu_factor(X.T.copy())
        perm = np.arange(n)
        for i, p in enumerate(ipiv):
            perm[i], perm[p] = perm[p], perm[i]
        assert piv.tolist() == perm[:k].tolist()


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_k_row_invariance_and_duality(fast):
    rng = np.random.default_rng(7)
    X = rng.standard_normal((40, 300))
    p_all = lupp.select_cols(X, 20, fast=fast)[0]
    p_k = lupp.select_cols(X[:20], 20, fast=fast)[0]
    assert p_all.tolist() == p_k.tolist()                              # reading R5
    C = rng.standard_normal((8, 3))
    assert lupp.select_rows(C, 3, fast=fast)[0].tolist() == lupp.select_cols(C.T, 3, fast=fast)[0].tolist()


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_kahan_witness_lemma2(fast):
    # Lemma 2 tightness: every step is a tie; pivots 0..l-1; max|R1^{-1}R2| = 2^{l-1},
    # row-wise 2^{l-i} (1-based i).
    for l in (5, 10, 20):
        X = kahan_witness(l, l + 7)
        piv, Lf, U, gaps = lupp.select_cols(X, l, fast=fast)
        assert piv.tolist() == list(range(l))
        assert np.all(gaps == 0.0)
        g = lupp.growth(Lf, piv)
        np.testing.assert_array_equal(g, 2.0 ** (l - 1 - np.arange(l)))
        _, T, eta = idcoef.id_coeffs(Lf, piv)
        assert np.max(np.abs(T)) == 2.0 ** (l - 1)
        assert eta >= 2.0 ** (l - 1)


@pytest.mark.parametrize("fast", [False, True], ids=["numpy", "c"])
def test_lupp_rank_deficiency(fast):
    rng = np.random.default_rng(8)
    C = rng.standard_normal((30, 3)) @ rng.standard_normal((3, 4))      # rank 3
    lupp.select_rows(C[:, :3], 3, fast=fast)
    with pytest.raises(lupp.RankError) as e:
        lupp.select_rows(C, 4, fast=fast)
    assert e.value.step == 4


@pytest.mark.parametrize("n,k,seed", [(500, 40, 1), (3001, 100, 2), (70, 70, 3), (20000, 64, 4)])
def test_lupp_c_equals_numpy_bitwise(n, k, seed):
    """The plain-C LUPP (oracle/c/lupp.c, used for the C5-size panels) reproduces the numpy loop
    bit for bit: pivots, multipliers, U and gaps; also with a forced pivot (near-tie rule) and on
    the all-ties Kahan witness."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((k + 3, n))
    for forced in (None, {k // 2: None}):
        if forced is not None:
            ref = lupp.select_cols(X, k)[0]
            forced = {k // 2: int(ref[k // 2 + 1])}        # a valid, non-argmax pivot
        a = lupp.select_cols(X, k, forced)
        b = lupp.select_cols(X, k, forced, fast=True)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    W = kahan_witness(12, 40)
    for x, y in zip(lupp.select_cols(W, 12), lupp.select_cols(W, 12, fast=True)):
        np.testing.assert_array_equal(x, y)


# ----------------------------------------------------------------------------- CPQR
def test_cpqr_spec_case():
    # X = diag(3,4) padded with a zero column -> pivots [2,1,(3)] (1-based)
    X = np.array([[3.0, 0.0, 0.0], [0.0, 4.0, 0.0]])
    piv, R = cpqr.select_cols_cpqr(X, 2)
    assert piv.tolist() == [1, 0]
    assert abs(abs(R[0, 1]) - 4) < 1e-15 and abs(abs(R[1, 0]) - 3) < 1e-15


def test_cpqr_matches_lapack_geqp3_and_factorizes():
    rng = np.random.default_rng(10)
    for trial in range(10):
        l, n, k = 14, 90, 12
        X = rng.standard_normal((l, n))
        piv, R = cpqr.select_cols_cpqr(X, k)
        _, Rq, P = sla.qr(X, pivoting=True, mode="economic")
        assert piv.tolist() == P[:k].tolist()
        d = np.abs(R[np.arange(k), piv])
        assert np.all(np.diff(d) <= 1e-12)                              # |diag R1| non-increasing
        np.testing.assert_allclose(d, np.abs(np.diag(Rq))[:k], rtol=1e-12)
        # ||X Pi_1 - Q R11||: the leading k pivoted columns are spanned exactly
        Q = np.linalg.qr(X[:, piv])[0]
        np.testing.assert_allclose(np.abs(Q.T @ X[:, piv]), np.abs(R[:, piv]), atol=1e-12)


# ----------------------------------------------------------------------------- ID coefficients
def test_idcoef_spec_eta_case():
    # X = [[1,0,.5],[0,1,.5]], pivots [1,2] -> X1^+X2 = (.5,.5)^T -> eta = sqrt(1.5)
    X = np.array([[1.0, 0.0, 0.5], [0.0, 1.0, 0.5]])
    piv, Lf, _, _ = lupp.select_cols(X, 2)
    Z, T, eta = idcoef.id_coeffs(Lf, piv)
    assert piv.tolist() == [0, 1]
    np.testing.assert_allclose(T[:, 0], [0.5, 0.5], atol=1e-16)
    assert abs(eta - math.sqrt(1.5)) < 1e-15


def test_idcoef_identity_block_and_library_solve():
    rng = np.random.default_rng(11)
    X = rng.standard_normal((30, 400))
    k = 25
    piv, Lf, _, _ = lupp.select_cols(X, k)
    Z, T, eta = idcoef.id_coeffs(Lf, piv)
    assert np.array_equal(Z[:, piv], np.eye(k))                         # bitwise identity block
    rest = np.setdiff1d(np.arange(400), piv)
    T_ref = np.linalg.solve(X[:k, piv], X[:k, rest])                    # X1^{-1} X2
    np.testing.assert_allclose(T, T_ref, atol=1e-10 * np.max(np.abs(T_ref)))
    # interpolation: X[:k] = X[:k, J] Z exactly up to rounding
    np.testing.assert_allclose(X[:k, piv] @ Z, X[:k], atol=1e-10)
    assert eta >= 1.0


def test_theorem41_certificate():
    # Theorem 4.1: ||A - CC^+A||_F <= eta ||A - A X^+ X||_F with X the k-row sketch (R5)
    rng = np.random.default_rng(12)
    for trial in range(30):
        m, n, k = 60, 50, 6
        sig = 0.7 ** np.arange(min(m, n))
        A = make_lowrank(m, n, sig, rng)
        X = sketch.sketch(A, k + 4, "gaussian", trial)
        piv, Lf, _, _ = lupp.select_cols(X, k)
        _, _, eta = idcoef.id_coeffs(Lf, piv)
        res, _ = residual.residual(A, piv, kind="col_id")
        Xk = X[:k]
        rf = np.linalg.norm(A - A @ np.linalg.pinv(Xk) @ Xk)
        assert res <= eta * rf * (1 + 1e-8)


# ----------------------------------------------------------------------------- residuals
def test_residual_closed_forms():
    n, k = 40, 7
    r, nA = residual.residual(np.eye(n), np.arange(k), kind="col_id")
    assert abs(r - math.sqrt(n - k)) < 1e-13 and abs(nA - math.sqrt(n)) < 1e-13
    r, _ = residual.residual(np.eye(n), Is=np.arange(k), kind="row_id")
    assert abs(r - math.sqrt(n - k)) < 1e-13
    # exact rank k: any independent skeleton gives a zero residual (SPEC acceptance 1)
    rng = np.random.default_rng(13)
    A = make_lowrank(80, 60, np.array([5.0, 3, 2, 1, 0.5]), rng)
    X = sketch.sketch(A, 5, "gaussian", 3)
    piv = lupp.select_cols(X, 5)[0]
    Ipiv = lupp.select_rows(A[:, piv], 5)[0]
    for kind in ("col_id", "row_id", "cur"):
        r, nA = residual.residual(A, piv, Ipiv, kind=kind)
        assert r <= 1e-13 * nA


def test_residual_against_lstsq_and_eckart_young():
    A, sigma = make_c1(seed=5, m=96, n=80)
    k = 10
    X = sketch.sketch(A, 20, "gaussian", 2)
    piv, Lf, _, _ = lupp.select_cols(X, k)
    r, nA = residual.residual(A, piv, kind="col_id")
    C = A[:, piv]
    r_ls = np.linalg.norm(A - C @ np.linalg.lstsq(C, A, rcond=None)[0])
    assert abs(r - r_ls) <= 1e-10 * r
    assert abs(nA - math.sqrt(np.sum(sigma ** 2))) < 1e-13
    assert r >= residual.optimal_error(sigma, k) * (1 - 1e-12)            # Eckart-Young
    Z, _, _ = idcoef.id_coeffs(Lf, piv)
    r_z, _ = residual.residual(A, piv, kind="id_coeffs", Z=Z)
    assert r_z >= r * (1 - 1e-12)                                           # CC^+A is the best C-based fit


def test_remark21_sandwich_and_identity():
    # Remark 2.1
    rng = np.random.default_rng(14)
    for trial in range(10):
        A = make_lowrank(50, 40, 0.8 ** np.arange(40), rng)
        k = 8
        piv = lupp.select_cols(sketch.sketch(A, k, "gaussian", trial), k)[0]
        Ipiv = lupp.select_rows(A[:, piv], k)[0]
        rc, _ = residual.residual(A, piv, kind="col_id")
        rr, _ = residual.residual(A, Is=Ipiv, kind="row_id")
        rcur, _ = residual.residual(A, piv, Ipiv, kind="cur")
        assert rc <= rcur * (1 + 1e-9)
        assert rcur ** 2 <= (rc ** 2 + rr ** 2) * (1 + 1e-9)
        Qc = residual.ortho(A[:, piv])
        Qr = residual.ortho(A[Ipiv].T)
        extra = np.linalg.norm(Qc @ Qc.T @ (A - A @ Qr @ Qr.T))
        assert abs(rcur ** 2 - (rc ** 2 + extra ** 2)) <= 1e-9 * rcur ** 2


def test_two_sided_id_equals_column_id():
    # (C S^{-1}) S (C^+ A) = C C^+ A
    rng = np.random.default_rng(15)
    A = make_lowrank(40, 30, 0.6 ** np.arange(30), rng)
    k = 5
    piv = lupp.select_cols(sketch.sketch(A, k, "gaussian", 0), k)[0]
    Ipiv = lupp.select_rows(A[:, piv], k)[0]
    C = A[:, piv]
    S = A[np.ix_(Ipiv, piv)]
    tsid = np.linalg.solve(S.T, C.T).T @ S @ np.linalg.lstsq(C, A, rcond=None)[0]
    r_ts = np.linalg.norm(A - tsid)
    r, nA = residual.residual(A, piv, kind="col_id")
    assert abs(r_ts - r) <= 1e-10 * nA


def test_brute_force_subset_bounds():
    # min_J ||A - CC^+A||_F <= sqrt(k+1) ||A - A_k||_F, and LUPP's subset is never below min_J
    rng = np.random.default_rng(16)
    k = 3
    for trial in range(25):
        A = rng.standard_normal((12, 10)) * (0.5 ** np.arange(10))
        sv = np.linalg.svd(A, compute_uv=False)
        opt = residual.optimal_error(sv, k)
        best = min(residual.residual(A, list(J), kind="col_id")[0]
                   for J in itertools.combinations(range(10), k))
        assert opt <= best * (1 + 1e-12)
        assert best <= math.sqrt(k + 1) * opt * (1 + 1e-12)
        piv = lupp.select_cols(sketch.sketch(A, k + 2, "gaussian", trial), k)[0]
        assert residual.residual(A, piv, kind="col_id")[0] >= best * (1 - 1e-12)


def test_c5_generator_wy_equals_reflectors_small():
    # C5's compact-WY construction (the GPU build path) equals the reflector-by-reflector
    # definition, and the spectrum is exactly sigma (small instance of the same code).
    from inputs import c5
    Y, Yp, s = c5.factors(7, 300, 200, 8)
    W, Z = c5.wy_operands(Y, Yp, s)
    A = -(Y @ W) - Z @ Yp.T
    A[np.arange(200), np.arange(200)] += s
    cols = np.stack([c5.column_by_reflectors(j, Y, Yp, s) for j in range(200)], 1)
    np.testing.assert_allclose(A, cols, atol=1e-14)
    np.testing.assert_allclose(np.linalg.svd(A, compute_uv=False), s, atol=1e-14)


def test_generators_spectra():
    A, sigma = make_c1(seed=3, m=64, n=64)
    s = np.linalg.svd(A, compute_uv=False)
    np.testing.assert_allclose(s, sigma, rtol=1e-12, atol=1e-15)
    Q = haar(50, 10, np.random.default_rng(0))
    np.testing.assert_allclose(Q.T @ Q, np.eye(10), atol=1e-14)


def test_streamed_sketch_and_residual_equal_the_plain_definitions():
    """The column-block forms used at C5 (68.7 GB) equal the plain definitions they restate:
    X(:, J) = Gamma A(:, J) and ||E||_F^2 = sum over column blocks."""
    rng = np.random.default_rng(12)
    A = make_lowrank(300, 211, 0.9 ** np.arange(211), rng)
    get = lambda a, b: A[:, a:b]  # noqa: E731
    for kind in ("gaussian", "sparse_sign"):
        X = sketch.sketch(A, 30, kind, 5)
        np.testing.assert_allclose(sketch.sketch_streamed(get, 300, 211, 30, kind, 5, block=64), X,
                                   rtol=0, atol=1e-14 * np.abs(X).max())
    piv = lupp.select_cols(sketch.sketch(A, 20, "gaussian", 3), 20)[0]
    r, nA = residual.residual(A, piv, kind="col_id")
    rs, nAs = residual.residual_col_id_streamed(get, 300, 211, piv, block=50)
    assert abs(r - rs) <= 1e-12 * r and abs(nA - nAs) <= 1e-13 * nA


def test_ortho_power_iteration_closed_forms():
    """eq:ortho_power_iter pinned by closed forms: for A with orthonormal columns
    (A^T A = I) the rows of X = ortho(Y_q)^T A are orthonormal (X X^T = Q^T A A^T Q = I); for q = 1,
    X = R^{-T} X_plain with Y_1 = A Omega^T = Q R (diag R > 0) and X_plain = Omega A^T A = Y_1^T A
    (eq:def_power_iter); for q = 2 the row space equals the plain iteration's, and column LUPP picks
    the same pivots (LUPP pivots are invariant under lower-triangular row mixing of X)."""
    rng = np.random.default_rng(17)
    V = haar(60, 25, rng)                                     # 60 x 25, orthonormal columns
    for q in (1, 2, 3):
        X = sketch.sketch_power_ortho(V, 10, "gaussian", 4, q)
        np.testing.assert_allclose(X @ X.T, np.eye(10), atol=1e-13)
    A = make_lowrank(80, 50, 0.8 ** np.arange(50), rng)
    Y1 = A @ omega.embedding("gaussian", 9, 12, 50).T
    _, R = np.linalg.qr(Y1)
    R *= np.sign(np.diag(R))[:, None]
    Xp = sketch.sketch_power(A, 12, "gaussian", 9, 1)
    np.testing.assert_allclose(Xp, Y1.T @ A, rtol=0, atol=1e-13 * np.abs(Xp).max())
    Xo = sketch.sketch_power_ortho(A, 12, "gaussian", 9, 1)
    np.testing.assert_allclose(R.T @ Xo, Xp, rtol=0, atol=1e-12 * np.abs(Xp).max())
    Xo2 = sketch.sketch_power_ortho(A, 12, "gaussian", 9, 2)
    Xp2 = sketch.sketch_power(A, 12, "gaussian", 9, 2)
    P1 = (lambda Q: Q @ Q.T)(np.linalg.qr(Xo2.T)[0])            # projectors onto the row spaces
    P2 = (lambda Q: Q @ Q.T)(np.linalg.qr(Xp2.T)[0])
    np.testing.assert_allclose(P1, P2, atol=1e-10)
    assert lupp.select_cols(Xo2, 10)[0].tolist() == lupp.select_cols(Xp2, 10)[0].tolist()


def test_alg3_estimates_closed_forms():
    """P:428-440 pinned by what the algebra fixes: on an exact-rank-k A with full-rank sketches the
    estimates are exact -- X_1^+ X = C^+ A (A = C Z with Z = C^+ A, X = Gamma C Z, X_1 = Gamma C),
    Y Y_1^+ = A R^+ and C S^{-1} R = A; for any A, X_1^+ X restricted to J_s is I_k and Y Y_1^+ restricted
    to I_s is I_k."""
    from oracle import estimates
    rng = np.random.default_rng(23)
    m, n, k, l = 90, 70, 6, 10
    A = rng.standard_normal((m, k)) @ rng.standard_normal((k, n))            # rank k exactly
    X = sketch.sketch(A, l, "gaussian", 1)
    Y = sketch.sketch_cols(A, l, "gaussian", 2)
    Js = lupp.select_cols(X, k)[0]
    Is = lupp.select_rows(Y, k)[0]
    C, R = A[:, Js], A[Is, :]
    Z = estimates.id_estimate_cols(X, Js)
    np.testing.assert_allclose(Z, np.linalg.lstsq(C, A, rcond=None)[0], atol=1e-10)
    W = estimates.id_estimate_rows(Y, Is)
    np.testing.assert_allclose(W, np.linalg.lstsq(R.T, A.T, rcond=None)[0].T, atol=1e-10)
    np.testing.assert_allclose(estimates.cur_css(A, Is, Js), A, atol=1e-10 * np.abs(A).max())
    B = make_lowrank(m, n, 0.7 ** np.arange(n), rng)                         # general A
    Xb = sketch.sketch(B, l, "gaussian", 3)
    Jb = lupp.select_cols(Xb, k)[0]
    np.testing.assert_allclose(estimates.id_estimate_cols(Xb, Jb)[:, Jb], np.eye(k), atol=1e-12)
    Yb = sketch.sketch_cols(B, l, "gaussian", 4)
    Ib = lupp.select_rows(Yb, k)[0]
    np.testing.assert_allclose(estimates.id_estimate_rows(Yb, Ib)[Ib, :], np.eye(k), atol=1e-12)
