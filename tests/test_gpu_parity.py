"""GPU parity: every C-ABI entry point against the oracle on the same seeded inputs.

Tolerances: sketch 1e-12 relative Frobenius; skeleton sets identical
except documented near-ties; Lf / Z 1e-10 relative; residuals 1e-9 relative + 4u||A||_F;
integer work (pivots, identity block) bit-exact.
"""
import math

import numpy as np
import pytest
import torch

import paper_2104_05877_b200 as sk
from inputs import kahan_witness, make_c1, make_lowrank
from oracle import cpqr as o_cpqr
from oracle import idcoef as o_id
from oracle import lupp as o_lupp
from oracle import residual as o_res
from oracle import sketch as o_sketch
from tests.parity import lupp_parity, rel_fro

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
U = 2.0 ** -53


def dev_f(a):
    """numpy (any order) -> column-major CUDA float64 tensor."""
    return sk.fortran(torch.from_numpy(np.ascontiguousarray(a)).to(DEV))


def dev_rowmajor(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def rand_mat(m, n, seed, decay=0.97):
    rng = np.random.default_rng(seed)
    r = min(m, n)
    return make_lowrank(m, n, decay ** np.arange(r), rng)


# ------------------------------------------------------------------ S0+S1 dense sketch
@pytest.mark.parametrize("m,n,l,seed", [
    (256, 256, 40, 2001),        # C1 shape
    (1000, 777, 37, 5),          # ragged tiles in every dimension, odd l
    (4096, 300, 26, 2018),       # C2 k=16 shape (column-reduced)
    (3000, 64, 200, 9),          # split-K path (small n)
    (65, 3, 65, 1),              # l = m, tiny n
])
def test_sketch_dense_parity(m, n, l, seed):
    A = rand_mat(m, n, seed)
    X = sk.sketch(dev_f(A), l, "gaussian", seed).cpu().numpy()
    ref = o_sketch.sketch(A, l, "gaussian", seed)
    assert rel_fro(X, ref) <= 1e-12


def test_sketch_dense_odd_lda():
    m, n, l = 300, 50, 20
    A = rand_mat(m, n, 3)
    buf = torch.zeros((n, m + 3), dtype=torch.float64, device=DEV)
    buf[:, :m] = torch.from_numpy(A.T.copy()).to(DEV)
    Av = buf.t()[:m]                       # column-major view, lda = m + 3 = 303 (odd: no TMA)
    assert Av.stride(1) % 2 == 1
    X = sk.sketch(Av, l, "gaussian", 11).cpu().numpy()
    assert rel_fro(X, o_sketch.sketch(A, l, "gaussian", 11)) <= 1e-12


# ------------------------------------------------------------------ S1 with power iterations (8(f))
@pytest.mark.parametrize("m,n,l,q,seed", [(256, 256, 40, 1, 2001), (700, 333, 37, 1, 5), (300, 200, 26, 2, 9)])
def test_sketch_power_parity(m, n, l, q, seed):
    A = rand_mat(m, n, seed, 0.9)
    X = sk.sketch_power(dev_f(A), l, "gaussian", seed, q).cpu().numpy()
    ref = o_sketch.sketch_power(A, l, "gaussian", seed, q)
    assert rel_fro(X, ref) <= 1e-12


def test_rand_lupp_1piter_c1():
    """Rand-LUPP-1piter on C1: pivots identical to the oracle, residual within tolerance."""
    A, sigma = make_c1(seed=1001)
    Ad = dev_f(A)
    k, l = 20, 40
    X = sk.sketch_power(Ad, l, "gaussian", 2001, 1)
    Js, _, _, _ = sk.select_cols(X, k)
    Xo = o_sketch.sketch_power(A, l, "gaussian", 2001, 1)
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    r, nA = sk.residual(Ad, Js, None, "col_id")
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert abs(r - ro) <= 1e-9 * ro + 4 * U * nAo
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-12)


def _align_rows(Xg, Xo):
    """X from an orthogonalised iteration is unique up to the signs of its rows (the basis' column
    signs, R21): flip the GPU's rows onto the oracle's before comparing."""
    s = np.sign(np.sum(Xg * Xo, axis=1))
    s[s == 0] = 1.0
    return Xg * s[:, None]


@pytest.mark.parametrize("m,n,l,q,seed", [(256, 256, 40, 1, 2001), (700, 333, 37, 2, 5), (300, 200, 26, 3, 9),
                                           (3000, 1500, 90, 2, 12)])
def test_sketch_power_ortho_parity(m, n, l, q, seed):
    """eq:ortho_power_iter against the oracle (bases up to column signs)."""
    A = rand_mat(m, n, seed, 0.9)
    X = sk.sketch_power(dev_f(A), l, "gaussian", seed, q, ortho=True).cpu().numpy()
    ref = o_sketch.sketch_power_ortho(A, l, "gaussian", seed, q)
    assert rel_fro(_align_rows(X, ref), ref) <= 1e-10


def test_rand_lupp_1piter_ortho_c2_k512():
    """Rand-LUPP-1piter at the C2 bench configuration (k = 512): the plain form X = Omega A^T A
    squares the spectrum (10^(-i/25)) and fails the rank test near step 390; the orthogonalised
    form keeps sigma_i and selects all 512 pivots, identical to the oracle's."""
    from inputs import make_c2
    A, sigma = make_c2(seed=1002)
    k, l, seed = 512, 522, 2002 + 512
    Ad = dev_f(A)
    X = sk.sketch_power(Ad, l, "gaussian", seed, 1, ortho=True)
    Js, _, _, _ = sk.select_cols(X, k)
    Xo = o_sketch.sketch_power_ortho(A, l, "gaussian", seed, 1)
    assert rel_fro(_align_rows(X.cpu().numpy(), Xo), Xo) <= 1e-10
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    r, nA = sk.residual(Ad, Js, None, "col_id")
    ro, nAo = o_res.residual(A, piv, kind="col_id")
    assert abs(r - ro) <= 1e-9 * ro + 4 * U * nAo
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-9)


# ------------------------------------------------------------------ Algorithm 3 (streaming two-sided selection, 8(f))
@pytest.mark.parametrize("m,n,l,emb,seed", [(256, 256, 40, "gaussian", 3), (600, 333, 37, "gaussian", 4),
                                             (500, 300, 30, "sparse_sign", 5), (1200, 20000, 1100, "gaussian", 6)])  # 3 Omega blocks
def test_sketch_cols_parity(m, n, l, emb, seed):
    A = rand_mat(m, n, seed)
    Y = sk.sketch_cols(dev_f(A), l, emb, seed).cpu().numpy()
    assert rel_fro(Y, o_sketch.sketch_cols(A, l, emb, seed)) <= 1e-12


@pytest.mark.parametrize("m,n,lx,ly,seed,host", [(1000, 777, 61, 45, 1, True), (1000, 777, 61, 45, 1, False),
                                                  (4096, 4096, 266, 266, 2, True), (3000, 20000, 1100, 300, 3, True)])
def test_sketch_dual_one_pass_parity(m, n, lx, ly, seed, host):
    """Algorithm 3 line 2: X = Gamma A and Y = A Omega^T -- from ONE pass of a host A over
    PCIe in column blocks (each block feeding both products), or from device memory -- equal the
    oracle's two sketches with the same (independent) seeds."""
    A = rand_mat(m, n, seed)
    Ain = torch.from_numpy(np.asfortranarray(A)).pin_memory() if host else dev_f(A)
    X, Y = sk.sketch_dual(Ain, lx, ly, seed_x=100 + seed, seed_y=200 + seed)
    assert rel_fro(X.cpu().numpy(), o_sketch.sketch(A, lx, "gaussian", 100 + seed)) <= 1e-12
    assert rel_fro(Y.cpu().numpy(), o_sketch.sketch_cols(A, ly, "gaussian", 200 + seed)) <= 1e-12


@pytest.mark.parametrize("k,l", [(20, 40), (20, 20)])
def test_alg3_sketch_only_estimates_c1(k, l):
    """The sketch-only estimates of P:428-440 on C1: Z = X_1^+ X, W = Y Y_1^+ and the three residuals
    ||A - C Z||, ||A - W R||, ||A - C S^{-1} R|| against the oracle's least-squares / solve."""
    from oracle import estimates as o_est
    A, sigma = make_c1(seed=1001)
    Ad = dev_f(A)
    X, Y = sk.sketch_dual(Ad, l, l, seed_x=2001, seed_y=3001)
    Js, _, _, _ = sk.select_cols(X, k)
    Is, _, _, _ = sk.select_rows(Y, k)
    Z = sk.id_estimate_cols(X, Js)
    W = sk.id_estimate_rows(Y, Is)
    rz, nA = sk.residual(Ad, Js, None, "id_coeffs", Z)
    rw, _ = sk.residual(Ad, None, Is, "row_coeffs", W)
    rc, _ = sk.residual(Ad, Js, Is, "cur_css")
    Xo = o_sketch.sketch(A, l, "gaussian", 2001)
    Yo = o_sketch.sketch_cols(A, l, "gaussian", 3001)
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    (ipiv, _, _, _), _ = lupp_parity(Is.cpu().numpy(), lambda f: o_lupp.select_rows(Yo, k, f))
    Zo = o_est.id_estimate_cols(Xo, piv)
    Wo = o_est.id_estimate_rows(Yo, ipiv)
    assert rel_fro(Z.cpu().numpy(), Zo) <= 1e-8
    assert rel_fro(W.cpu().numpy(), Wo) <= 1e-8
    nAo = float(np.linalg.norm(A))
    for r, approx in ((rz, A[:, piv] @ Zo), (rw, Wo @ A[ipiv, :]), (rc, o_est.cur_css(A, ipiv, piv))):
        ro = float(np.linalg.norm(A - approx))
        assert abs(r - ro) <= 1e-8 * ro + 4 * U * nAo, (r, ro)
        assert ro >= o_res.optimal_error(sigma, k) * (1 - 1e-9)


def test_stream_select_alg3_c1():
    A, sigma = make_c1(seed=1001)
    k, l = 20, 40
    Js, Is = sk.stream_select(dev_f(A), k, l, seed_x=2001, seed_y=3001)
    Xo = o_sketch.sketch(A, l, "gaussian", 2001)
    Yo = o_sketch.sketch_cols(A, l, "gaussian", 3001)
    lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))
    lupp_parity(Is.cpu().numpy(), lambda f: o_lupp.select_rows(Yo, k, f))
    r, nA = sk.residual(dev_f(A), Js, Is, "cur")
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-12)


# ------------------------------------------------------------------ SRTT embedding (8(f) rank 3)
@pytest.mark.parametrize("m,n,l,seed", [(8, 5, 3, 1), (256, 256, 40, 2001), (4096, 333, 266, 7), (16384, 70, 510, 3),
                                         (32768, 301, 300, 11), (65536, 37, 1100, 12), (131072, 160, 777, 13),
                                         (131072, 3, 1, 14)])
def test_sketch_srtt_parity(m, n, l, seed):
    """m <= 16384 (l permitting): one CTA per column; beyond: the four-step transform, a cluster of
    m / 16384 CTAs per column whose partial Hartley values meet in distributed shared memory."""
    A = rand_mat(m, n, seed)
    X = sk.sketch(dev_f(A), l, "srtt", seed).cpu().numpy()
    assert rel_fro(X, o_sketch.sketch_srtt_fft(A, l, seed)) <= 1e-12


def test_sketch_srtt_large_m_limits():
    """Beyond the four-step kernel's reach: m > 131072, or l past its shared-memory table."""
    with pytest.raises(sk.SkelError) as e:
        sk.sketch(dev_f(rand_mat(262144, 2, 1)), 8, "srtt", 1)
    assert e.value.status == 1
    with pytest.raises(sk.SkelError) as e:
        sk.sketch(dev_f(rand_mat(32768, 2, 1)), 6000, "srtt", 1)
    assert e.value.status == 1


def test_srtt_rand_lupp_c1():
    A, sigma = make_c1(seed=1001)
    k, l = 20, 40
    X = sk.sketch(dev_f(A), l, "srtt", 2001)
    Js, _, _, _ = sk.select_cols(X, k)
    Xo = o_sketch.sketch_srtt_fft(A, l, 2001)
    lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(Xo, k, f))


def test_sketch_srtt_rejects_non_power_of_two():
    with pytest.raises(sk.SkelError) as e:
        sk.sketch(dev_f(rand_mat(100, 10, 1)), 8, "srtt", 1)
    assert e.value.status == 1


# ------------------------------------------------------------------ RSVD-DEIM (8(f) rank 4)
@pytest.mark.parametrize("k,l", [(20, 40), (10, 30)])
def test_select_cols_deim_c1(k, l):
    from oracle import deim as o_deim
    A, sigma = make_c1(seed=1001)
    Ad = dev_f(A)
    X = sk.sketch(Ad, l, "gaussian", 2001)
    Js = sk.select_cols_deim(Ad, X, k)
    Xo = o_sketch.sketch(A, l, "gaussian", 2001)
    assert Js.cpu().tolist() == o_deim.select_cols_deim(A, Xo, k).tolist()
    r, nA = sk.residual(Ad, Js, None, "col_id")
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-12)


# ------------------------------------------------------------------ S1' sparse sketch
@pytest.mark.parametrize("m,n,l,zeta,seed", [
    (1000, 100, 60, 8, 2003),
    (300, 33, 16, 8, 1),
    (517, 70, 510, 8, 4),
    (129, 5, 40, 33, 6),
    (1300, 4000, 700, 8, 7),     # 48 rows per warp, ragged last chunk and column tile, one i-half per CTA
    (2048, 9000, 510, 8, 8),     # C3's l, whole chunks, full waves (no i-split)
    (300, 70, 8, 4, 9),          # zeta < 8
])
def test_sketch_sparse_parity(m, n, l, zeta, seed):
    A = rand_mat(m, n, seed)
    Ad = dev_f(A)
    X = sk.sketch(Ad, l, "sparse_sign", seed, zeta).cpu().numpy()
    ref = o_sketch.sketch(A, l, "sparse_sign", seed, zeta)
    assert rel_fro(X, ref) <= 1e-12
    X2 = sk.sketch(Ad, l, "sparse_sign", seed, zeta).cpu().numpy()
    np.testing.assert_array_equal(X, X2)                     # fixed summation order: deterministic


# ------------------------------------------------------------------ S2 select_cols
@pytest.mark.parametrize("n,l,k,seed", [
    (256, 40, 20, 1),            # C1 shape
    (1000, 74, 64, 2),           # one panel
    (3000, 140, 130, 3),         # several panels + trailing GEMM
    (777, 70, 70, 4),            # k = l, ragged n
    (70, 70, 70, 5),             # k = n (square)
    (40001, 80, 70, 6),          # tall: several clusters exchanging winners in global memory, ragged
    (70000, 40, 36, 7),          # taller than one cluster can hold (> 65536 rows)
    (131000, 30, 24, 8),         # C5 row-LUPP height class (32 clusters of 4), ragged
    # k >= 512 takes the planner's "fewest rows per thread" order (lupp.cu): these reach the
    # multi-cluster instantiations C5's column LUPP runs
    (30000, 522, 512, 9),        # v2<1,64,multi>: 15 clusters of 8, 1 row per thread
    (65536, 522, 512, 10),       # v2<2,32,multi>: 32 clusters of 4 (C5 columns, k = 512)
    (65536, 1010, 1000, 11),     # v2<2,32,multi> at C5's k = 1000
    (131072, 522, 512, 12),      # v2<4,16,multi>: 32 clusters of 4, 4 rows per thread
])
def test_select_cols_parity(n, l, k, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((l, n))
    fast = n * k > 4_000_000                 # the plain-C oracle LUPP (bitwise equal to the numpy loop)
    Xd = dev_rowmajor(X)
    Js, Lf, Ug, gaps = sk.select_cols(Xd, k, want_gaps=True)
    Js2, _, _, _ = sk.select_cols(Xd, k)     # the instantiation without the gap output (the bench's)
    assert torch.equal(Js, Js2)
    (piv, Lo, Uo, go), ties = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.select_cols(X, k, f, fast=fast))
    Lg = Lf.cpu().numpy()
    assert np.max(np.abs(Lg)) <= 1.0 + 1e-14
    np.testing.assert_array_equal(Lg[Js.cpu().numpy(), np.arange(k)], 1.0)
    if ties == 0:
        assert rel_fro(Lg, Lo) <= 1e-10
        assert rel_fro(Ug.cpu().numpy(), Uo) <= 1e-10
        np.testing.assert_allclose(gaps.cpu().numpy(), go, atol=1e-9)


def test_select_cols_cluster_exhausted_first():
    """Multi-cluster panel (30000 rows: 15 clusters of 2048 rows at k >= 512) where k exceeds the
    rows of one cluster: cluster 0's rows are scaled up so they are all pivoted first, after which
    that cluster has no active row and its message carries key 0 while the others keep going."""
    n, k = 30000, 2100
    rng = np.random.default_rng(21)
    X = rng.standard_normal((k, n))
    X[:, :2048] *= 1e6
    Js, Lf, _, _ = sk.select_cols(dev_rowmajor(X), k)
    jg = Js.cpu().numpy()
    assert sorted(jg[:2048].tolist()) == list(range(2048))
    (piv, Lo, _, _), ties = lupp_parity(jg, lambda f: o_lupp.select_cols(X, k, f, fast=True))
    assert np.max(np.abs(Lf.cpu().numpy())) <= 1.0 + 1e-14


def test_select_cols_kahan_all_ties():
    # Lemma 2 witness: every step is an exact tie -> lowest index -> 0..l-1
    l = 20
    X = kahan_witness(l, l + 9)
    Js, Lf, _, _ = sk.select_cols(dev_rowmajor(X), l)
    assert Js.cpu().tolist() == list(range(l))
    Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
    T = Z.cpu().numpy()[:, l:]
    assert np.max(np.abs(T)) == 2.0 ** (l - 1)
    assert eta >= 2.0 ** (l - 1)


@pytest.mark.parametrize("n", [40001, 70000, 131000])
def test_select_cols_tall_all_ties_across_clusters(n):
    """Lemma 2's all-ties witness spread over a panel tall enough to run in several clusters:
    every step is an exact tie between rows in different clusters, so the lowest global index
    must win each cross-cluster exchange (R6); gaps are exactly 0."""
    l = 12
    W = kahan_witness(l, l + 9)
    pos = np.sort(np.random.default_rng(n).choice(n, size=l + 9, replace=False))
    X = np.zeros((l, n))
    X[:, pos] = W
    Js, _, _, gaps = sk.select_cols(dev_rowmajor(X), l, want_gaps=True)
    assert Js.cpu().tolist() == pos[:l].tolist()
    assert not gaps.cpu().numpy().any()


def test_select_cols_ties_lowest_original_index():
    X = np.array([[1.0, 1.0, 3.0], [5.0, -5.0, 0.0]])
    Js, _, _, _ = sk.select_cols(dev_rowmajor(X), 2)
    assert Js.cpu().tolist() == [2, 0]


def test_select_cols_rank_failure():
    rng = np.random.default_rng(8)
    C = rng.standard_normal((30, 3)) @ rng.standard_normal((3, 4))
    X = C.T.copy()                                   # 4 x 30 of rank 3
    with pytest.raises(sk.SkelError) as e:
        sk.select_cols(dev_rowmajor(X), 4)
    assert e.value.status == 2 and e.value.info == 4


def test_select_cols_bad_args():
    X = dev_rowmajor(np.ones((4, 10)))
    with pytest.raises(sk.SkelError) as e:
        sk.select_cols(X, 5)                          # k > l
    assert e.value.status == 1


# ------------------------------------------------------------------ S4 select_rows
@pytest.mark.parametrize("m,k,seed", [(500, 20, 1), (3000, 100, 2), (129, 129, 3), (20000, 12, 4)])
def test_select_rows_parity(m, k, seed):
    rng = np.random.default_rng(seed)
    C = rng.standard_normal((m, k))
    Is, Lf, _, _ = sk.select_rows(dev_f(C), k)
    (piv, Lo, _, _), ties = lupp_parity(Is.cpu().numpy(), lambda f: o_lupp.select_rows(C, k, f))
    if ties == 0:
        assert rel_fro(Lf.cpu().numpy(), Lo) <= 1e-10


def test_gather_cols_bitwise():
    A = rand_mat(300, 50, 1)
    J = torch.tensor([7, 3, 49, 0], dtype=torch.int64, device=DEV)
    C = sk.gather_cols(dev_f(A), J).cpu().numpy()
    np.testing.assert_array_equal(C, A[:, [7, 3, 49, 0]])


# ------------------------------------------------------------------ S2' CPQR
@pytest.mark.parametrize("l,n,k,seed", [(26, 400, 16, 1), (74, 1000, 64, 2), (30, 5000, 30, 3)])
def test_cpqr_parity(l, n, k, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((l, n))
    Js, R = sk.select_cols_cpqr(dev_rowmajor(X), k, want_r=True)
    piv, Ro = o_cpqr.select_cols_cpqr(X, k)
    assert Js.cpu().tolist() == piv.tolist()
    assert rel_fro(R.cpu().numpy(), Ro) <= 1e-10


def test_cpqr_spec_case():
    X = np.array([[3.0, 0.0, 0.0], [0.0, 4.0, 0.0]])
    Js, _ = sk.select_cols_cpqr(dev_rowmajor(X), 2)
    assert Js.cpu().tolist() == [1, 0]


# ------------------------------------------------------------------ S5 id_coeffs
@pytest.mark.parametrize("n,k,seed", [(300, 20, 1), (2000, 100, 2), (64, 64, 3)])
def test_id_coeffs_parity(n, k, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((k + 5, n))
    Js, Lf, _, _ = sk.select_cols(dev_rowmajor(X), k)
    Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
    Zg = Z.cpu().numpy()
    jg = Js.cpu().numpy()
    np.testing.assert_array_equal(Zg[:, jg], np.eye(k))          # identity block, bitwise
    Zo, _, eta_o = o_id.id_coeffs(Lf.cpu().numpy(), jg)          # same factor -> isolates S5
    assert rel_fro(Zg, Zo) <= 1e-10
    assert abs(eta - eta_o) <= 1e-8 * eta_o


def test_id_coeffs_spec_eta():
    X = np.array([[1.0, 0.0, 0.5], [0.0, 1.0, 0.5]])
    Js, Lf, _, _ = sk.select_cols(dev_rowmajor(X), 2)
    Z, eta = sk.id_coeffs(Lf, Js, want_eta=True)
    np.testing.assert_allclose(Z.cpu().numpy()[:, 2], [0.5, 0.5], atol=1e-16)
    assert abs(eta - math.sqrt(1.5)) < 1e-12


# ------------------------------------------------------------------ S6 residual
@pytest.mark.parametrize("kind", ["col_id", "row_id", "cur", "id_coeffs"])
def test_residual_parity(kind):
    A, sigma = make_c1(seed=1001)
    k, l = 20, 40
    Ad = dev_f(A)
    X = sk.sketch(Ad, l, "gaussian", 2001)
    Js, Lf, _, _ = sk.select_cols(X, k)
    C = sk.gather_cols(Ad, Js)
    Is, _, _, _ = sk.select_rows(C, k)
    Z = sk.id_coeffs(Lf, Js)[0] if kind == "id_coeffs" else None
    r, nA = sk.residual(Ad, Js, Is, kind, Z)
    ro, nAo = o_res.residual(A, Js.cpu().numpy(), Is.cpu().numpy(), kind,
                             Z.cpu().numpy() if Z is not None else None)
    assert abs(r - ro) <= 1e-9 * ro + 4 * U * nAo
    assert abs(nA - nAo) <= 1e-13 * nAo
    assert r >= o_res.optimal_error(sigma, k) * (1 - 1e-12)


def test_residual_exact_rank_is_zero():
    rng = np.random.default_rng(4)
    A = make_lowrank(400, 300, np.array([5.0, 3, 2, 1, 0.5, 0.25]), rng)
    Ad = dev_f(A)
    X = sk.sketch(Ad, 6, "gaussian", 1)
    Js, _, _, _ = sk.select_cols(X, 6)
    Is, _, _, _ = sk.select_rows(sk.gather_cols(Ad, Js), 6)
    for kind in ("col_id", "row_id", "cur"):
        r, nA = sk.residual(Ad, Js, Is, kind)
        assert r <= 1e-12 * nA


def test_residual_identity_closed_form():
    n, k = 200, 17
    Ad = dev_f(np.eye(n))
    J = torch.arange(k, dtype=torch.int64, device=DEV)
    r, nA = sk.residual(Ad, J, J, "col_id")
    assert abs(r - math.sqrt(n - k)) < 1e-12 and abs(nA - math.sqrt(n)) < 1e-12


# ------------------------------------------------------------------ Algorithm 2 end to end
def test_rand_lupp_host_and_device_agree():
    A = rand_mat(600, 500, 7, 0.95)
    Af = np.asfortranarray(A)
    Js_h, Is_h = sk.rand_lupp(torch.from_numpy(Af.T.copy()).t(), 30, 40, rows=True, seed=5)
    Ad = dev_f(A)
    X = sk.sketch(Ad, 40, "gaussian", 5)
    Js, _, _, _ = sk.select_cols(X, 30)
    Is, _, _, _ = sk.select_rows(sk.gather_cols(Ad, Js), 30)
    assert Js_h.tolist() == Js.cpu().tolist()
    assert Is_h.tolist() == Is.cpu().tolist()


# ------------------------------------------------------------------ column-sharded entry points (8(e))
def test_gather_cols_shard_bitwise():
    A = rand_mat(300, 50, 2)
    Ad = dev_f(A)
    J = torch.tensor([7, 3, 49, 0, 20, 21], dtype=torch.int64, device=DEV)
    col0, nc = 20, 25                                    # this "rank" owns columns 20..44
    C = sk.gather_cols_shard(Ad[:, col0:col0 + nc], J, col0).cpu().numpy()
    ref = np.zeros((300, 6))
    for t, j in enumerate([7, 3, 49, 0, 20, 21]):
        if col0 <= j < col0 + nc:
            ref[:, t] = A[:, j]
    np.testing.assert_array_equal(C, ref)


def test_residual_cols_matches_oracle_and_adds_over_shards():
    A, _ = make_c1(seed=1001)
    k = 20
    Ad = dev_f(A)
    X = sk.sketch(Ad, 40, "gaussian", 2001)
    Js, _, _, _ = sk.select_cols(X, k)
    C = sk.gather_cols(Ad, Js)
    r2a, a2a = sk.residual_cols(Ad[:, :100], C)
    r2b, a2b = sk.residual_cols(Ad[:, 100:], C)
    ro, nAo = o_res.residual(A, Js.cpu().numpy(), kind="col_id")
    r = math.sqrt(r2a + r2b)
    assert abs(r - ro) <= 1e-9 * ro + 4 * U * nAo
    assert abs(math.sqrt(a2a + a2b) - nAo) <= 1e-13 * nAo


def test_dist_rand_lupp_nccl_world1():
    import torch.distributed as tdist
    from paper_2104_05877_b200.dist import dist_rand_lupp
    os_env = __import__("os").environ
    os_env.setdefault("MASTER_ADDR", "127.0.0.1")
    os_env.setdefault("MASTER_PORT", "29517")
    tdist.init_process_group("nccl", rank=0, world_size=1)
    try:
        A, _ = make_c1(seed=1001)
        out = dist_rand_lupp(dev_f(A), A.shape[1], 20, 40, "gaussian", 2001, rows=True, residual=True)
        X = o_sketch.sketch(A, 40, "gaussian", 2001)
        piv, _, _, _ = o_lupp.select_cols(X, 20)
        assert out["Js"].cpu().tolist() == piv.tolist()
        ipiv, _, _, _ = o_lupp.select_rows(A[:, piv], 20)
        assert out["Is"].cpu().tolist() == ipiv.tolist()
        ro, nAo = o_res.residual(A, piv, kind="col_id")
        assert abs(out["residual"] - ro) <= 1e-9 * ro + 4 * U * nAo
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("emb", ["gaussian", "sparse_sign"])
def test_rand_lupp_host_pipelined(emb):
    """sk_rand_lupp with a HOST A large enough (64 MB) for the pipelined path: the copy of column
    block b+1 overlaps the sketch of block b (8 blocks of 256 columns).  J_s and I_s equal the
    oracle's (near-tie rule) and the device-A path's."""
    m, n, k, l, seed = 4096, 2048, 64, 74, 31
    A = rand_mat(m, n, seed, 0.995)
    Ah = torch.from_numpy(np.asfortranarray(A)).t().contiguous().t()          # column-major host tensor
    assert Ah.stride() == (1, m)
    Js, Is = sk.rand_lupp(Ah.pin_memory() if emb == "gaussian" else Ah, k, l, emb, seed, rows=True)
    Jd, Id = sk.rand_lupp(dev_f(A), k, l, emb, seed, rows=True)
    X = o_sketch.sketch(A, l, emb, seed)
    lupp_parity(Js.numpy(), lambda f: o_lupp.select_cols(X, k, f))
    assert Js.tolist() == Jd.tolist() and Is.tolist() == Id.tolist()
    lupp_parity(Is.numpy(), lambda f: o_lupp.select_rows(A[:, Js.numpy()], k, f))


@pytest.mark.parametrize("plan", [
    (0, 48, 1, 0), (0, 64, 1, 0), (0, 32, 1, 0), (0, 40, 1, 0), (0, 56, 1, 0),   # tile heights, one K range
    (2, 48, 4, 0), (3, 48, 4, 0), (3, 64, 2, 0), (3, 32, 8, 0),        # K-splits via HBM partials / cluster DSMEM
    (0, 48, 1, 256), (2, 40, 3, 320), (3, 48, 2, 512),                  # K-chunked Omega (ragged last chunk)
    (0, 40, 1, 0, 7), (2, 48, 3, 256, 7), (3, 40, 2, 0, 7),             # 7 warps: 224-column tiles, 32-column boxes
    (0, 80, 1, 0, 4), (3, 80, 4, 0, 4), (2, 80, 3, 256, 4),            # 112-column tiles: 2 x 2 warps of 40 x 56,
    (0, 40, 1, 0, 2), (3, 40, 4, 320, 2), (2, 40, 2, 0, 2),             # or 2 warps of 40 x 56 (16-column boxes)
    (0, 80, 1, 0, 12), (2, 80, 3, 256, 12), (0, 48, 1, 0, 12),          # 12 warps: 80 x 192 (2 x 6), 48 x 384
    (0, 96, 1, 0, 8), (3, 96, 2, 0, 8),                                 # 96 x 128 (2 x 4 warps of 48 x 32)
    (0, 48, 1, 128, 12), (0, 80, 1, 96, 4), (0, 40, 1, 112, 7),         # >= 3 chunks, one K range, small grids
    (1, 0, 0, 0),                                                       # shared-memory generation fallback
])
def test_sketch_dense_plans(plan):
    """Every dense-sketch kernel configuration against the oracle (sk_set_sketch_tuning): the
    TMA + DMMA GEMM at each tile height, K-splits through HBM partials and through cluster DSMEM,
    Omega generated chunk by chunk into the reused slot with X accumulated across chunks, and the
    fallback kernel.  Ragged l, m and n span several tiles."""
    m, n, l = 1000, 700, 61
    A = rand_mat(m, n, 41)
    sk.set_sketch_tuning(*plan[:4], warps=plan[4] if len(plan) > 4 else 0)
    try:
        X = sk.sketch(dev_f(A), l, "gaussian", 77).cpu().numpy()
    finally:
        sk.set_sketch_tuning()
    assert rel_fro(X, o_sketch.sketch(A, l, "gaussian", 77)) <= 1e-12


@pytest.mark.parametrize("plan,n", [((0, 32, 1, 256, 8), 4100), ((0, 48, 1, 256, 12), 8200), ((0, 48, 1, 160, 8), 6000)])
def test_sketch_dense_chained(plan, n):
    """The chained K-chunk path (>= 3 chunks of one K range, >= one wave of tiles per chunk): chunk
    GEMMs linked by programmatic dependent launch, the next chunk's Omega image made by generator CTAs
    inside the current GEMM, device counters for image readiness and slot reuse.  Ragged last chunk
    and column tile; l spans several row tiles.  Repeated calls give the same X."""
    m, l = 800, 300
    A = rand_mat(m, n, 43)
    Ad = dev_f(A)
    sk.set_sketch_tuning(*plan[:4], warps=plan[4])
    try:
        X = sk.sketch(Ad, l, "gaussian", 79).cpu().numpy()
        X2 = sk.sketch(Ad, l, "gaussian", 79).cpu().numpy()
    finally:
        sk.set_sketch_tuning()
    assert rel_fro(X, o_sketch.sketch(A, l, "gaussian", 79)) <= 1e-12
    np.testing.assert_array_equal(X, X2)


@pytest.mark.parametrize("k,l", [(64, 74), (256, 266)])
def test_select_cols_deim_c2(k, l):
    """RSVD-DEIM at C2 (4096^2, sigma_i = 10^(-i/50)): the l x l factor of A Q_X through the row LUPP +
    Cholesky QR and its right singular vectors by one-sided Jacobi, against the oracle's Householder
    QR + LAPACK SVD; singular values are distinct, so V^_k is unique up to column signs and the DEIM
    pivots must agree."""
    from inputs import make_c2
    from oracle import deim as o_deim
    A, sigma = make_c2(seed=1002)
    Ad = dev_f(A)
    X = sk.sketch(Ad, l, "gaussian", 2002 + k)
    Js = sk.select_cols_deim(Ad, X, k)
    Xo = o_sketch.sketch(A, l, "gaussian", 2002 + k)
    V = o_deim.rsvd_vectors(A, Xo)
    (piv, _, _, _), _ = lupp_parity(Js.cpu().numpy(), lambda f: o_lupp.lupp_panel(V[:, :k], k, f))
    assert len(set(Js.cpu().tolist())) == k
