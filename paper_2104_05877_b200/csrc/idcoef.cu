// idcoef.cu -- S5: interpolative-decomposition coefficients and the Theorem 4.1 certificate.
//
// Paper: A ~ C Z (eq:colID); classical form A Pi ~ (A Pi_1)[I_k, R11^{-1} R12]
// (P:599); Theorem 4.1 eta <= sqrt(1 + ||X1^+ X2||_2^2) computable in O(l^2 (n-l)).
// Reading R10: Z(:, J_s) = I_k (assigned, exact) and Z(:, rest) = T = X1^{-1} X2 = L1^{-T} L2^T
// from the LUPP factor Lf of X^T (L1 = Lf(J_s, :), L2 = Lf(rest, :)).
//
// GPU formulation: Y = Lf L1^{-1} (n x k) by a blocked right triangular solve (DMMA GEMM
// updates + 32 x 32 diagonal solves); rows `rest` of Y are T^T; Z = Y^T with the identity
// assigned on J_s.  eta: ||T||_2^2 = lambda_max(T T^T) by power iteration on the k x k Gram.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace skel {
namespace {

// Out(t, c) = In(I[t] - off, c); an index outside [0, nrows) after the shift (e.g. the -1 of a
// rank failure, or a pivot another rank owns) gives 0.
__global__ void k_gather_rows(const double* In, int64_t ldin, int64_t nrows, const int64_t* I, int64_t off, int64_t k,
                              int64_t ncols, double* Out, int64_t ldout) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * ncols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e % k, c = e / k;
    const int64_t i = I[t] - off;
    Out[t + c * ldout] = (i >= 0 && i < nrows) ? In[i + c * ldin] : 0.0;
  }
}

__global__ void k_copy_cols(const double* In, int64_t ldin, int64_t rows, int64_t cols, double* Out,
                            int64_t ldout) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % rows, c = e / rows;
    Out[i + c * ldout] = In[i + c * ldin];
  }
}

// Z (k x n, ldz) = Y^T, Y n x k (ld n); 32 x 32 tiles through shared memory.
__global__ void k_transpose(const double* Y, int64_t n, int64_t k, double* Z, int64_t ldz) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, t0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, t = t0 + r;
    if (i < n && t < k) tile[r][threadIdx.x] = Y[i + t * n];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t t = t0 + threadIdx.x, i = i0 + r;
    if (i < n && t < k) Z[t + i * ldz] = tile[threadIdx.x][r];
  }
}

// Z(:, Js[t]) = e_t exactly; Y(Js[t], :) = 0 (so that Y^T Y = T T^T).
// Z(:, Js - off) = I_k and the skeleton rows of Y zeroed; indices outside [0, n) after the shift are
// skipped (no out-of-bounds store for the Js = -1 left by a rank failure, or another rank's pivots).
__global__ void k_identity_block(const int64_t* Js, int64_t off, int64_t k, double* Z, int64_t ldz, double* Y, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tp = e % k, t = e / k;
    const int64_t j = Js[t] - off;
    if (j < 0 || j >= n) continue;
    Z[tp + j * ldz] = (tp == t) ? 1.0 : 0.0;
    Y[j + tp * n] = 0.0;
  }
}

__global__ void k_eta(const double* lam, double* eta) { *eta = sqrt(1.0 + fmax(*lam, 0.0)); }

}  // namespace

sk_status id_l1(sk_ctx* c, const double* Lf, int64_t nrows, int64_t ldlf, const int64_t* Js, int64_t k, int64_t off,
                double* L1) {
  k_gather_rows<<<(unsigned)std::min<int64_t>(cdiv(k * k, 256), 4LL * c->num_sms), 256, 0, c->stream>>>(
      Lf, ldlf, nrows, Js, off, k, k, L1, k);
  return launched(c);
}

sk_status id_finish(sk_ctx* c, double* Y, int64_t n, int64_t k, const int64_t* Js, int64_t off, double* Z, int64_t ldz) {
  if (n > 0) {
    const dim3 tg((unsigned)cdiv(n, 32), (unsigned)cdiv(k, 32));
    k_transpose<<<tg, dim3(32, 8), 0, c->stream>>>(Y, n, k, Z, ldz);
    SK_TRY(launched(c));
  }
  k_identity_block<<<(unsigned)std::min<int64_t>(cdiv(k * k, 256), 4LL * c->num_sms), 256, 0, c->stream>>>(
      Js, off, k, Z, ldz, Y, n);
  return launched(c);
}

sk_status id_coeffs(sk_ctx* c, const double* Lf, int64_t n, int64_t k, int64_t ldlf, const int64_t* Js,
                    double* Z, int64_t ldz, double* eta_dev) {
  DBuf L1, Y;
  SK_TRY(L1.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Y.alloc(c, (size_t)n * k * sizeof(double)));
  const int blocks = (int)std::min<int64_t>(cdiv(n * k, 256), 8LL * c->num_sms);
  SK_TRY(id_l1(c, Lf, n, ldlf, Js, k, 0, L1.as<double>()));
  k_copy_cols<<<blocks, 256, 0, c->stream>>>(Lf, ldlf, n, k, Y.as<double>(), n);
  SK_TRY(launched(c));
  SK_TRY(trsm_right_l_unit(c, Y.as<double>(), n, k, n, L1.as<double>(), k));
  SK_TRY(id_finish(c, Y.as<double>(), n, k, Js, 0, Z, ldz));
  if (eta_dev) {
    DBuf G, lam;
    SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
    SK_TRY(lam.alloc(c, sizeof(double)));
    SK_TRY(gemm(c, true, false, k, k, n, 1.0, Y.as<double>(), n, Y.as<double>(), n, 0.0, G.as<double>(), k));
    SK_TRY(lambda_max(c, G.as<double>(), k, k, lam.as<double>()));
    k_eta<<<1, 1, 0, c->stream>>>(lam.as<double>(), eta_dev);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

// S5 on a column-sharded context: L1 = Lf(J_s, :) is assembled across ranks (each pivot row comes
// from its owner, zeros elsewhere, one exact sum all-reduce of k x k); Y = Lf_local L1^{-1} for this
// rank's rows; Z = Y^T with the identity on the pivots this rank owns; eta from sum_r Y_r^T Y_r.
sk_status dist_id_coeffs(sk_ctx* c, const double* Lf, int64_t k, int64_t ldlf, const int64_t* Js, double* Z,
                         int64_t ldz, double* eta_dev) {
  const DistView d = dist_view(c);
  const int64_t n = d.ncols;
  DBuf L1, Y;
  SK_TRY(L1.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Y.alloc(c, (size_t)std::max<int64_t>(n, 1) * k * sizeof(double)));
  SK_TRY(id_l1(c, Lf, n, ldlf, Js, k, d.col0, L1.as<double>()));
  SK_TRY(dist_allreduce_sum(c, L1.as<double>(), k * k));
  if (n > 0) {
    const int blocks = (int)std::min<int64_t>(cdiv(n * k, 256), 8LL * c->num_sms);
    k_copy_cols<<<blocks, 256, 0, c->stream>>>(Lf, ldlf, n, k, Y.as<double>(), n);
    SK_TRY(launched(c));
    SK_TRY(trsm_right_l_unit(c, Y.as<double>(), n, k, n, L1.as<double>(), k));
  }
  SK_TRY(id_finish(c, Y.as<double>(), n, k, Js, d.col0, Z, ldz));
  if (eta_dev) {
    DBuf G, lam;
    SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
    SK_TRY(lam.alloc(c, sizeof(double)));
    if (n > 0) SK_TRY(gemm(c, true, false, k, k, n, 1.0, Y.as<double>(), n, Y.as<double>(), n, 0.0, G.as<double>(), k));
    else SK_CUDA(c, cudaMemsetAsync(G.p, 0, (size_t)k * k * sizeof(double), c->stream));
    SK_TRY(dist_allreduce_sum(c, G.as<double>(), k * k));
    SK_TRY(lambda_max(c, G.as<double>(), k, k, lam.as<double>()));
    k_eta<<<1, 1, 0, c->stream>>>(lam.as<double>(), eta_dev);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

}  // namespace skel
