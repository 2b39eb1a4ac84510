// dense.cu -- the small dense building blocks around the hot path:
//   gather (S3: C = A(:, J_s)), blocked Cholesky, blocked triangular solves,
//   two-pass Cholesky QR (ortho()) and a power iteration for ||T||_2 (Thm 4.1 eta).
// Heavy lifting is delegated to the DMMA GEMM (gemm.cu); the kernels here only handle
// the 32 x 32 diagonal blocks.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace skel {
namespace {

constexpr int TB = 32;   // diagonal block size

// C(:, t) = A(:, J[t] - col0) when col0 <= J[t] < col0 + ncols (this rank's column block), else 0.
// Unsharded use: col0 = 0, ncols = n.
__global__ void k_gather_cols(const double* A, int64_t m, int64_t lda, const int64_t* J, int64_t k,
                              int64_t col0, int64_t ncols, double* C, int64_t ldc) {
  const int64_t t = blockIdx.y;
  const int64_t j = J[t] - col0;
  const bool own = j >= 0 && j < ncols;
  const double* src = A + (own ? j : 0) * lda;
  double* dst = C + t * ldc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = own ? src[i] : 0.0;
}

// Rt(:, t) = A(I[t], :)^T  (row gather; reads are strided by lda, writes coalesced)
__global__ void k_gather_rows_t(const double* A, int64_t n, int64_t lda, const int64_t* I, int64_t k,
                                double* Rt, int64_t ldrt) {
  const int64_t t = blockIdx.y;
  const int64_t i = I[t];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    Rt[j + t * ldrt] = A[i + j * lda];
}

// Unblocked Cholesky of one jb x jb diagonal block (lower, in place), jb <= TB.
__global__ void k_potrf_diag(double* G, int64_t ld, int jb, int64_t col0, int64_t* status) {
  if (*status != 0) return;
  __shared__ double a[TB][TB + 1];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    a[i][j] = G[i + j * ld];
  }
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    if (tid == 0) {
      const double d = a[c][c];
      if (!(d > 0.0)) {
        bad = c + 1;
      } else {
        a[c][c] = sqrt(d);
      }
    }
    __syncthreads();
    if (bad) break;
    const double d = a[c][c];
    for (int i = c + 1 + tid; i < jb; i += blockDim.x) a[i][c] /= d;
    __syncthreads();
    for (int e = tid; e < (jb - c - 1) * (jb - c - 1); e += blockDim.x) {
      const int i = c + 1 + e % (jb - c - 1), j = c + 1 + e / (jb - c - 1);
      if (j <= i) a[i][j] = fma(-a[i][c], a[j][c], a[i][j]);
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *status = col0 + bad;
    return;
  }
  for (int e = tid; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    G[i + j * ld] = j <= i ? a[i][j] : 0.0;
  }
}

// X(rows x jb) <- X * Ljj^{-T}, Ljj lower non-unit (jb <= TB).  One thread per row.
__global__ void k_trsm_diag_lt(double* X, int64_t rows, int64_t ldx, int jb, const double* L,
                               int64_t ldl, const int64_t* status) {
  if (status && *status != 0) return;
  __shared__ double l[TB][TB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    l[i][j] = L[i + j * ldl];
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[TB];
#pragma unroll
    for (int c = 0; c < TB; ++c) {
      if (c < jb) {
        double s = X[r + c * ldx];
#pragma unroll
        for (int cp = 0; cp < TB; ++cp)
          if (cp < c) s = fma(-x[cp], l[c][cp], s);
        x[c] = s / l[c][c];
      }
    }
#pragma unroll
    for (int c = 0; c < TB; ++c)
      if (c < jb) X[r + c * ldx] = x[c];
  }
}

// X(rows x jb) <- X * Ljj^{-1}, Ljj unit lower (jb <= TB): x[c] = y[c] - sum_{c'>c} x[c'] L[c'][c].
__global__ void k_trsm_diag_l_unit(double* X, int64_t rows, int64_t ldx, int jb, const double* L,
                                   int64_t ldl) {
  __shared__ double l[TB][TB + 1];
  for (int e = threadIdx.x; e < jb * jb; e += blockDim.x) {
    const int i = e % jb, j = e / jb;
    l[i][j] = L[i + j * ldl];
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double x[TB];
#pragma unroll
    for (int c = TB - 1; c >= 0; --c) {
      if (c < jb) {
        double s = X[r + c * ldx];
#pragma unroll
        for (int cp = TB - 1; cp > 0; --cp)
          if (cp > c && cp < jb) s = fma(-x[cp], l[cp][c], s);
        x[c] = s;
      }
    }
#pragma unroll
    for (int c = 0; c < TB; ++c)
      if (c < jb) X[r + c * ldx] = x[c];
  }
}

// One power-iteration step: y = G x / ||x||; done early when converged (flag).
__global__ void k_power_step(const double* G, int64_t k, int64_t ld, const double* x, double* y,
                             double* lam, int* done) {
  if (*done) return;
  __shared__ double sred[34];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) s = fma(x[i], x[i], s);
  s = dev::block_sum(s, sred);
  const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
  const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  for (int64_t r = blockIdx.x * warps + (threadIdx.x >> 5); r < k; r += (int64_t)gridDim.x * warps) {
    double d = 0.0;
    for (int64_t j = lane; j < k; j += 32) d = fma(G[r + j * ld], x[j], d);   // G symmetric
    d = dev::warp_sum(d);
    if (lane == 0) y[r] = d * inv;
  }
  (void)lam;
}

// Rayleigh-type estimate lam = ||y|| (y = G u, ||u|| = 1); convergence flag on relative change.
__global__ void k_power_check(const double* y, int64_t k, double* lam, int* done) {
  if (*done) return;
  __shared__ double sred[34];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) s = fma(y[i], y[i], s);
  s = dev::block_sum(s, sred);
  if (threadIdx.x == 0) {
    const double nl = sqrt(s);
    if (fabs(nl - lam[0]) <= 1e-15 * nl) *done = 1;
    lam[0] = nl;
  }
}

__global__ void k_fill_ones(double* x, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 1.0 + 1e-3 * (double)((i * 2654435761LL) % 1000) / 1000.0;
}

}  // namespace

sk_status gather_cols(sk_ctx* c, const double* A, int64_t m, int64_t lda, const int64_t* J, int64_t k,
                      double* C, int64_t ldc) {
  return gather_cols_shard(c, A, m, lda, 0, INT64_MAX, J, k, C, ldc);
}

sk_status gather_cols_shard(sk_ctx* c, const double* A, int64_t m, int64_t lda, int64_t col0, int64_t ncols,
                            const int64_t* J, int64_t k, double* C, int64_t ldc) {
  if (m == 0 || k == 0) return SK_OK;
  const unsigned bx = (unsigned)std::min<int64_t>(cdiv(m, 256), 64);
  k_gather_cols<<<dim3(bx, (unsigned)k), 256, 0, c->stream>>>(A, m, lda, J, k, col0, ncols, C, ldc);
  return launched(c);
}

sk_status gather_rows_t(sk_ctx* c, const double* A, int64_t n, int64_t lda, const int64_t* I, int64_t k,
                        double* Rt, int64_t ldrt) {
  if (k == 0 || n == 0) return SK_OK;
  const int bx = (int)std::min<int64_t>(cdiv(n, 256), 64);
  k_gather_rows_t<<<dim3(bx, (unsigned)k), 256, 0, c->stream>>>(A, n, lda, I, k, Rt, ldrt);
  return launched(c);
}

sk_status potrf_lower(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t* status_dev) {
  for (int64_t j0 = 0; j0 < k; j0 += TB) {
    const int jb = (int)std::min<int64_t>(TB, k - j0);
    k_potrf_diag<<<1, 256, 0, c->stream>>>(G + j0 + j0 * ld, ld, jb, j0, status_dev);
    SK_TRY(launched(c));
    const int64_t j1 = j0 + jb;
    if (j1 < k) {
      const int64_t rows = k - j1;
      const int blocks = (int)std::min<int64_t>(cdiv(rows, 128), 4LL * c->num_sms);
      k_trsm_diag_lt<<<blocks, 128, 0, c->stream>>>(G + j1 + j0 * ld, rows, ld, jb, G + j0 + j0 * ld, ld,
                                                     status_dev);
      SK_TRY(launched(c));
      SK_TRY(gemm(c, false, true, rows, rows, jb, -1.0, G + j1 + j0 * ld, ld, G + j1 + j0 * ld, ld, 1.0,
                  G + j1 + j1 * ld, ld));
    }
  }
  return SK_OK;
}

sk_status trsm_right_lt(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                        int64_t ldl) {
  for (int64_t j0 = 0; j0 < k; j0 += TB) {
    const int jb = (int)std::min<int64_t>(TB, k - j0);
    if (j0 > 0)
      SK_TRY(gemm(c, false, true, rows, jb, j0, -1.0, X, ldx, L + j0, ldl, 1.0, X + j0 * ldx, ldx));
    const int blocks = (int)std::min<int64_t>(cdiv(rows, 128), 8LL * c->num_sms);
    k_trsm_diag_lt<<<blocks, 128, 0, c->stream>>>(X + j0 * ldx, rows, ldx, jb, L + j0 + j0 * ldl, ldl,
                                                   nullptr);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

sk_status trsm_right_l_unit(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                            int64_t ldl) {
  const int64_t nblk = cdiv(k, TB);
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t j0 = b * TB;
    const int jb = (int)std::min<int64_t>(TB, k - j0);
    const int64_t j1 = j0 + jb;
    if (j1 < k)
      SK_TRY(gemm(c, false, false, rows, jb, k - j1, -1.0, X + j1 * ldx, ldx, L + j1 + j0 * ldl, ldl, 1.0,
                  X + j0 * ldx, ldx));
    const int blocks = (int)std::min<int64_t>(cdiv(rows, 128), 8LL * c->num_sms);
    k_trsm_diag_l_unit<<<blocks, 128, 0, c->stream>>>(X + j0 * ldx, rows, ldx, jb, L + j0 + j0 * ldl, ldl);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

sk_status cholqr2(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev) {
  DBuf G;
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  for (int pass = 0; pass < 2; ++pass) {
    SK_TRY(gemm(c, true, false, k, k, m, 1.0, Q, ldq, Q, ldq, 0.0, G.as<double>(), k));
    SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
    SK_TRY(trsm_right_lt(c, Q, m, k, ldq, G.as<double>(), k));
  }
  return SK_OK;
}

sk_status lambda_max(sk_ctx* c, const double* G, int64_t k, int64_t ld, double* out_dev) {
  DBuf xb, yb, flag;
  SK_TRY(xb.alloc(c, (size_t)k * sizeof(double)));
  SK_TRY(yb.alloc(c, (size_t)k * sizeof(double)));
  SK_TRY(flag.alloc(c, sizeof(int)));
  SK_CUDA(c, cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
  SK_CUDA(c, cudaMemsetAsync(out_dev, 0, sizeof(double), c->stream));
  k_fill_ones<<<(unsigned)cdiv(k, 256), 256, 0, c->stream>>>(xb.as<double>(), k);
  SK_TRY(launched(c));
  double* x = xb.as<double>();
  double* y = yb.as<double>();
  const int warps = 8;
  const int blocks = (int)std::min<int64_t>(cdiv(k, warps), 2LL * c->num_sms);
  for (int it = 0; it < 400; ++it) {
    k_power_step<<<blocks, warps * 32, 0, c->stream>>>(G, k, ld, x, y, out_dev, flag.as<int>());
    k_power_check<<<1, 256, 0, c->stream>>>(y, k, out_dev, flag.as<int>());
    SK_TRY(launched(c, 2));
    std::swap(x, y);
  }
  return SK_OK;
}

}  // namespace skel
