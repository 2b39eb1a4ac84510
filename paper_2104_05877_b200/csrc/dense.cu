// dense.cu -- the small dense building blocks around the hot path:
//   gather (S3: C = A(:, J_s)), blocked Cholesky, blocked triangular solves,
//   two-pass Cholesky QR (ortho()) and a power iteration for ||T||_2 (Thm 4.1 eta).
// Heavy lifting is delegated to the DMMA GEMM (gemm.cu); the kernels here only handle
// the 32 x 32 diagonal blocks.
#include <algorithm>
#include <cmath>

#include <cstdlib>

#include "common.cuh"
#include "dmma.cuh"
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
// Rt(:, t) = A(I[t], :)^T; a row index outside [0, m) gives a zero column (no out-of-bounds read).
__global__ void k_gather_rows_t(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I, int64_t k,
                                double* Rt, int64_t ldrt) {
  const int64_t t = blockIdx.y;
  const int64_t i = I[t];
  const bool ok = i >= 0 && i < m;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    Rt[j + t * ldrt] = ok ? A[i + j * lda] : 0.0;
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

// lambda_max of the SPD k x k matrix G by power iteration in ONE persistent launch: the grid's CTAs
// are co-resident (cooperative launch); iteration t: every CTA loads x = y_{t-1} / ||y_{t-1}|| into
// shared memory, computes its rows of y_t = G x (a warp per row, G read through L2), publishes the
// partial sum of y_t^2 and releases its flag (st.release.gpu); after every flag reached t + 1 each
// CTA sums the partials in the same fixed order, so all CTAs see the same lambda_t = ||y_t|| and
// stop at the same iteration: when lambda stops increasing (relative change <= 1e-15; for SPD G the
// sequence is non-decreasing) or after max_it iterations.  Buffers by iteration parity: a CTA
// overwrites buffer t & 1 only after every CTA finished iteration t - 1, i.e. read buffer t & 1.
__device__ __forceinline__ double power_init(int64_t i) {
  return 1.0 + 1e-3 * (double)((i * 2654435761LL) % 1000) / 1000.0;
}

__global__ void __launch_bounds__(256) k_power_persistent(const double* __restrict__ G, int64_t k, int64_t ld,
                                                          double* ybuf, double* part, unsigned long long* flags,
                                                          double* lam_out, int max_it) {
  extern __shared__ double xs[];                       // [k]
  __shared__ double s_nrm, s_lam;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nb = gridDim.x;
  const int warps = blockDim.x >> 5;
  double lam_prev = 0.0;
  if (tid == 0) s_nrm = 0.0;
  // x_0 = init / ||init||
  for (int64_t i = tid; i < k; i += blockDim.x) xs[i] = power_init(i);
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
    for (int64_t i = lane; i < k; i += 32) s = fma(xs[i], xs[i], s);
    s = dev::warp_sum(s);
    if (lane == 0) s_nrm = sqrt(s);
  }
  __syncthreads();
  for (int64_t i = tid; i < k; i += blockDim.x) xs[i] /= s_nrm;
  __syncthreads();
  for (int it = 0; it < max_it; ++it) {
    double* y = ybuf + (int64_t)(it & 1) * k;
    double* pt = part + (int64_t)(it & 1) * nb;
    double acc = 0.0;
    for (int64_t r = (int64_t)blockIdx.x * warps + warp; r < k; r += (int64_t)nb * warps) {
      double d = 0.0;
      for (int64_t j = lane; j < k; j += 32) d = fma(__ldcg(G + r + j * ld), xs[j], d);   // G symmetric
      d = dev::warp_sum(d);
      if (lane == 0) { y[r] = d; acc = fma(d, d, acc); }
    }
    __shared__ double wpart[32];
    if (lane == 0) wpart[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < warps; ++w) s += wpart[w];
      pt[blockIdx.x] = s;
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + (int64_t)blockIdx.x * 16),
                   "l"((unsigned long long)it + 1ull) : "memory");
    }
    for (int b = tid; b < nb; b += blockDim.x) {
      unsigned long long f;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flags + (int64_t)b * 16) : "memory");
      } while (f < (unsigned long long)it + 1ull);
    }
    __syncthreads();
    if (tid == 0) {                                    // fixed order: identical in every CTA
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += __ldcg(pt + b);
      s_lam = sqrt(s);
    }
    __syncthreads();
    const double lam = s_lam;
    const bool done = lam <= 0.0 || (it > 0 && lam - lam_prev <= 1e-15 * lam) || it + 1 == max_it;
    if (done) {
      if (blockIdx.x == 0 && tid == 0) *lam_out = lam;
      return;
    }
    lam_prev = lam;
    for (int64_t i = tid; i < k; i += blockDim.x) xs[i] = __ldcg(y + i) / lam;
    __syncthreads();
  }
}

__global__ void k_fill_ones(double* x, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = power_init(i);
}


// ---- 64-wide diagonal blocks: factor / invert in one CTA, apply by an in-place row kernel ----
constexpr int TB2 = 64;

// MODE 0: G (jb x jb SPD, ld) -> its Cholesky factor L (lower, upper zeroed, in place) and
//         W = L^{-1} (lower, ldw).  MODE 1: G holds a unit lower L (read only) -> W = L^{-1}.
//         MODE 2: G holds a non-unit lower L (read only) -> W = L^{-1}.
// status: 1-based failing column (+ col0) on a non-positive pivot (MODE 0).
// Blocked by 16.  A 16 x 16 diagonal block is factored AND inverted by one warp in registers
// (lane i < 16 holds row i; columns broadcast by shuffles, no shared-memory round trips), the
// panel below it is L_ip = A_ip W_pp^T (independent 16-term dot products over all threads), the
// trailing triangle gets the rank-16 update; the off-diagonal blocks of W = L^{-1} follow by block
// distance d: W_ij = -W_ii (sum_{j<=k<i} L_ik W_kj).
constexpr int DB = 16;

// lane i < 16: row i of a 16 x 16 lower factor L in r[0..15] (unit diagonal for MODE 1); on return
// v = L^{-1} (row i), by forward elimination with shuffled rows.
template <int MODE>
__device__ __forceinline__ bool block16(double (&r)[DB], double (&v)[DB], int lane, int* badc) {
  const unsigned full = 0xffffffffu;
  // inverse by forward elimination on [L | I]: row t final after scaling; rows i > t drop L(i,t) row t
#pragma unroll
  for (int j = 0; j < DB; ++j) v[j] = (lane == j) ? 1.0 : 0.0;
#pragma unroll
  for (int t = 0; t < DB; ++t) {
    const double inv = MODE == 1 ? 1.0 : 1.0 / __shfl_sync(full, r[t], t);
    if (lane == t) {
#pragma unroll
      for (int j = 0; j <= t; ++j) v[j] *= inv;
    }
#pragma unroll
    for (int j = 0; j <= t; ++j) {
      const double wt = __shfl_sync(full, v[j], t);
      if (lane > t && lane < DB) v[j] = fma(-r[t], wt, v[j]);
    }
  }
  return true;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_diag_inv(double* G, int64_t ld, int jb, double* W, int64_t ldw,
                                                  int64_t col0, int64_t* status) {
  dev::griddep_wait();
  if (status && *status != 0) return;
  extern __shared__ double dinv_sm[];
  double (*a)[TB2 + 1] = reinterpret_cast<double (*)[TB2 + 1]>(dinv_sm);
  double (*w)[TB2 + 1] = reinterpret_cast<double (*)[TB2 + 1]>(dinv_sm + TB2 * (TB2 + 1));
  double* tmp = dinv_sm + 2 * TB2 * (TB2 + 1);                      // [3][DB][DB]
  __shared__ int bad;
  __shared__ double rdg[TB2];                                        // 1 / L(c, c) (MODE 0)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad = 0;
  for (int e = tid; e < TB2 * TB2; e += 256) {          // cp.async: all loads in flight at once
    const int i = e & (TB2 - 1), j = e >> 6;
    if (i < jb && j < jb) dev::cp_async8(&a[i][j], G + i + j * ld, true);
    else a[i][j] = i == j ? 1.0 : 0.0;
    w[i][j] = 0.0;
  }
  dev::cp_async_commit();
  dev::cp_async_wait<0>();
  __syncthreads();
  if (MODE == 0) {
    for (int c0 = 0; c0 < TB2; c0 += DB) {
      if (warp == 0) {
        // factor the diagonal block in shared memory, one column per step; the trailing update of
        // the block is two-phase (all loads, then FMAs and stores) so its loads overlap
        const int i = c0 + 1 + (lane & 15);                          // row offset added per column below
        for (int c = c0; c < c0 + DB; ++c) {
          const double d = a[c][c];
          if (!(d > 0.0)) {
            if (lane == 0) bad = c + 1;
            break;
          }
          const double rs = rsqrt(d);
          __syncwarp();
          if (lane == 0) { a[c][c] = d * rs; rdg[c] = rs; }
          if (lane < c0 + DB - c - 1) a[c + 1 + lane][c] *= rs;
          __syncwarp();
          const int ii = c + 1 + (lane & 15);
          const int jb0 = c + 1 + (lane >> 4);
          double lj[8], aij[8];
          const double li = ii < c0 + DB ? a[ii][c] : 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = jb0 + 2 * q;
            const bool ok = ii < c0 + DB && j <= ii;
            lj[q] = ok ? a[j][c] : 0.0;
            aij[q] = ok ? a[ii][j] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int j = jb0 + 2 * q;
            if (ii < c0 + DB && j <= ii) a[ii][j] = fma(-li, lj[q], aij[q]);
          }
          __syncwarp();
        }
        (void)i;
      }
      __syncthreads();
      if (bad) {
        if (tid == 0 && status && bad <= jb) *status = col0 + bad;
        if (bad <= jb) return;
        __syncthreads();
        if (tid == 0) bad = 0;                                       // pivot in the identity padding
      }
      // panel: rows i >= c0 + 16, L(i, :) = A(i, :) L_pp^{-T} by forward substitution (one row per thread)
      for (int i = c0 + DB + tid; i < TB2; i += 256) {
        double x[DB];
#pragma unroll
        for (int j = 0; j < DB; ++j) {
          double v = a[i][c0 + j];
#pragma unroll
          for (int q = 0; q < j; ++q) v = fma(-x[q], a[c0 + j][c0 + q], v);
          x[j] = v * rdg[c0 + j];
        }
#pragma unroll
        for (int j = 0; j < DB; ++j) a[i][c0 + j] = x[j];
      }
      __syncthreads();
      // trailing update of the lower triangle: A(i, j) -= L(i, panel) . L(j, panel)
      {
        const int ti = tid >> 4, tj = tid & 15;
        for (int i = c0 + DB + ti; i < TB2; i += 16)
          for (int j = c0 + DB + tj; j <= i; j += 16) {
            double v = a[i][j];
#pragma unroll
            for (int q = 0; q < DB; ++q) v = fma(-a[i][c0 + q], a[j][c0 + q], v);
            a[i][j] = v;
          }
      }
      __syncthreads();
    }
  }
  {                                                                  // invert the 4 diagonal blocks (warp p)
    if (warp < TB2 / DB) {
      const int c0 = warp * DB, i = lane & (DB - 1);
      double r[DB], v[DB];
#pragma unroll
      for (int j = 0; j < DB; ++j) r[j] = (j <= i) ? a[c0 + i][c0 + j] : 0.0;
      int badc = 0;
      block16<MODE == 1 ? 1 : 2>(r, v, lane, &badc);
      if (lane < DB) {
#pragma unroll
        for (int j = 0; j < DB; ++j) w[c0 + i][c0 + j] = j <= i ? v[j] : 0.0;
      }
    }
    __syncthreads();
  }
  // off-diagonal blocks by block distance d: W_ij = -W_ii * sum_{k=j}^{i-1} L_ik W_kj
  for (int d = 1; d < TB2 / DB; ++d) {
    const int npair = TB2 / DB - d;
    for (int e = tid; e < npair * DB * DB; e += 256) {
      const int pr = e / (DB * DB), r = (e / DB) % DB, cc = e % DB;
      const int bj = pr, bi = pr + d;
      double v = 0.0;
      for (int k = bj * DB; k < bi * DB; ++k) v = fma(a[bi * DB + r][k], w[k][bj * DB + cc], v);
      tmp[pr * DB * DB + r * DB + cc] = v;
    }
    __syncthreads();
    for (int e = tid; e < npair * DB * DB; e += 256) {
      const int pr = e / (DB * DB), r = (e / DB) % DB, cc = e % DB;
      const int bj = pr, bi = pr + d;
      double v = 0.0;
      for (int q = 0; q <= r; ++q) v = fma(w[bi * DB + r][bi * DB + q], tmp[pr * DB * DB + q * DB + cc], v);
      w[bi * DB + r][bj * DB + cc] = -v;
    }
    __syncthreads();
  }
  for (int e = tid; e < TB2 * TB2; e += 256) {
    const int i = e & (TB2 - 1), jj = e >> 6;
    if (i < jb && jj < jb) {
      W[i + jj * ldw] = jj <= i ? w[i][jj] : 0.0;
      if (MODE == 0) G[i + jj * ld] = jj <= i ? a[i][jj] : 0.0;
    }
  }
}

// X (rows x jb, ldx) <- X * M in place, M = W^T (TRANS) or W, W jb x jb (ldw).  A CTA owns 64 whole
// rows, so reading and writing X never race.  DMMA m8n8k4: warp w computes rows 8w..8w+7 x the 64
// columns (8 accumulator tiles) over K = 64; both shared tiles use a row stride of 68 doubles
// (= 4 mod 16), which makes the 8x4 A-fragment and 4x8 B-fragment loads conflict-free.
constexpr int RTS = TB2 + 4;
template <bool TRANS>
__global__ void __launch_bounds__(256) k_right_tri_mul(double* X, int64_t rows, int64_t ldx, const double* W,
                                                       int64_t ldw, int jb) {
  dev::griddep_wait();
  extern __shared__ double rtm_sm[];
  double (*m)[RTS] = reinterpret_cast<double (*)[RTS]>(rtm_sm);                  // m[t][c] = M(t, c)
  double (*x)[RTS] = reinterpret_cast<double (*)[RTS]>(rtm_sm + TB2 * RTS);      // x[rr][t] = X(r0+rr, t)
  // both tiles by 8-byte cp.async (zero-fill outside), all in flight at once: a load-then-store
  // loop would serialise 32 global round trips per thread
  for (int e = threadIdx.x; e < TB2 * TB2; e += 256) {   // coalesced along W's leading dimension
    const int f = e % TB2, g = e / TB2;
    const bool ok = f < jb && g < jb;
    dev::cp_async8(TRANS ? &m[g][f] : &m[f][g], ok ? W + f + (int64_t)g * ldw : W, ok);   // M(t,c) = W(c,t) / W(t,c)
  }
  const int64_t r0 = (int64_t)blockIdx.x * TB2;
  for (int e = threadIdx.x; e < TB2 * TB2; e += 256) {
    const int rr = e % TB2, t = e / TB2;
    const int64_t r = r0 + rr;
    const bool ok = r < rows && t < jb;
    dev::cp_async8(&x[rr][t], ok ? X + r + t * ldx : X, ok);
  }
  dev::cp_async_commit();
  dev::cp_async_wait<0>();
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
  for (int kk = 0; kk < TB2 / 4; ++kk) {
    const double a = x[8 * w + g][4 * kk + q];
#pragma unroll
    for (int j = 0; j < 8; ++j) dev::dmma_8x8x4(acc[j][0], acc[j][1], a, m[4 * kk + q][8 * j + g]);
  }
  const int64_t r = r0 + 8 * w + g;
  if (r < rows) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = 8 * j + 2 * q;
      if (c < jb) X[r + c * ldx] = acc[j][0];
      if (c + 1 < jb) X[r + (c + 1) * ldx] = acc[j][1];
    }
  }
}
// Out (cols x rows, ldout) = In^T for In rows x cols (ldin), both column-major; 32 x 32 tiles.
__global__ void k_transpose_any(const double* In, int64_t rows, int64_t cols, int64_t ldin, double* Out,
                                int64_t ldout) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + r;
    if (i < rows && j < cols) tile[r][threadIdx.x] = In[i + j * ldin];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + r;
    if (i < rows && j < cols) Out[j + i * ldout] = tile[threadIdx.x][r];
  }
}

__global__ void k_upper_triangle(const double* B, int64_t ldb, int64_t n, double* R, int64_t ldr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    R[i + j * ldr] = i <= j ? B[i + j * ldb] : 0.0;
  }
}

constexpr size_t kDiagInvSmem = (2 * TB2 * (TB2 + 1) + 3 * DB * DB) * sizeof(double);
constexpr size_t kRtmSmem = 2 * TB2 * RTS * sizeof(double);

sk_status dense_attrs(sk_ctx* c) {
  static bool done_dev[kMaxDevices] = {};                  // function attributes are per device
  bool& done = done_dev[c->device % kMaxDevices];
  if (done) return SK_OK;
  SK_CUDA(c, cudaFuncSetAttribute(k_diag_inv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagInvSmem));
  SK_CUDA(c, cudaFuncSetAttribute(k_diag_inv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagInvSmem));
  SK_CUDA(c, cudaFuncSetAttribute(k_diag_inv<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDiagInvSmem));
  SK_CUDA(c, cudaFuncSetAttribute(k_right_tri_mul<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRtmSmem));
  SK_CUDA(c, cudaFuncSetAttribute(k_right_tri_mul<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRtmSmem));
  done = true;
  return SK_OK;
}

}  // namespace

sk_status gather_cols(sk_ctx* c, const double* A, int64_t m, int64_t lda, const int64_t* J, int64_t k,
                      double* C, int64_t ldc) {
  return gather_cols_shard(c, A, m, lda, 0, INT64_MAX, J, k, C, ldc);
}

sk_status upper_triangle(sk_ctx* c, const double* B, int64_t ldb, int64_t n, double* R, int64_t ldr) {
  if (n == 0) return SK_OK;
  const int blocks = (int)std::min<int64_t>(cdiv(n * n, 256), 4LL * c->num_sms);
  k_upper_triangle<<<blocks, 256, 0, c->stream>>>(B, ldb, n, R, ldr);
  return launched(c);
}

sk_status transpose(sk_ctx* c, const double* In, int64_t rows, int64_t cols, int64_t ldin, double* Out,
                    int64_t ldout) {
  if (rows == 0 || cols == 0) return SK_OK;
  const dim3 g((unsigned)cdiv(rows, 32), (unsigned)cdiv(cols, 32));
  if (g.y > 65535) return fail(c, SK_E_ARG, "transpose: too many columns");
  k_transpose_any<<<g, dim3(32, 8), 0, c->stream>>>(In, rows, cols, ldin, Out, ldout);
  return launched(c);
}

sk_status gather_cols_shard(sk_ctx* c, const double* A, int64_t m, int64_t lda, int64_t col0, int64_t ncols,
                            const int64_t* J, int64_t k, double* C, int64_t ldc) {
  if (m == 0 || k == 0) return SK_OK;
  const unsigned bx = (unsigned)std::min<int64_t>(cdiv(m, 256), 64);
  k_gather_cols<<<dim3(bx, (unsigned)k), 256, 0, c->stream>>>(A, m, lda, J, k, col0, ncols, C, ldc);
  return launched(c);
}

sk_status gather_rows_t(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I, int64_t k,
                        double* Rt, int64_t ldrt) {
  if (k == 0 || n == 0) return SK_OK;
  const int bx = (int)std::min<int64_t>(cdiv(n, 256), 64);
  k_gather_rows_t<<<dim3(bx, (unsigned)k), 256, 0, c->stream>>>(A, m, n, lda, I, k, Rt, ldrt);
  return launched(c);
}

sk_status potrf_lower(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t* status_dev) {
  SK_TRY(dense_attrs(c));
  // right-looking, 64-wide blocks: L_jj and W_jj = L_jj^{-1} in one CTA, panel L_rj = G_rj W_jj^T
  // in place, trailing update by DMMA GEMM.  The W_jj blocks are kept (diagonal of c->tri_w) for
  // the triangular solve that follows.
  DBuf Wd;
  SK_TRY(Wd.alloc(c, (size_t)k * TB2 * sizeof(double)));
  for (int64_t j0 = 0; j0 < k; j0 += TB2) {
    const int jb = (int)std::min<int64_t>(TB2, k - j0);
    SK_TRY(launch_pdl(c, k_diag_inv<0>, dim3(1), dim3(256), kDiagInvSmem, G + j0 + j0 * ld, ld, jb,
                      Wd.as<double>() + j0, (int64_t)k, j0, status_dev));
    const int64_t j1 = j0 + jb;
    if (j1 < k) {
      const int64_t rows = k - j1;
      SK_TRY(launch_pdl(c, k_right_tri_mul<true>, dim3((unsigned)cdiv(rows, TB2)), dim3(256), kRtmSmem,
                        G + j1 + j0 * ld, rows, ld, (const double*)(Wd.as<double>() + j0), (int64_t)k, jb));
      c->pdl = true;
      const sk_status gs = gemm(c, false, true, rows, rows, jb, -1.0, G + j1 + j0 * ld, ld, G + j1 + j0 * ld, ld, 1.0,
                                G + j1 + j1 * ld, ld);
      c->pdl = false;
      SK_TRY(gs);
    }
  }
  return SK_OK;
}

sk_status trsm_right_lt(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                        int64_t ldl) {
  SK_TRY(dense_attrs(c));
  // X_j <- (X_j - X_<j L_j,<j^T) L_jj^{-T}, 64-wide blocks; L_jj^{-1} re-formed per block (cheap)
  DBuf Wd;
  SK_TRY(Wd.alloc(c, (size_t)TB2 * TB2 * sizeof(double)));
  DBuf Lc;
  SK_TRY(Lc.alloc(c, (size_t)TB2 * TB2 * sizeof(double)));
  for (int64_t j0 = 0; j0 < k; j0 += TB2) {
    const int jb = (int)std::min<int64_t>(TB2, k - j0);
    // W = L_jj^{-1}: L_jj is already a Cholesky factor; invert it as a (non-unit) lower matrix
    SK_CUDA(c, cudaMemcpy2DAsync(Lc.p, TB2 * sizeof(double), L + j0 + j0 * ldl, ldl * sizeof(double),
                                 jb * sizeof(double), jb, cudaMemcpyDeviceToDevice, c->stream));
    SK_TRY(launch_pdl(c, k_diag_inv<2>, dim3(1), dim3(256), kDiagInvSmem, Lc.as<double>(), (int64_t)TB2, jb,
                      Wd.as<double>(), (int64_t)TB2, (int64_t)0, (int64_t*)nullptr));
    if (j0 > 0) {
      c->pdl = true;
      const sk_status gs = gemm(c, false, true, rows, jb, j0, -1.0, X, ldx, L + j0, ldl, 1.0, X + j0 * ldx, ldx);
      c->pdl = false;
      SK_TRY(gs);
    }
    SK_TRY(launch_pdl(c, k_right_tri_mul<true>, dim3((unsigned)cdiv(rows, TB2)), dim3(256), kRtmSmem, X + j0 * ldx,
                      rows, ldx, (const double*)Wd.as<double>(), (int64_t)TB2, jb));
  }
  return SK_OK;
}

template <int MODE>
static sk_status trsm_right_l_impl(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                                   int64_t ldl);

sk_status trsm_right_l_unit(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                            int64_t ldl) {
  return trsm_right_l_impl<1>(c, X, rows, k, ldx, L, ldl);
}

sk_status trsm_right_l(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L, int64_t ldl) {
  return trsm_right_l_impl<2>(c, X, rows, k, ldx, L, ldl);
}

// X <- X L^{-1} for a unit (MODE 1) or non-unit (MODE 2) lower L
template <int MODE>
static sk_status trsm_right_l_impl(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                                   int64_t ldl) {
  SK_TRY(dense_attrs(c));
  // X_j <- (X_j - X_>j L_>j,j) L_jj^{-1} (unit lower), 64-wide blocks from the last
  DBuf Wd, Lc;
  SK_TRY(Wd.alloc(c, (size_t)TB2 * TB2 * sizeof(double)));
  SK_TRY(Lc.alloc(c, (size_t)TB2 * TB2 * sizeof(double)));
  const int64_t nblk = cdiv(k, TB2);
  for (int64_t b = nblk - 1; b >= 0; --b) {
    const int64_t j0 = b * TB2;
    const int jb = (int)std::min<int64_t>(TB2, k - j0);
    const int64_t j1 = j0 + jb;
    SK_CUDA(c, cudaMemcpy2DAsync(Lc.p, TB2 * sizeof(double), L + j0 + j0 * ldl, ldl * sizeof(double),
                                 jb * sizeof(double), jb, cudaMemcpyDeviceToDevice, c->stream));
    SK_TRY(launch_pdl(c, k_diag_inv<MODE>, dim3(1), dim3(256), kDiagInvSmem, Lc.as<double>(), (int64_t)TB2, jb,
                      Wd.as<double>(), (int64_t)TB2, (int64_t)0, (int64_t*)nullptr));
    if (j1 < k) {
      c->pdl = true;
      const sk_status gs = gemm(c, false, false, rows, jb, k - j1, -1.0, X + j1 * ldx, ldx, L + j1 + j0 * ldl, ldl,
                                1.0, X + j0 * ldx, ldx);
      c->pdl = false;
      SK_TRY(gs);
    }
    SK_TRY(launch_pdl(c, k_right_tri_mul<false>, dim3((unsigned)cdiv(rows, TB2)), dim3(256), kRtmSmem,
                      X + j0 * ldx, rows, ldx, (const double*)Wd.as<double>(), (int64_t)TB2, jb));
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
  if ((size_t)k * sizeof(double) <= 96 * 1024) {      // x fits shared memory: one persistent launch
    const size_t smem = (size_t)k * sizeof(double);
    SK_CUDA(c, cudaFuncSetAttribute(k_power_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_power_persistent, 256, smem));
    const int nb = (int)std::min<int64_t>(std::min<int64_t>(c->num_sms, (int64_t)per_sm * c->num_sms), cdiv(k, 8));
    DBuf yb, pb, fb;
    SK_TRY(yb.alloc(c, (size_t)2 * k * sizeof(double)));
    SK_TRY(pb.alloc(c, (size_t)2 * nb * sizeof(double)));
    SK_TRY(fb.alloc(c, (size_t)nb * 16 * sizeof(unsigned long long)));
    SK_CUDA(c, cudaMemsetAsync(fb.p, 0, (size_t)nb * 16 * sizeof(unsigned long long), c->stream));
    double* y = yb.as<double>();
    double* pt = pb.as<double>();
    unsigned long long* fl = fb.as<unsigned long long>();
    int max_it = 4000;
    void* args[] = {(void*)&G, (void*)&k, (void*)&ld, (void*)&y, (void*)&pt, (void*)&fl, (void*)&out_dev, (void*)&max_it};
    SK_CUDA(c, cudaLaunchCooperativeKernel((void*)k_power_persistent, dim3(nb), dim3(256), args, smem, c->stream));
    return launched(c);
  }
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
