// dense.cu -- the small dense building blocks around the hot path:
//   gather (S3: C = A(:, J_s)), blocked Cholesky, blocked triangular solves,
//   two-pass Cholesky QR (ortho()) and a power iteration for ||T||_2 (Thm 4.1 eta).
// Heavy lifting is delegated to the DMMA GEMM (gemm.cu); the kernels here only handle
// the 32 x 32 diagonal blocks.
#include <algorithm>
#include <cmath>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dmma.cuh"
#include "internal.h"

namespace skel {
namespace {

namespace cg = cooperative_groups;

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

// ------------------------------------------------------------------ single-launch Cholesky and row solve
// The CholeskyQR chain (G = Q^T Q, G = L L^T, Q <- Q L^{-T}) as two launches instead of ~50:
//   k_potrf_cluster: right-looking Cholesky of a k x k SPD G (k <= 1024) by ONE cluster of 16 CTAs in
//     32-wide block steps p, phases separated by cluster barriers (release/acquire: they order the
//     global-memory updates; G stays in global memory, L2-resident, loads bypass L1):
//       D  one warp factors the diagonal block in registers (row per lane; pivot by shuffle, column
//          by shared memory, rsqrt by MUFU + one fourth-order step; tools/microbench/chol32_bench:
//          ~6k cycles per 32 columns);
//       P  L_ip = G_ip L_pp^{-T} by forward substitution (a warp per 32-row block, a row per lane),
//          and, off the critical path, W_pp = L_pp^{-1} by the same substitution on unit rows;
//       U  G_ij -= L_ip L_jp^T, 32 x 32 x 32 DMMA units spread over the cluster's 128 warps; the warp
//          that updates the next diagonal block factors it right away (D of step p+1 under U of p).
//   k_trsm_rows: X <- X L^{-T} (X rows x k) with no inter-CTA dependency: a CTA owns RB whole rows of X
//     in shared memory and walks the 32-wide column blocks, X_j = (X_j - sum_c X_c L_jc^T) W_jj^T,
//     row block j of L streamed in 32 x 64 chunks (then W_jj) through a cp.async ring.
constexpr int CB = 32;           // block width of both kernels
constexpr int CL = 16;           // cluster size of k_potrf_cluster
constexpr int kCholMaxK = 1024;
constexpr int LS = CB + 1;       // shared 32 x 32 tile stride

// x = g L^{-T} for one row per lane: x_t = (g_t - sum_{q<t} x_q L(t, q)) / L(t, t); Ls = L (stride LS),
// rinv[t] = 1 / L(t, t).  With g = e_lane it gives column `lane` of L^{-1}.
__device__ __forceinline__ void rowsolve32(double (&g)[CB], const double* Ls, const double* rinv) {
#pragma unroll
  for (int t = 0; t < CB; ++t) {
    g[t] *= rinv[t];
#pragma unroll
    for (int q = t + 1; q < CB; ++q) g[q] = fma(-g[t], Ls[q * LS + t], g[q]);
  }
}

// 1/sqrt(d) for a normal d > 0 without the library routine's slow-path call (which would spill the
// live row around every call site): the MUFU approximation refined by three Newton steps.
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  // one fourth-order step: e = 1 - d y^2, y' = y (1 + e/2 + 3e^2/8 + 5e^3/16), relative error ~e^4
  const double e = fma(-d * y, y, 1.0);
  const double p = fma(e, fma(0.3125, e, 0.375), 0.5);
  return fma(y * e, p, y);
}

// column T of the register Cholesky (template recursion: every register index is a literal, so the
// row never falls back to local memory)
template <int T>
struct Chol32Col {
  static __device__ __forceinline__ void run(double (&r)[CB], double* colbuf, int lane, int& bad) {
    double d = __shfl_sync(0xffffffffu, r[T], T);    // the pivot A(T, T), held by lane T
    if (!(d > 0.0)) {
      if (!bad) bad = T + 1;
      d = 1.0;
    }
    const double rs = rsqrt_nr(d);
    const double lit = lane == T ? d * rs : (lane > T ? r[T] * rs : 0.0);
    r[T] = lit;
    colbuf[(T & 1) * CB + lane] = lit;                 // column T of L, broadcast through shared memory
    __syncwarp();                                      // (double-buffered: no second barrier per column)
    double cj[CB];
#pragma unroll
    for (int j = T + 1; j < CB; ++j) cj[j] = colbuf[(T & 1) * CB + j];
    // unpredicated: lanes above the diagonal update entries that are never read (lit = 0 for lanes < T)
#pragma unroll
    for (int j = T + 1; j < CB; ++j) r[j] = fma(-lit, cj[j], r[j]);
    Chol32Col<T + 1>::run(r, colbuf, lane, bad);
  }
};
template <>
struct Chol32Col<CB> {
  static __device__ __forceinline__ void run(double (&)[CB], double*, int, int&) {}
};

// one warp: Cholesky of a 32 x 32 block held row-per-lane in registers (r[j] = A(lane, j), j <= lane),
// in place (r = row `lane` of L); colbuf: 64 doubles of shared scratch.  Returns the 1-based failing
// column (a failed pivot continues with 1 so no NaN spreads), 0 if none.
__device__ __forceinline__ int chol32_regs(double (&r)[CB], double* colbuf, int lane) {
  int bad = 0;
  Chol32Col<0>::run(r, colbuf, lane, bad);
  return bad;
}

// one warp: D (32 x 32 at (d0r, d0c), ldd) = sgn Aop Bop^T (+ D if ACC), Aop(i, kk) = A(a0r + i, a0c + kk),
// Bop(n, kk) = B(b0r + n, b0c + kk), K = 32 (column-major A, B, D), everything inside k x k.
// LOWER: only the 8 x 8 tiles on or below the diagonal.
template <bool ACC, bool LOWER>
__device__ __forceinline__ void unit32(const double* A, int a0r, int a0c, const double* B, int b0r, int b0c, double* D,
                                       int d0r, int d0c, int64_t ld, int k, double sgn, int lane) {
  const int g = lane >> 2, q = lane & 3;
  double bf[4][8];
#pragma unroll
  for (int bb = 0; bb < 4; ++bb)
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int rb = b0r + 8 * bb + g, cb = b0c + 4 * s + q;
      bf[bb][s] = (rb < k && cb < k) ? __ldcg(B + rb + (int64_t)cb * ld) : 0.0;
    }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double af[8];
    const int ra = a0r + 8 * a + g;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int ca = a0c + 4 * s + q;
      af[s] = (ra < k && ca < k) ? sgn * __ldcg(A + ra + (int64_t)ca * ld) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (LOWER && b > a) continue;
      const int r = d0r + 8 * a + g, c = d0c + 8 * b + 2 * q;
      const bool ok0 = r < k && c < k, ok1 = r < k && c + 1 < k;
      double c0 = 0.0, c1 = 0.0;
      if (ACC) {
        if (ok0) c0 = __ldcg(D + r + (int64_t)c * ld);
        if (ok1) c1 = __ldcg(D + r + (int64_t)(c + 1) * ld);
      }
#pragma unroll
      for (int s = 0; s < 8; ++s) dev::dmma_8x8x4(c0, c1, af[s], bf[b][s]);
      if (ok0) D[r + (int64_t)c * ld] = c0;
      if (ok1) D[r + (int64_t)(c + 1) * ld] = c1;
    }
  }
}

// G (k x k, ld, lower part read) -> L in place (strict upper triangle zeroed), Wd (kp x 32, ld ldw):
// rows 32p.. = L_pp^{-1}.  status: 1-based failing column on a non-positive pivot.
__global__ void __launch_bounds__(256, 1)
    k_potrf_cluster(double* G, int64_t ld, int k, double* Wd, int64_t ldw, int64_t* status) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ int fail;
  __shared__ double Ls[CB * LS], rinv[CB];
  const int rank = (int)cluster.block_rank(), warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = warp * CL + rank, nw = CL * 8;                     // consecutive units on different SMs
  const int nb = (k + CB - 1) / CB;
  if (threadIdx.x == 0) fail = status ? (int)(__ldcg(status) != 0) : 0;
  cluster.sync();
  const int* fail0 = cluster.map_shared_rank(&fail, 0);
  const bool f0 = *fail0 != 0;
  cluster.sync();                                                  // uniform decision, read before any write
  if (f0) return;
  // D (warp 0 of CTA 0): factor diagonal block p in registers, write L_pp back
  auto diag = [&](int p) {
    const int p0 = p * CB, i = p0 + lane;
    double r[CB];
#pragma unroll
    for (int j = 0; j < CB; ++j)
      r[j] = (i < k && j <= lane) ? __ldcg(G + i + (int64_t)(p0 + j) * ld) : (j == lane ? 1.0 : 0.0);
    const int bad = chol32_regs(r, Ls, lane);                      // (Ls: broadcast scratch here)
#pragma unroll
    for (int j = 0; j < CB; ++j)
      if (i < k && p0 + j < k) G[i + (int64_t)(p0 + j) * ld] = j <= lane ? r[j] : 0.0;
    if (bad && p0 + bad <= k && lane == 0) {
      fail = 1;
      if (status) *status = p0 + bad;
    }
  };
  if (gw == 0) diag(0);
  for (int p = 0; p < nb; ++p) {
    const int p0 = p * CB;
    cluster.sync();                                                // L_pp (and the step-(p-1) update) in place
    if (*fail0) {                                                  // every CTA sees the same flag
      cluster.sync();                                              // CTA 0 stays until all have read it
      return;
    }
    // P: L_ip = G_ip L_pp^{-T} (i > p) and W_pp = L_pp^{-1}; the mirrored upper block G_pi is zeroed
    const int npu = nb - p;                                        // units: row blocks p+1.., then W_pp
    if (rank < npu) {                                              // (unit u on CTA u % CL)
      __syncthreads();
      for (int e = threadIdx.x; e < CB * CB; e += 256) {
        const int r = e & 31, cc = e >> 5;
        Ls[r * LS + cc] = (p0 + r < k && cc <= r) ? __ldcg(G + (p0 + r) + (int64_t)(p0 + cc) * ld) : (r == cc ? 1.0 : 0.0);
      }
      __syncthreads();
      if (threadIdx.x < CB) rinv[threadIdx.x] = __drcp_rn(Ls[threadIdx.x * LS + threadIdx.x]);
      __syncthreads();
      for (int u = gw; u < npu; u += nw) {
        double x[CB];
        if (u < npu - 1) {
          const int i0 = (p + 1 + u) * CB, i = i0 + lane;
#pragma unroll
          for (int t = 0; t < CB; ++t) x[t] = (i < k && p0 + t < k) ? __ldcg(G + i + (int64_t)(p0 + t) * ld) : 0.0;
          rowsolve32(x, Ls, rinv);
#pragma unroll
          for (int t = 0; t < CB; ++t)
            if (i < k && p0 + t < k) {
              G[i + (int64_t)(p0 + t) * ld] = x[t];
              G[(p0 + t) + (int64_t)i * ld] = 0.0;
            }
        } else {
#pragma unroll
          for (int t = 0; t < CB; ++t) x[t] = t == lane ? 1.0 : 0.0;
          rowsolve32(x, Ls, rinv);                                 // x_t = L_pp^{-1}(t, lane)
#pragma unroll
          for (int t = 0; t < CB; ++t) Wd[(p0 + t) + (int64_t)lane * ldw] = x[t];
        }
      }
    }
    cluster.sync();
    // U: G_ij -= L_ip L_jp^T, p < j <= i (unit index -> (i, j) in the lower triangle).  Unit 0 is the
    // next diagonal block; its warp (gw 0) factors it right after updating it (look-ahead: the D of
    // step p+1 overlaps the rest of this update)
    const int nt = nb - p - 1;
    int ii = 0, jj = 0;
    for (int u = gw; u < nt * (nt + 1) / 2; u += nw) {
      while ((ii + 1) * (ii + 2) / 2 <= u) ++ii;                   // u increases: ii only moves forward
      jj = u - ii * (ii + 1) / 2;
      const int i0 = (p + 1 + ii) * CB, j0 = (p + 1 + jj) * CB;
      if (ii == jj) unit32<true, true>(G, i0, p0, G, j0, p0, G, i0, j0, ld, k, -1.0, lane);
      else unit32<true, false>(G, i0, p0, G, j0, p0, G, i0, j0, ld, k, -1.0, lane);
      if (u == 0) diag(p + 1);
    }
  }
}

// Wd (kp x 32) rows 32p.. = L_pp^{-1} for a lower L (k x k, ld): one warp per diagonal block
__global__ void __launch_bounds__(32) k_diag_inv32(const double* L, int64_t ld, int k, double* Wd, int64_t ldw) {
  __shared__ double Ls[CB * LS], rinv[CB];
  const int lane = threadIdx.x, p0 = blockIdx.x * CB;
  for (int j = 0; j < CB; ++j) {
    const int i = p0 + lane;
    Ls[lane * LS + j] = (i < k && j <= lane) ? L[i + (int64_t)(p0 + j) * ld] : (j == lane ? 1.0 : 0.0);
  }
  __syncwarp();
  rinv[lane] = __drcp_rn(Ls[lane * LS + lane]);
  __syncwarp();
  double x[CB];
#pragma unroll
  for (int t = 0; t < CB; ++t) x[t] = t == lane ? 1.0 : 0.0;
  rowsolve32(x, Ls, rinv);
#pragma unroll
  for (int t = 0; t < CB; ++t) Wd[(p0 + t) + (int64_t)lane * ldw] = x[t];
}

// Newton-Schulz step for a nearly orthonormal Q (second CholeskyQR pass): M = (3 I - G) / 2 with
// G = Q^T Q, and eta = max |G - I| (non-negative doubles order like their bit patterns).
__global__ void k_ns_prep(const double* G, int64_t k, double* M, unsigned long long* eta) {
  double mx = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % k, j = e / k;
    const double d = G[i >= j ? e : j + i * k] - (i == j ? 1.0 : 0.0);   // G's lower triangle (gram_lower)
    mx = fmax(mx, fabs(d));
    M[e] = (i == j ? 1.0 : 0.0) - 0.5 * d;
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(eta, (unsigned long long)__double_as_longlong(mx));
}

constexpr int TRS = CB + 4;      // ring / temp tile stride (doubles): conflict-free fragment reads
constexpr int TRR = 4;           // ring slots
constexpr int TKC = 64;          // L columns per ring slot

__host__ __device__ inline size_t trsm_rows_smem(int rb, int kp) {
  return ((size_t)rb * (kp + 4) + (size_t)TRR * TKC * TRS + (size_t)rb * TRS) * sizeof(double);
}

// X (rows x k, ldx) <- X L^{-T}; L lower (k x k, ldl), Wd = diagonal-block inverses (kp x 32, ldw).
// Stages, in order, for each column block j: chunks of row block j of L (columns [0, 32 j) in
// TKC-wide pieces), then W_jj.  A stage is described by (j, c0, width); width 0 = the W_jj stage.
template <int RB>
__global__ void __launch_bounds__(256) k_trsm_rows(double* X, int64_t rows, int64_t ldx, int k, const double* L,
                                                   int64_t ldl, const double* Wd, int64_t ldw) {
  extern __shared__ __align__(16) double trs_sm[];
  const int nb = (k + CB - 1) / CB, kp = nb * CB, xst = kp + 4;
  double* xs = trs_sm;                                   // [RB][kp + 4]: xs[r][t] = X(r0 + r, t)
  double* ring = xs + (size_t)RB * xst;                  // [TRR][TKC][TRS]: S[kk][n]
  double* tt = ring + (size_t)TRR * TKC * TRS;           // [RB][TRS]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, g = lane >> 2, q = lane & 3;
  constexpr int TPW = RB / 16;                           // 8 x 8 tiles per warp (same column tile b)
  const int b = w & 3, abase = TPW * (w >> 2);
  const int64_t r0 = (int64_t)blockIdx.x * RB;
  const bool vec = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(L) & 15) == 0);
  for (int e = tid; e < RB * kp; e += 256) {
    const int rr = e % RB, t = e / RB;
    const bool ok = r0 + rr < rows && t < k;
    dev::cp_async8(xs + (size_t)rr * xst + t, ok ? X + (r0 + rr) + (int64_t)t * ldx : X, ok);
  }
  // issuer state (uniform): the next stage to load
  int ij = 0, ic = 0, nis = 0;
  auto issue = [&]() {
    if (ij < nb) {
      double* S = ring + (size_t)(nis % TRR) * TKC * TRS;
      if (ic < ij * CB) {                                // L(32 ij + n, ic + kk), kk < width
        const int wdt = min(TKC, ij * CB - ic);
        if (vec) {
          for (int e = tid; e < wdt * (CB / 2); e += 256) {
            const int n2 = 2 * (e & 15), kk = e >> 4;
            const int rowg = ij * CB + n2, colg = ic + kk;
            const int nbytes = colg < k ? 8 * max(0, min(2, k - rowg)) : 0;
            dev::cp_async16(S + kk * TRS + n2, nbytes ? L + rowg + (int64_t)colg * ldl : L, nbytes);
          }
        } else {
          for (int e = tid; e < wdt * CB; e += 256) {
            const int n = e & 31, kk = e >> 5;
            const int rowg = ij * CB + n, colg = ic + kk;
            const bool ok = rowg < k && colg < k;
            dev::cp_async8(S + kk * TRS + n, ok ? L + rowg + (int64_t)colg * ldl : L, ok);
          }
        }
        ic += wdt;
      } else {                                           // W_jj(n, kk) = Wd(32 ij + n, kk)
        for (int e = tid; e < CB * (CB / 2); e += 256) {
          const int n2 = 2 * (e & 15), kk = e >> 4;
          dev::cp_async16(S + kk * TRS + n2, Wd + (ij * CB + n2) + (int64_t)kk * ldw, 16);
        }
        ++ij;
        ic = 0;
      }
      ++nis;
    }
    dev::cp_async_commit();
  };
  for (int st = 0; st < TRR - 1; ++st) issue();
  double acc[TPW][2];
  int j = 0, c = 0, st = 0;
  while (j < nb) {
    dev::cp_async_wait<TRR - 2>();
    __syncthreads();
    issue();
    const double* S = ring + (size_t)(st % TRR) * TKC * TRS;
    ++st;
    if (c == 0) {
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        const double* xr = xs + (size_t)(8 * (abase + t) + g) * xst + j * CB + 8 * b + 2 * q;
        acc[t][0] = xr[0];
        acc[t][1] = xr[1];
      }
    }
    if (c < j * CB) {                                    // acc -= X(:, c..c+wdt) L(j block, c..c+wdt)^T
      const int wdt = min(TKC, j * CB - c);
      for (int s = 0; s < wdt / 4; ++s) {
        const double bv = S[(4 * s + q) * TRS + 8 * b + g];
#pragma unroll
        for (int t = 0; t < TPW; ++t)
          dev::dmma_8x8x4(acc[t][0], acc[t][1], -xs[(size_t)(8 * (abase + t) + g) * xst + c + 4 * s + q], bv);
      }
      c += wdt;
    } else {                                             // X_j = acc W_jj^T
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        double* tr = tt + (8 * (abase + t) + g) * TRS + 8 * b + 2 * q;
        tr[0] = acc[t][0];
        tr[1] = acc[t][1];
        acc[t][0] = acc[t][1] = 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const double bv = S[(4 * s + q) * TRS + 8 * b + g];
#pragma unroll
        for (int t = 0; t < TPW; ++t)
          dev::dmma_8x8x4(acc[t][0], acc[t][1], tt[(8 * (abase + t) + g) * TRS + 4 * s + q], bv);
      }
#pragma unroll
      for (int t = 0; t < TPW; ++t) {
        double* xr = xs + (size_t)(8 * (abase + t) + g) * xst + j * CB + 8 * b + 2 * q;
        xr[0] = acc[t][0];
        xr[1] = acc[t][1];
      }
      ++j;
      c = 0;
    }
  }
  dev::cp_async_wait<0>();
  __syncthreads();
  for (int e = tid; e < RB * k; e += 256) {
    const int rr = e % RB, t = e / RB;
    if (r0 + rr < rows) X[(r0 + rr) + (int64_t)t * ldx] = xs[(size_t)rr * xst + t];
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

namespace {
// the single-launch pair (k <= kCholMaxK): Cholesky with the diagonal-block inverses kept in Wd
// (kp x 32), and the row-block solve X <- X L^{-T}
sk_status potrf_cluster(sk_ctx* c, double* G, int64_t k, int64_t ld, double* Wd, int64_t ldw, int64_t* status_dev) {
  static bool attr_done[kMaxDevices] = {};
  if (!attr_done[c->device % kMaxDevices]) {
    SK_CUDA(c, cudaFuncSetAttribute(k_potrf_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done[c->device % kMaxDevices] = true;
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(CL);
  lc.blockDim = dim3(256);
  lc.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  lc.attrs = at; lc.numAttrs = 1;
  SK_CUDA(c, cudaLaunchKernelEx(&lc, k_potrf_cluster, G, ld, (int)k, Wd, ldw, status_dev));
  return launched(c);
}

sk_status trsm_rows(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L, int64_t ldl,
                    const double* Wd, int64_t ldw) {
  if (rows == 0) return SK_OK;
  const int kp = (int)cdiv(k, CB) * CB;
  // rows per CTA: as many as shared memory holds beside the ring (more rows amortise the L stream)
  const int rb = kp <= 256 ? 64 : (kp <= 512 ? 32 : 16);
  const size_t smem = trsm_rows_smem(rb, kp);
  if (rb == 64) {
    SK_CUDA(c, cudaFuncSetAttribute(k_trsm_rows<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_trsm_rows<64><<<(unsigned)cdiv(rows, 64), 256, smem, c->stream>>>(X, rows, ldx, (int)k, L, ldl, Wd, ldw);
  } else if (rb == 32) {
    SK_CUDA(c, cudaFuncSetAttribute(k_trsm_rows<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_trsm_rows<32><<<(unsigned)cdiv(rows, 32), 256, smem, c->stream>>>(X, rows, ldx, (int)k, L, ldl, Wd, ldw);
  } else {
    SK_CUDA(c, cudaFuncSetAttribute(k_trsm_rows<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_trsm_rows<16><<<(unsigned)cdiv(rows, 16), 256, smem, c->stream>>>(X, rows, ldx, (int)k, L, ldl, Wd, ldw);
  }
  return launched(c);
}
}  // namespace

sk_status potrf_lower(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t* status_dev) {
  SK_TRY(dense_attrs(c));
  if (k <= kCholMaxK) {
    DBuf Wd;
    SK_TRY(Wd.alloc(c, (size_t)cdiv(k, CB) * CB * CB * sizeof(double)));
    return potrf_cluster(c, G, k, ld, Wd.as<double>(), cdiv(k, CB) * CB, status_dev);
  }
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
  if (k <= kCholMaxK) {
    const int64_t kp = cdiv(k, CB) * CB;
    DBuf Wd;
    SK_TRY(Wd.alloc(c, (size_t)kp * CB * sizeof(double)));
    k_diag_inv32<<<(unsigned)(kp / CB), 32, 0, c->stream>>>(L, ldl, (int)k, Wd.as<double>(), kp);
    SK_TRY(launched(c));
    return trsm_rows(c, X, rows, k, ldx, L, ldl, Wd.as<double>(), kp);
  }
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
  if (k <= kCholMaxK) {
    // per pass: Gram (DMMA GEMM, lower tiles), Cholesky (one cluster launch), Q <- Q L^{-T} (one launch)
    const int64_t kp = cdiv(k, CB) * CB;
    DBuf Wd;
    SK_TRY(Wd.alloc(c, (size_t)kp * CB * sizeof(double)));
    SK_TRY(gram_lower(c, Q, m, k, ldq, G.as<double>(), k));
    SK_TRY(potrf_cluster(c, G.as<double>(), k, k, Wd.as<double>(), kp, status_dev));
    SK_TRY(trsm_rows(c, Q, m, k, ldq, G.as<double>(), k, Wd.as<double>(), kp));
    return cholqr_tail(c, Q, m, k, ldq, status_dev);
  }
  for (int pass = 0; pass < 2; ++pass) {
    SK_TRY(gemm(c, true, false, k, k, m, 1.0, Q, ldq, Q, ldq, 0.0, G.as<double>(), k));
    SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
    SK_TRY(trsm_right_lt(c, Q, m, k, ldq, G.as<double>(), k));
  }
  return SK_OK;
}

// The second CholeskyQR pass (k <= kCholMaxK): Gram, then one Newton-Schulz step when the pass before
// left |Q^T Q - I| <= 1e-10, else a Cholesky pass.
sk_status cholqr_tail(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev) {
  DBuf G;
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  {
    const int64_t kp = cdiv(k, CB) * CB;
    DBuf Wd;
    SK_TRY(Wd.alloc(c, (size_t)kp * CB * sizeof(double)));
    // second pass: after the first, Q^T Q = I + E with |E| ~ u cond(Q_0)^2.  When |E| <= 1e-10 one
    // Newton-Schulz step Q <- Q (3 I - Q^T Q) / 2 leaves |E|^2 (below u: the orthogonality CholeskyQR2
    // reaches) with two GEMMs and no sequential chain, and moves Q from the thin-QR factor by at most
    // |E| / 2 (a symmetric right factor); otherwise the Cholesky pass again.
    SK_TRY(gram_lower(c, Q, m, k, ldq, G.as<double>(), k));
    DBuf M, eta;
    SK_TRY(M.alloc(c, (size_t)k * k * sizeof(double)));
    SK_TRY(eta.alloc(c, sizeof(unsigned long long)));
    SK_CUDA(c, cudaMemsetAsync(eta.p, 0, sizeof(unsigned long long), c->stream));
    k_ns_prep<<<(unsigned)std::min<int64_t>(cdiv(k * k, 256), 2LL * c->num_sms), 256, 0, c->stream>>>(
        G.as<double>(), k, M.as<double>(), eta.as<unsigned long long>());
    SK_TRY(launched(c));
    unsigned long long eb = 0;
    SK_CUDA(c, cudaMemcpyAsync(&eb, eta.p, sizeof(eb), cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    double e;
    memcpy(&e, &eb, sizeof(e));
    if (e <= 1e-10) {
      DBuf T;
      SK_TRY(T.alloc(c, (size_t)m * k * sizeof(double)));
      SK_TRY(gemm(c, false, false, m, k, k, 1.0, Q, ldq, M.as<double>(), k, 0.0, T.as<double>(), m));
      SK_CUDA(c, cudaMemcpy2DAsync(Q, (size_t)ldq * sizeof(double), T.p, (size_t)m * sizeof(double),
                                   (size_t)m * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
      return SK_OK;
    }
    SK_TRY(potrf_cluster(c, G.as<double>(), k, k, Wd.as<double>(), kp, status_dev));
    return trsm_rows(c, Q, m, k, ldq, G.as<double>(), k, Wd.as<double>(), kp);
  }
}

// max L(i, i) / min L(i, i) of a Cholesky factor (a lower bound on its condition number) into out[0],
// +inf when the factorisation reported a breakdown (status != 0); one CTA
__global__ void k_diag_ratio(const double* L, int64_t k, int64_t ld, const int64_t* status, double* out) {
  __shared__ double smx[32], smn[32];
  double mx = 0.0, mn = INFINITY;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) {
    const double d = fabs(L[i + i * ld]);
    mx = fmax(mx, d);
    mn = fmin(mn, d);
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if ((threadIdx.x & 31) == 0) { smx[threadIdx.x >> 5] = mx; smn[threadIdx.x >> 5] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mx = fmax(mx, smx[w]); mn = fmin(mn, smn[w]); }
    out[0] = (*status != 0 || !(mn > 0.0)) ? INFINITY : mx / mn;
  }
}

// The first pass of the residual's orthonormal basis (k <= kCholMaxK) with the shift only where it is
// needed: G = Q^T Q is factored twice AT ONCE -- unshifted on the context stream, shifted (shifted
// CholeskyQR3's s = 11 (m k + k (k + 1)) u tr G) on the helper stream, each one 16-CTA cluster -- and
// the unshifted factor is used when it exists and max L_ii / min L_ii <= 1e3 (cond(Q) about that, so
// the next Gram shows |Q^T Q - I| ~ cond^2 u <= 1e-10 and one Newton-Schulz step finishes: two passes
// instead of three; C3 and C4 have cond(C) ~ 5e2, C2 1.6e11).  Then the CholeskyQR tail.
sk_status cholqr_adaptive(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev) {
  const int64_t kp = cdiv(k, CB) * CB;
  DBuf G, Gs, Wu, Ws, su, rb;
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Gs.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Wu.alloc(c, (size_t)kp * CB * sizeof(double)));
  SK_TRY(Ws.alloc(c, (size_t)kp * CB * sizeof(double)));
  SK_TRY(su.alloc(c, sizeof(int64_t)));
  SK_TRY(rb.alloc(c, sizeof(double)));
  SK_TRY(gram_lower(c, Q, m, k, ldq, G.as<double>(), k));
  SK_CUDA(c, cudaMemcpyAsync(Gs.p, G.p, (size_t)k * k * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  SK_CUDA(c, cudaMemsetAsync(su.p, 0, sizeof(int64_t), c->stream));
  SK_TRY(add_shift(c, Gs.as<double>(), k, k, m));
  SK_TRY(ensure_aux(c));
  SK_CUDA(c, cudaEventRecord(c->ev_a, c->stream));
  SK_CUDA(c, cudaStreamWaitEvent(c->aux, c->ev_a, 0));
  cudaStream_t main_stream = c->stream;
  c->stream = c->aux;
  const sk_status ss = potrf_cluster(c, Gs.as<double>(), k, k, Ws.as<double>(), kp, status_dev);
  c->stream = main_stream;
  SK_TRY(ss);
  SK_CUDA(c, cudaEventRecord(c->ev_b, c->aux));
  SK_TRY(potrf_cluster(c, G.as<double>(), k, k, Wu.as<double>(), kp, su.as<int64_t>()));
  k_diag_ratio<<<1, 256, 0, c->stream>>>(G.as<double>(), k, k, su.as<int64_t>(), rb.as<double>());
  SK_TRY(launched(c));
  SK_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_b, 0));
  double ratio = INFINITY;
  SK_CUDA(c, cudaMemcpyAsync(&ratio, rb.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  if (ratio <= 1e3) {
    SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));   // the shifted run is not used
    SK_TRY(trsm_rows(c, Q, m, k, ldq, G.as<double>(), k, Wu.as<double>(), kp));
    return cholqr_tail(c, Q, m, k, ldq, status_dev);
  }
  SK_TRY(trsm_rows(c, Q, m, k, ldq, Gs.as<double>(), k, Ws.as<double>(), kp));
  return cholqr2(c, Q, m, k, ldq, status_dev);
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
