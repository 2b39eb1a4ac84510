// deim.cu -- RSVD-DEIM column skeletons (the paper's pivoting comparator,
// Sec. 5 item 3; eq:rsvd_procedures P:237-243):
//     Q_X = ortho(X^T)                    (n x l, X = Gamma A the row sketch)
//     [U, S, V~] = svd(A Q_X, 'econ'),   V^ = Q_X V~               (eq:rsvd_procedures)
//     J_s = DEIM on V^(:, 0:k) = column-wise LUPP of V^(:, 0:k)^T  (Sorensen-Embree)
// Every step runs in this library's kernels:
//   * Q_X: the LUPP-basis CholeskyQR2 of S6 (shifted CholeskyQR3 for very tall panels);
//   * B = A Q_X (m x l): the DMMA GEMM;
//   * the l x l triangular factor of B without a Householder QR: the row LUPP of B gives
//     B = Lf U with |Lf| <= 1 (well conditioned), CholeskyQR2 gives Lf = Q_L R_L with R_L = Q_L^T Lf,
//     so B = Q_L (R_L U) and R = R_L U has the right singular vectors of B (and B's conditioning is
//     never squared -- a Gram / eigh route would lose the trailing vectors at C2's 1e10 range);
//   * svd(R)'s right factor: one-sided (Hestenes) Jacobi on the columns of R in ONE cooperative
//     launch -- round-robin pairings, one warp per column pair (the three dot products, the
//     rotation of R's and V's columns), a grid barrier per round, sweeps until no pair needs a
//     rotation (|r_p . r_q| <= 1e-15 ||r_p|| ||r_q||); sigma_j = ||R(:, j)||, columns sorted by
//     decreasing sigma (host argsort of l values);
//   * V^_k = Q_X V~(:, 0:k) by the DMMA GEMM and DEIM = the cluster LUPP.
// (Round 1 used cuSOLVER's geqrf + gesvd for the two small factorisations.)
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace skel {

namespace {

__device__ __forceinline__ void jac_grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1u) : "memory");
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
      } while (v == g);
    }
  }
  __syncthreads();
}

// One-sided Jacobi on the columns of R (lp x lp, column-major, lp even; padded columns are zero):
// R <- R J, V <- V J with J the product of the rotations; on return R = U Sigma (columns), V = V~.
// sync[0..1] = grid barrier (count, generation), sync[2..] per-sweep "rotated" flags.
__global__ void __launch_bounds__(256) k_jacobi_svd(double* R, double* V, int lp, int max_sweeps, unsigned* sync) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const unsigned nb = gridDim.x;
  const int npair = lp / 2;
  for (int sw = 0; sw < max_sweeps; ++sw) {
    unsigned* rotated = sync + 2 + sw;
    for (int r = 0; r < lp - 1; ++r) {
      for (int pi = blockIdx.x * warps + warp; pi < npair; pi += (int)nb * warps) {
        // circle method: position 0 fixed, the others rotate by r
        const int a0 = pi, b0 = lp - 1 - pi;
        int p = a0 == 0 ? 0 : 1 + (a0 - 1 + r) % (lp - 1);
        int q = 1 + (b0 - 1 + r) % (lp - 1);
        if (p > q) { const int t = p; p = q; q = t; }
        double* rp = R + (int64_t)p * lp;
        double* rq = R + (int64_t)q * lp;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < lp; i += 32) {
          const double x = rp[i], y = rq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga != 0.0 && fabs(ga) > 1e-15 * sqrt(al * be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int i = lane; i < lp; i += 32) {
            const double x = rp[i], y = rq[i];
            rp[i] = cs * x - sn * y;
            rq[i] = sn * x + cs * y;
          }
          double* vp = V + (int64_t)p * lp;
          double* vq = V + (int64_t)q * lp;
          for (int i = lane; i < lp; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          if (lane == 0) atomicOr(rotated, 1u);
        }
      }
      jac_grid_barrier(sync, sync + 1, nb);
    }
    unsigned any;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(any) : "l"(rotated) : "memory");
    if (!any) return;                                     // a sweep without rotations: converged
  }
}

__global__ void k_eye(double* V, int lp) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)lp * lp; e += (int64_t)gridDim.x * blockDim.x)
    V[e] = (e % lp) == (e / lp) ? 1.0 : 0.0;
}

__global__ void k_col_norms(const double* R, int lp, double* s) {
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= lp) return;
  double a = 0.0;
  for (int i = lane; i < lp; i += 32) a = fma(R[i + (int64_t)j * lp], R[i + (int64_t)j * lp], a);
#pragma unroll
  for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) s[j] = sqrt(a);
}

}  // namespace

// The right singular vectors of R (l x l, column-major, ld l), columns in decreasing singular value
// order, into Vout (l x l, ld l).
static sk_status jacobi_right_vectors(sk_ctx* c, const double* R, int64_t l, double* Vout) {
  const int lp = (int)(l + (l & 1));
  DBuf Rw, V, sync, sig, idx;
  SK_TRY(Rw.alloc(c, (size_t)lp * lp * sizeof(double)));
  SK_TRY(V.alloc(c, (size_t)lp * lp * sizeof(double)));
  const int max_sweeps = 40;
  SK_TRY(sync.alloc(c, (size_t)(2 + max_sweeps) * sizeof(unsigned)));
  SK_TRY(sig.alloc(c, (size_t)lp * sizeof(double)));
  SK_TRY(idx.alloc(c, (size_t)lp * sizeof(int64_t)));
  SK_CUDA(c, cudaMemsetAsync(Rw.p, 0, (size_t)lp * lp * sizeof(double), c->stream));
  SK_CUDA(c, cudaMemcpy2DAsync(Rw.p, (size_t)lp * sizeof(double), R, (size_t)l * sizeof(double),
                               (size_t)l * sizeof(double), (size_t)l, cudaMemcpyDeviceToDevice, c->stream));
  SK_CUDA(c, cudaMemsetAsync(sync.p, 0, (size_t)(2 + max_sweeps) * sizeof(unsigned), c->stream));
  k_eye<<<(unsigned)std::min<int64_t>(cdiv((int64_t)lp * lp, 256), 4LL * c->num_sms), 256, 0, c->stream>>>(V.as<double>(), lp);
  SK_TRY(launched(c));
  int per_sm = 0;
  SK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_svd, 256, 0));
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)c->num_sms, (int64_t)per_sm * c->num_sms,
                                                               cdiv(lp / 2, 8)}));
  double* Rp = Rw.as<double>();
  double* Vp = V.as<double>();
  unsigned* sp = sync.as<unsigned>();
  int lpv = lp, msw = max_sweeps;
  void* args[] = {(void*)&Rp, (void*)&Vp, (void*)&lpv, (void*)&msw, (void*)&sp};
  SK_CUDA(c, cudaLaunchCooperativeKernel((void*)k_jacobi_svd, dim3(nb), dim3(256), args, 0, c->stream));
  SK_TRY(launched(c));
  k_col_norms<<<(unsigned)cdiv(lp, 8), 256, 0, c->stream>>>(Rw.as<double>(), lp, sig.as<double>());
  SK_TRY(launched(c));
  std::vector<double> s(lp);
  SK_CUDA(c, cudaMemcpyAsync(s.data(), sig.p, (size_t)lp * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  std::vector<int64_t> order(lp);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return s[a] > s[b]; });
  SK_CUDA(c, cudaMemcpyAsync(idx.p, order.data(), (size_t)lp * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  // Vout(:, j) = V(0:l, order[j]) for j < l (the padded column, if any, has sigma 0 and sorts last)
  SK_TRY(gather_cols_shard(c, V.as<double>(), l, lp, 0, lp, idx.as<int64_t>(), l, Vout, l));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));                  // `order` goes out of scope
  return SK_OK;
}

sk_status select_cols_deim(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* X, int64_t l,
                           int64_t ldx, int64_t k, int64_t* Js, int64_t* status_dev) {
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  // Q_X = ortho(X^T): X row-major l x n (ldx) == X^T column-major n x l (ld ldx)
  DBuf Xt, Q, B, Lf, U, piv, G, RL, R, Vt, Vk;
  SK_TRY(Xt.alloc(c, (size_t)n * l * sizeof(double)));
  SK_TRY(Q.alloc(c, (size_t)n * l * sizeof(double)));
  SK_CUDA(c, cudaMemcpy2DAsync(Xt.p, n * sizeof(double), X, ldx * sizeof(double), n * sizeof(double), l,
                               cudaMemcpyDeviceToDevice, c->stream));
  SK_TRY(orthonormal_basis(c, Xt.as<double>(), n, l, Q.as<double>(), status_dev));
  Xt.release();
  // B = A Q_X (m x l); B = Lf U (row LUPP), Lf -> Q_L (CholeskyQR2 in place), R_L = Q_L^T Lf, R = R_L U
  SK_TRY(B.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(gemm(c, false, false, m, l, n, 1.0, A, lda, Q.as<double>(), n, 0.0, B.as<double>(), m));
  SK_TRY(Lf.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(U.alloc(c, (size_t)l * l * sizeof(double)));
  SK_TRY(piv.alloc(c, (size_t)l * sizeof(int64_t)));
  SK_CUDA(c, cudaMemsetAsync(U.p, 0, (size_t)l * l * sizeof(double), c->stream));
  SK_TRY(lupp(c, B.as<double>(), false, m, l, m, piv.as<int64_t>(), Lf.as<double>(), m, U.as<double>(), l, nullptr,
              status_dev));
  SK_TRY(G.alloc(c, (size_t)m * l * sizeof(double)));
  SK_CUDA(c, cudaMemcpyAsync(G.p, Lf.p, (size_t)m * l * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  SK_TRY(cholqr2(c, G.as<double>(), m, l, m, status_dev));                                      // Q_L
  SK_TRY(RL.alloc(c, (size_t)l * l * sizeof(double)));
  SK_TRY(R.alloc(c, (size_t)l * l * sizeof(double)));
  SK_TRY(gemm(c, true, false, l, l, m, 1.0, G.as<double>(), m, Lf.as<double>(), m, 0.0, RL.as<double>(), l));
  SK_TRY(gemm(c, false, false, l, l, l, 1.0, RL.as<double>(), l, U.as<double>(), l, 0.0, R.as<double>(), l));
  B.release();
  Lf.release();
  G.release();
  // V~ (l x l, columns by decreasing sigma) = the right singular vectors of R
  SK_TRY(Vt.alloc(c, (size_t)l * l * sizeof(double)));
  SK_TRY(jacobi_right_vectors(c, R.as<double>(), l, Vt.as<double>()));
  // V^_k = Q_X V~(:, 0:k)  (n x k, column-major)
  SK_TRY(Vk.alloc(c, (size_t)n * k * sizeof(double)));
  SK_TRY(gemm(c, false, false, n, k, l, 1.0, Q.as<double>(), n, Vt.as<double>(), l, 0.0, Vk.as<double>(), n));
  // DEIM = LUPP on V^_k^T: pivot over the rows of the n x k panel V^_k, column t at step t
  return lupp(c, Vk.as<double>(), false, n, k, n, Js, nullptr, 0, nullptr, 0, nullptr, status_dev);
}

}  // namespace skel
