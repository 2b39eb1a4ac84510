// cpqr.cu -- S2': column-pivoted Householder QR on the sketch (the paper's Rand-CPQR comparison).
//
// Paper: eq:def_QRCP and the pivot rule: step t searches the
// ENTIRE active submatrix X^{(t)}(t:l, :) for the column of largest l2 norm, then applies
// a Householder (rank-1 orthogonal) update.  Readings: R6 (ties -> lowest
// index), R9 (norms recomputed exactly every step, no downdating).
//
// B200 design: unlike LUPP the pivot rule needs every column's full remaining norm, so
// the l x n sketch (17 MB at C2) is spread over ALL SMs: one persistent cooperative
// kernel, each CTA holding a block of columns in shared memory (global workspace when it
// does not fit), one grid-wide exchange per step.  The exchange publishes each CTA's
// best (norm^2, index) and that column's remaining entries into double-buffered global
// slots, then releases a per-CTA flag (st.release.gpu); readers poll with ld.acquire.gpu.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace skel {
namespace {

constexpr int QNT = 512;

struct QParams {
  const double* X; int64_t ldx; int l; int64_t n; int k;
  int NC;                         // columns per CTA
  double* gX;                     // global fallback storage (l x n col-major) or nullptr
  int64_t* Js; double* R; int64_t ldr;
  double* cand;                   // [2][G][4]: norm2, idx(as double bits), fro2, pad
  double* colbuf;                 // [2][G][l]
  unsigned long long* flags;      // [G * 16]
  int64_t* status;
  unsigned long long epoch0;      // flags from earlier launches are < epoch0 + 1
};

__device__ __forceinline__ void flag_release(unsigned long long* f, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long flag_acquire(const unsigned long long* f) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
  return v;
}

__global__ void __launch_bounds__(QNT, 1) k_cpqr(QParams p) {
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, gid = blockIdx.x;
  const int64_t j0 = (int64_t)gid * p.NC;
  const int nc = (int)std::max<int64_t>(0, std::min<int64_t>(p.NC, p.n - j0));
  const int l = p.l;
  double* Xc = p.gX ? p.gX + j0 * l : sm;            // [nc][l] column-major
  double* v = p.gX ? sm : sm + (size_t)p.NC * l;     // [l]
  double* nrm = v + l;                               // [NC]
  int* active = reinterpret_cast<int*>(nrm + p.NC);  // [NC]
  __shared__ dev::Cand red[33];
  __shared__ double sred[34];
  __shared__ double s_beta, s_alpha;
  __shared__ long long s_piv;
  __shared__ double sca[QNT], scf[QNT];                 // per-CTA candidates of this step (G <= QNT)
  __shared__ long long sci[QNT];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = QNT / 32;

  // load own columns (X row-major: consecutive threads -> consecutive columns)
  double fro2 = 0.0;
  for (int64_t e = threadIdx.x; e < (int64_t)nc * l; e += QNT) {
    const int jl = (int)(e % nc), i = (int)(e / nc);
    const double x = p.X[(int64_t)i * p.ldx + j0 + jl];
    Xc[(int64_t)jl * l + i] = x;
    fro2 = fma(x, x, fro2);
  }
  for (int jl = threadIdx.x; jl < nc; jl += QNT) active[jl] = 1;
  fro2 = dev::block_sum(fro2, sred);
  double tol2 = 0.0;

  for (int t = 0; t < p.k; ++t) {
    const int par = t & 1;
    // (1) exact remaining norms of own active columns, rows t..l-1 (warp per column)
    for (int jl = warp; jl < nc; jl += nw) {
      double s = 0.0;
      if (active[jl]) {
        const double* col = Xc + (int64_t)jl * l;
        for (int i = t + lane; i < l; i += 32) s = fma(col[i], col[i], s);
        s = dev::warp_sum(s);
      }
      if (lane == 0) nrm[jl] = active[jl] ? s : -1.0;
    }
    __syncthreads();
    // (2) local argmax (ties -> lowest index)
    dev::Cand c = dev::cand_none();
    for (int jl = threadIdx.x; jl < nc; jl += QNT)
      if (active[jl]) c = dev::cand_merge(c, dev::Cand{nrm[jl], -1.0, (long long)(j0 + jl)});
    c = dev::block_cand_reduce(c, red);
    // (3) publish candidate + its remaining column, then release the flag
    double* mycand = p.cand + ((size_t)par * G + gid) * 4;
    double* mycol = p.colbuf + ((size_t)par * G + gid) * l;
    if (c.a1 >= 0.0) {
      const double* col = Xc + (c.i1 - j0) * l;
      for (int i = t + threadIdx.x; i < l; i += QNT) mycol[i] = col[i];
    }
    if (threadIdx.x == 0) {
      mycand[0] = c.a1;
      mycand[1] = __longlong_as_double(c.i1);
      mycand[2] = fro2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      flag_release(p.flags + (size_t)gid * 16, p.epoch0 + t + 1);
    }
    // (4) wait for every CTA; the thread that saw CTA r's flag also fetches its candidate (one L2
    //     round trip fewer on the critical path), then warp 0 reduces them in a fixed order
    for (int r = threadIdx.x; r < G; r += QNT) {
      while (flag_acquire(p.flags + (size_t)r * 16) < p.epoch0 + t + 1) {
      }
      const double* cr = p.cand + ((size_t)par * G + r) * 4;
      const double2 c01 = __ldcg(reinterpret_cast<const double2*>(cr));
      sca[r] = c01.x;
      sci[r] = __double_as_longlong(c01.y);
      if (t == 0) scf[r] = __ldcg(cr + 2);
    }
    __syncthreads();
    if (warp == 0) {
      dev::Cand w = dev::cand_none();
      double f2 = 0.0;
      for (int r = lane; r < G; r += 32) {
        const double a = sca[r];
        if (a >= 0.0) w = dev::cand_merge(w, dev::Cand{a, -1.0, sci[r]});
        if (t == 0) f2 += scf[r];
      }
      w = dev::warp_cand_reduce(w);
      if (t == 0) {
        // fixed-order sum of the per-CTA Frobenius partials (lane-strided then tree)
        f2 = dev::warp_sum(f2);
      }
      if (lane == 0) {
        s_piv = w.a1 >= 0.0 ? w.i1 : -1;
        if (t == 0) sred[33] = f2;
        s_alpha = w.a1;   // norm^2 of the winner for now
      }
    }
    __syncthreads();
    if (t == 0) tol2 = (1e-14 * 1e-14) * sred[33];
    const long long piv = s_piv;
    if (piv < 0 || !(s_alpha > tol2)) {
      if (gid == 0 && threadIdx.x == 0) {
        *p.status = t + 1;
        for (int tt = t; tt < p.k; ++tt) p.Js[tt] = -1;
      }
      return;   // same decision in every CTA
    }
    // (5) Householder vector from the winner's column (every CTA, redundantly)
    const int owner = (int)(piv / p.NC);
    const double* wcol = p.colbuf + ((size_t)par * G + owner) * l;
    for (int i = t + threadIdx.x; i < l; i += QNT) v[i] = *(volatile const double*)&wcol[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      // the winner's remaining squared norm is the value every CTA just reduced (computed once by
      // its owner in a fixed order), so no serial O(l) pass on the critical path
      const double s = s_alpha;
      const double nx = sqrt(s);
      const double alpha = v[t] >= 0.0 ? -nx : nx;
      const double vt = v[t] - alpha;
      const double vv = s - v[t] * v[t] + vt * vt;
      v[t] = vt;
      s_alpha = alpha;
      s_beta = vv > 0.0 ? 2.0 / vv : 0.0;
    }
    __syncthreads();
    const double beta = s_beta, alpha = s_alpha;
    // (6) apply H = I - beta v v^T to own active columns; write row t of R
    for (int jl = warp; jl < nc; jl += nw) {
      const int64_t j = j0 + jl;
      double* col = Xc + (int64_t)jl * l;
      if (j == piv) {
        if (lane == 0) {
          col[t] = alpha;
          if (p.R) p.R[t + j * p.ldr] = alpha;
        }
        continue;
      }
      if (!active[jl]) {
        if (lane == 0 && p.R) p.R[t + j * p.ldr] = 0.0;
        continue;
      }
      double d = 0.0;
      for (int i = t + lane; i < l; i += 32) d = fma(v[i], col[i], d);
      d = dev::warp_sum(d) * beta;
      for (int i = t + lane; i < l; i += 32) col[i] = fma(-d, v[i], col[i]);
      __syncwarp();
      if (lane == 0 && p.R) p.R[t + j * p.ldr] = col[t];
    }
    if (piv >= j0 && piv < j0 + nc && threadIdx.x == 0) active[piv - j0] = 0;
    if (gid == 0 && threadIdx.x == 0) p.Js[t] = piv;
    __syncthreads();
  }
}

}  // namespace

sk_status cpqr(sk_ctx* c, const double* X, int64_t l, int64_t n, int64_t ldx, int64_t k, int64_t* Js,
               double* R, int64_t ldr, int64_t* status_dev) {
  int G = (int)std::min<int64_t>(std::min<int64_t>(c->num_sms, QNT), n);
  const int NC = (int)cdiv(n, G);
  G = (int)cdiv(n, NC);
  const size_t small = (size_t)l * 8 + (size_t)NC * 12 + 256;
  const size_t full = (size_t)NC * l * 8 + small;
  const bool in_smem = full <= (size_t)c->max_smem_optin - 2048;
  const size_t smem = in_smem ? full : small;
  DBuf gX, cand, colbuf, flags;
  if (!in_smem) SK_TRY(gX.alloc(c, (size_t)l * NC * G * sizeof(double)));
  SK_TRY(cand.alloc(c, (size_t)2 * G * 4 * sizeof(double)));
  SK_TRY(colbuf.alloc(c, (size_t)2 * G * l * sizeof(double)));
  SK_TRY(flags.alloc(c, (size_t)G * 16 * sizeof(unsigned long long)));
  SK_CUDA(c, cudaMemsetAsync(flags.p, 0, (size_t)G * 16 * sizeof(unsigned long long), c->stream));
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  SK_CUDA(c, cudaFuncSetAttribute(k_cpqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cpqr, QNT, smem));
  if (per_sm * c->num_sms < G) return fail(c, SK_E_CUDA, "CPQR grid cannot be co-resident");
  QParams p{};
  p.X = X; p.ldx = ldx; p.l = (int)l; p.n = n; p.k = (int)k; p.NC = NC;
  p.gX = in_smem ? nullptr : gX.as<double>();
  p.Js = Js; p.R = R; p.ldr = ldr;
  p.cand = cand.as<double>(); p.colbuf = colbuf.as<double>();
  p.flags = flags.as<unsigned long long>(); p.status = status_dev; p.epoch0 = 0;
  void* args[] = {&p};
  SK_CUDA(c, cudaLaunchCooperativeKernel((void*)k_cpqr, dim3(G), dim3(QNT), args, smem, c->stream));
  return launched(c);
}

}  // namespace skel
