// lupp.cu -- S2 / S4: k-step LU with partial pivoting on a tall n x k panel.
//
// Paper: eq:def_LUPP and the pivot rule: step t scans ONE line of the
// active submatrix, picks j_t = argmax |X^{(t)}(t, j)| and applies the Schur-complement
// update.  Column LUPP on the sketch X gives J_s (Alg. 2 line 3); row LUPP
// on C = A(:, J_s) gives I_s (line 4).  Both are the same computation on an n x k
// panel M whose ROWS are pivoted (M = X(0:k, :)^T, resp. M = C).  Readings: R5 (only
// rows 0..k-1 of X enter), R6 (ties -> lowest original index, no physical swaps),
// R7 (rank failure when |pivot| <= 1e-14 max|M|).
//
// B200 design: the k-long chain of global argmaxes is the
// critical path, so the pivot search runs inside ONE thread-block cluster (16 CTAs,
// distributed shared memory) where an exchange costs a cluster barrier (~0.2 us)
// instead of a grid-wide barrier (~3.7 us measured).  The panel is factored in column
// blocks of width bp held in the cluster's shared memory; between blocks the whole GPU
// applies the trailing update with the DMMA GEMM:
//     per block [c0, c1):  k_panel  (cluster)  : bp pivot steps, L block, U(c0:c1, c0:c1)
//                          k_u12    (grid)     : U(c0:c1, c1:k) = L11^{-1} M(piv, c1:k)
//                          gemm     (grid)     : M(:, c1:k) -= Lf(:, c0:c1) U(c0:c1, c1:k)
// The blocked and unblocked eliminations are the same algorithm; only rounding differs.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace skel {
namespace {

constexpr int PNT = 512;   // threads per panel CTA

struct Slot {
  double a1, a2;
  long long idx;
  long long pad;
};

struct PanelParams {
  double* W;  int64_t n;  int k;        // working panel, n x k col-major (ld n), trailing-updated
  int c0, bp;                            // this column block
  int R;                                 // rows per CTA
  int pstride;                           // smem row stride (odd)
  int* rowstate;                         // global: -1 active, else step at which picked
  int64_t* Js; double* Lf; int64_t ldlf; double* Uw;   // Uw: k x k col-major (ld k)
  double* gaps;
  const unsigned long long* maxbits;     // max |M| (bit pattern)
  int64_t* status;                       // 0 or 1-based failing step
};

__global__ void k_lupp_init(const double* P, bool row_major, int64_t n, int k, int64_t ld, double* W,
                            int* rowstate, unsigned long long* maxbits) {
  double mx = 0.0;
  const int64_t total = n * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, t = e / n;
    const double v = row_major ? P[t * ld + i] : P[i + t * ld];
    W[e] = v;
    mx = fmax(mx, fabs(v));
    if (t == 0) rowstate[i] = -1;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(mx));
}

__global__ void __launch_bounds__(PNT, 1) k_lupp_panel(PanelParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  extern __shared__ __align__(16) double sm[];
  double* P = sm;                                               // [R][pstride]
  double* urow = P + (size_t)p.R * p.pstride;                   // [bp]
  Slot* slots = reinterpret_cast<Slot*>(urow + ((p.bp + 1) & ~1));   // [2][csize]
  dev::Cand* red = reinterpret_cast<dev::Cand*>(slots + 2 * csize);  // [33]
  int* state = reinterpret_cast<int*>(red + 33);                 // [R]
  __shared__ int s_stop;

  const int64_t r0 = (int64_t)crank * p.R;
  const int Rc = (int)std::max<int64_t>(0, std::min<int64_t>(p.R, p.n - r0));
  if (threadIdx.x == 0) s_stop = (*p.status != 0);
  // load this CTA's rows of the column block (coalesced along rows)
  for (int e = threadIdx.x; e < Rc * p.bp; e += PNT) {
    const int li = e % Rc, s = e / Rc;
    P[li * p.pstride + s] = p.W[(r0 + li) + (int64_t)(p.c0 + s) * p.n];
  }
  for (int li = threadIdx.x; li < Rc; li += PNT) state[li] = p.rowstate[r0 + li];
  const double tol = 1e-14 * __longlong_as_double((long long)*p.maxbits);
  cluster.sync();
  const bool stopped = s_stop;

  // thread -> (row, column-lane) map for the Schur update
  int tpr = 1;
  while (tpr < 32 && Rc > 0 && tpr * 2 * Rc <= PNT) tpr *= 2;
  const int rows_per_pass = PNT / tpr;
  const int my_cj = threadIdx.x % tpr;

  int s_end = stopped ? 0 : p.bp;
  for (int s = 0; s < s_end; ++s) {
    const int t = p.c0 + s;
    // (a) local candidate over active rows
    dev::Cand c = dev::cand_none();
    for (int li = threadIdx.x; li < Rc; li += PNT)
      if (state[li] < 0) {
        dev::Cand d{fabs(P[li * p.pstride + s]), -1.0, (long long)(r0 + li)};
        c = dev::cand_merge(c, d);
      }
    c = dev::block_cand_reduce(c, red);
    // (b) publish to every CTA of the cluster (distributed shared memory)
    Slot* mine = slots + (s & 1) * csize + crank;
    if (threadIdx.x < csize) {
      Slot* dst = cluster.map_shared_rank(mine, (int)threadIdx.x);
      *dst = Slot{c.a1, c.a2, c.i1, 0};
    }
    cluster.sync();
    // (c) identical reduction in every CTA
    dev::Cand w = dev::cand_none();
    for (int r = 0; r < csize; ++r) {
      const Slot& sl = slots[(s & 1) * csize + r];
      w = dev::cand_merge(w, dev::Cand{sl.a1, sl.a2, sl.idx});
    }
    if (!(w.a1 > tol)) {   // rank failure (R7): same decision in every CTA
      if (crank == 0 && threadIdx.x == 0) {
        *p.status = t + 1;
        for (int tt = t; tt < p.k; ++tt) p.Js[tt] = -1;
      }
      break;
    }
    const int wr = (int)(w.i1 / p.R);
    const int wl = (int)(w.i1 - (int64_t)wr * p.R);
    // (d) fetch the pivot row's remaining block entries from its owner
    {
      const double* rp = cluster.map_shared_rank(P + (size_t)wl * p.pstride, wr);
      for (int j = s + threadIdx.x; j < p.bp; j += PNT) urow[j] = rp[j];
    }
    __syncthreads();
    if (crank == 0) {
      if (threadIdx.x == 0) {
        p.Js[t] = w.i1;
        if (p.gaps) p.gaps[t] = (w.a1 - fmax(w.a2, 0.0)) / w.a1;
      }
      for (int j = s + threadIdx.x; j < p.bp; j += PNT) p.Uw[t + (int64_t)(p.c0 + j) * p.k] = urow[j];
    }
    if (wr == crank && threadIdx.x == 0) state[wl] = t;
    __syncthreads();
    // (e) Schur-complement update of the active rows (columns s..bp-1 of the block)
    const double piv = urow[s];
    for (int base = 0; base < Rc; base += rows_per_pass) {
      const int li = base + threadIdx.x / tpr;
      double L = 0.0;
      const bool act = li < Rc && state[li] < 0;
      if (act) L = P[li * p.pstride + s] / piv;
      __syncwarp();
      if (act) {
        double* row = P + (size_t)li * p.pstride;
        for (int j = s + 1 + my_cj; j < p.bp; j += tpr) row[j] = fma(-L, urow[j], row[j]);
      }
      __syncthreads();
      if (act && my_cj == 0) P[li * p.pstride + s] = L;
    }
    __syncthreads();
  }
  // write the L block and the row states back
  for (int e = threadIdx.x; e < Rc * p.bp; e += PNT) {
    const int li = e % Rc, s = e / Rc;
    const int st = state[li], t = p.c0 + s;
    double v;
    if (st < 0 || st > t) v = P[li * p.pstride + s];
    else v = (st == t) ? 1.0 : 0.0;
    p.Lf[(r0 + li) + (int64_t)t * p.ldlf] = v;
  }
  for (int li = threadIdx.x; li < Rc; li += PNT) p.rowstate[r0 + li] = state[li];
  cluster.sync();   // no CTA leaves while a peer may still read its shared memory
}

// U(c0+s, j) = M(piv_s, j) - sum_{s'<s} L11(s, s') U(c0+s', j), j in [c1, k).  One warp per column.
__global__ void k_lupp_u12(const double* W, int64_t n, int k, int c0, int bp, const int64_t* Js,
                           const double* Lf, int64_t ldlf, double* Uw, const int64_t* status) {
  if (*status != 0) return;
  extern __shared__ double L11[];   // bp x bp, row s holds L11(s, 0..s-1)
  for (int e = threadIdx.x; e < bp * bp; e += blockDim.x) {
    const int s = e / bp, sp = e % bp;
    L11[e] = sp < s ? Lf[Js[c0 + s] + (int64_t)(c0 + sp) * ldlf] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int c1 = c0 + bp;
  for (int j = c1 + blockIdx.x * warps + (threadIdx.x >> 5); j < k; j += gridDim.x * warps) {
    double u0 = 0.0, u1 = 0.0;   // u[lane], u[lane + 32]
    for (int s = 0; s < bp; ++s) {
      double part = 0.0;
      if (lane < s) part = L11[s * bp + lane] * u0;
      if (lane + 32 < s) part = fma(L11[s * bp + lane + 32], u1, part);
      part = dev::warp_sum(part);
      const double v = W[Js[c0 + s] + (int64_t)j * n] - part;
      if (s == lane) u0 = v;
      if (s == lane + 32) u1 = v;
    }
    if (lane < bp) Uw[(c0 + lane) + (int64_t)j * k] = u0;
    if (lane + 32 < bp) Uw[(c0 + lane + 32) + (int64_t)j * k] = u1;
  }
}

__global__ void k_copy_u(const double* Uw, int k, double* U, int64_t ldu) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % k), j = (int)(e / k);
    U[i + j * ldu] = i <= j ? Uw[e] : 0.0;
  }
}

struct ClusterCfg {
  int cs = 0;
  bool ok = false;
  int max_dyn = 0;
  std::string why;
};

ClusterCfg pick_cluster(sk_ctx* c) {
  static ClusterCfg cfg;
  static bool done = false;
  if (done) return cfg;
  done = true;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k_lupp_panel);
  cfg.max_dyn = c->max_smem_optin - (int)fa.sharedSizeBytes;
  cudaFuncSetAttribute(k_lupp_panel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const cudaError_t ea = cudaFuncSetAttribute(k_lupp_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.max_dyn);
  if (ea != cudaSuccess) cfg.why += std::string("smem attribute: ") + cudaGetErrorString(ea) + "; ";
  for (int cs : {16, 8, 4, 2, 1}) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(PNT);
    lc.dynamicSmemBytes = (size_t)cfg.max_dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    int nclusters = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k_lupp_panel, &lc);
    if (e == cudaSuccess && nclusters > 0) {
      cfg.cs = cs; cfg.ok = true;
      break;
    }
    cfg.why += "cs=" + std::to_string(cs) + ": " + cudaGetErrorString(e) + " (" + std::to_string(nclusters) + "); ";
    cudaGetLastError();
  }
  return cfg;
}

}  // namespace

sk_status lupp(sk_ctx* c, const double* Pin, bool row_major, int64_t n, int64_t k, int64_t ld,
               int64_t* Js, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* gaps,
               int64_t* status_dev) {
  const ClusterCfg cfg = pick_cluster(c);
  if (!cfg.ok) return fail(c, SK_E_CUDA, "no thread-block cluster configuration for the LUPP panel: " + cfg.why);
  const int cs = cfg.cs;
  const int64_t R = cdiv(n, cs);
  const size_t fixed = 2 * cs * sizeof(Slot) + 33 * sizeof(dev::Cand) + (size_t)R * sizeof(int) +
                       (64 + 2) * sizeof(double) + 1024;
  const int64_t budget = (int64_t)cfg.max_dyn - (int64_t)fixed;
  int64_t bp = budget / (R * 8) - 1;
  bp = std::min<int64_t>(bp, 64);
  bp = std::min<int64_t>(bp, k);
  if (bp < 1) return fail(c, SK_E_ARG, "LUPP panel too tall for one cluster (n too large)");
  // odd smem stride (bank-conflict-free row-per-thread access)
  auto stride_of = [](int64_t b) { return (b % 2 == 0) ? b + 1 : b; };
  while (bp > 1 && R * stride_of(bp) * 8 > budget) --bp;

  DBuf Wb, Ub, stateb, maxb, Lfb;
  SK_TRY(Wb.alloc(c, (size_t)n * k * sizeof(double)));
  SK_TRY(Ub.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(stateb.alloc(c, (size_t)n * sizeof(int)));
  SK_TRY(maxb.alloc(c, sizeof(unsigned long long)));
  if (!Lf) {
    SK_TRY(Lfb.alloc(c, (size_t)n * k * sizeof(double)));
    Lf = Lfb.as<double>();
    ldlf = n;
  }
  SK_CUDA(c, cudaMemsetAsync(maxb.p, 0, sizeof(unsigned long long), c->stream));
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  {
    const int blocks = (int)std::min<int64_t>(cdiv(n * k, 256), 8LL * c->num_sms);
    k_lupp_init<<<blocks, 256, 0, c->stream>>>(Pin, row_major, n, (int)k, ld, Wb.as<double>(),
                                               stateb.as<int>(), maxb.as<unsigned long long>());
    SK_TRY(launched(c));
  }
  for (int64_t c0 = 0; c0 < k; c0 += bp) {
    const int b = (int)std::min<int64_t>(bp, k - c0);
    PanelParams pp{};
    pp.W = Wb.as<double>(); pp.n = n; pp.k = (int)k;
    pp.c0 = (int)c0; pp.bp = b; pp.R = (int)R; pp.pstride = (int)stride_of(b);
    pp.rowstate = stateb.as<int>();
    pp.Js = Js; pp.Lf = Lf; pp.ldlf = ldlf; pp.Uw = Ub.as<double>(); pp.gaps = gaps;
    pp.maxbits = maxb.as<unsigned long long>(); pp.status = status_dev;
    const size_t smem = (size_t)R * pp.pstride * 8 + (size_t)((b + 1) & ~1) * 8 + 2 * cs * sizeof(Slot) +
                        33 * sizeof(dev::Cand) + (size_t)R * sizeof(int);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(PNT);
    lc.dynamicSmemBytes = smem;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    SK_CUDA(c, cudaLaunchKernelEx(&lc, k_lupp_panel, pp));
    SK_TRY(launched(c));
    const int64_t c1 = c0 + b;
    if (c1 < k) {
      const int warps = 8;
      const int blocks = (int)std::min<int64_t>(cdiv(k - c1, warps), 4LL * c->num_sms);
      const size_t s2 = (size_t)b * b * sizeof(double);
      k_lupp_u12<<<blocks, warps * 32, s2, c->stream>>>(Wb.as<double>(), n, (int)k, (int)c0, b, Js, Lf,
                                                       ldlf, Ub.as<double>(), status_dev);
      SK_TRY(launched(c));
      SK_TRY(gemm(c, false, false, n, k - c1, b, -1.0, Lf + c0 * ldlf, ldlf, Ub.as<double>() + c0 + c1 * k,
                  k, 1.0, Wb.as<double>() + c1 * n, n));
    }
  }
  if (U) {
    const int blocks = (int)std::min<int64_t>(cdiv(k * k, 256), 4LL * c->num_sms);
    k_copy_u<<<blocks, 256, 0, c->stream>>>(Ub.as<double>(), (int)k, U, ldu);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

}  // namespace skel
