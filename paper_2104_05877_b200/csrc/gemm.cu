// gemm.cu -- FP64 tensor-core (DMMA.8x8x4) GEMM used by the trailing LUPP updates,
// the triangular solves, Cholesky-QR and the fused residual reduction.
//
// Tile 64 x 64 x 16, 128 threads (2 x 2 warps, 32 x 32 per warp = 4 x 4 DMMA
// fragments), 3-stage cp.async pipeline.  Shared-memory layouts are chosen per
// transpose case so that global loads are coalesced along the contiguous
// dimension and every fragment load is bank-conflict free (strides = 4 mod 16
// doubles: lanes (g, q) hit bank pair 4q + g or 4g + q).
#include "common.cuh"
#include "dmma.cuh"
#include "internal.h"

namespace skel {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 128, STAGES = 3;
constexpr int SA = BM + 4;   // As[k][m] stride (!TA)
constexpr int SAT = BK + 4;  // As[m][k] stride (TA)
constexpr int SB = BK + 4;   // Bs[n][k] stride (!TB)
constexpr int SBT = BN + 4;  // Bs[k][n] stride (TB)
constexpr int A_ELEMS = (BK * SA > BM * SAT) ? BK * SA : BM * SAT;
constexpr int B_ELEMS = (BN * SB > BK * SBT) ? BN * SB : BK * SBT;
constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_ELEMS * sizeof(double);

enum { EPI_STORE = 0, EPI_SUMSQ = 1, EPI_PARTIAL = 2 };

struct Params {
  int M, N, K;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  const double* Cin; double* C; int64_t ldc;
  double alpha, beta;
  int k_per_split;
  double* out;   // EPI_PARTIAL: [splits][M*N]; EPI_SUMSQ: [ctas][2]
  int lower;     // M == N and only the tiles on or below the diagonal (blockIdx.x enumerates them)
};

template <bool TA>
__device__ __forceinline__ int a_off(int m, int k) { return TA ? m * SAT + k : k * SA + m; }
template <bool TB>
__device__ __forceinline__ int b_off(int k, int n) { return TB ? k * SBT + n : n * SB + k; }

template <bool TA, bool TB>
__device__ __forceinline__ void load_tile(const Params& p, double* As, double* Bs, int m0, int n0,
                                          int k0, int kend) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int r = 0; r < (BM * BK) / NT; ++r) {
    const int e = tid + r * NT;
    int m, k;
    if (!TA) { m = e % BM; k = e / BM; } else { m = e / BK; k = e % BK; }
    const int gm = m0 + m, gk = k0 + k;
    const bool ok = gm < p.M && gk < kend;
    const double* src = ok ? (TA ? p.A + gk + (int64_t)gm * p.lda : p.A + gm + (int64_t)gk * p.lda) : p.A;
    dev::cp_async8(As + a_off<TA>(m, k), src, ok);
  }
#pragma unroll
  for (int r = 0; r < (BN * BK) / NT; ++r) {
    const int e = tid + r * NT;
    int n, k;
    if (!TB) { n = e / BK; k = e % BK; } else { n = e % BN; k = e / BN; }
    const int gn = n0 + n, gk = k0 + k;
    const bool ok = gn < p.N && gk < kend;
    const double* src = ok ? (TB ? p.B + gn + (int64_t)gk * p.ldb : p.B + gk + (int64_t)gn * p.ldb) : p.B;
    dev::cp_async8(Bs + b_off<TB>(k, n), src, ok);
  }
}

template <bool TA, bool TB, int MODE>
__global__ void __launch_bounds__(NT) k_gemm(Params p) {
  dev::griddep_wait();
  extern __shared__ __align__(16) double sm[];
  int mb = blockIdx.x, nbk = blockIdx.y;
  if (p.lower) {                                   // lower-triangle tile t -> (mb, nbk), mb >= nbk
    mb = (int)((sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
    while (mb * (mb + 1) / 2 > (int)blockIdx.x) --mb;
    while ((mb + 1) * (mb + 2) / 2 <= (int)blockIdx.x) ++mb;
    nbk = (int)blockIdx.x - mb * (mb + 1) / 2;
  }
  const int m0 = mb * BM, n0 = nbk * BN;
  const int kbeg = blockIdx.z * p.k_per_split;
  const int kend = min(p.K, kbeg + p.k_per_split);
  const int ktiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_tile<TA, TB>(p, sm + s * STAGE_ELEMS, sm + s * STAGE_ELEMS + A_ELEMS, m0, n0,
                                      kbeg + s * BK, kend);
    dev::cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    dev::cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nx = kt + STAGES - 1;
    if (nx < ktiles) {
      const int st = nx % STAGES;
      load_tile<TA, TB>(p, sm + st * STAGE_ELEMS, sm + st * STAGE_ELEMS + A_ELEMS, m0, n0,
                        kbeg + nx * BK, kend);
    }
    dev::cp_async_commit();
    const double* As = sm + (kt % STAGES) * STAGE_ELEMS;
    const double* Bs = As + A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[a_off<TA>(wm + i * 8 + g, kk * 4 + q)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[b_off<TB>(kk * 4 + q, wn + j * 8 + g)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dev::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  dev::cp_async_wait<0>();

  if (MODE == EPI_STORE) {
    // issue every C load before the first store (the compiler cannot reorder them: aliasing)
    double cv[4][4][2];
    const bool rd = p.beta != 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + wm + i * 8 + g, n = n0 + wn + j * 8 + 2 * q + h;
          cv[i][j][h] = (rd && m < p.M && n < p.N) ? p.C[m + (int64_t)n * p.ldc] : 0.0;
        }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + wm + i * 8 + g, n = n0 + wn + j * 8 + 2 * q + h;
          if (m < p.M && n < p.N)
            p.C[m + (int64_t)n * p.ldc] = rd ? fma(p.beta, cv[i][j][h], p.alpha * acc[i][j][h])
                                             : p.alpha * acc[i][j][h];
        }
  } else if (MODE == EPI_PARTIAL) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm + i * 8 + g;
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = n0 + wn + j * 8 + 2 * q + h;
          if (n >= p.N) continue;
          p.out[(int64_t)blockIdx.z * p.M * p.N + m + (int64_t)n * p.M] = acc[i][j][h];
        }
    }
  } else {  // EPI_SUMSQ: e = alpha*acc + beta*Cin; accumulate e^2 and Cin^2 (never written)
    double s1 = 0.0, s2 = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm + i * 8 + g;
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = n0 + wn + j * 8 + 2 * q + h;
          if (n >= p.N) continue;
          const double cv = p.Cin[m + (int64_t)n * p.ldc];
          const double e = fma(p.beta, cv, p.alpha * acc[i][j][h]);
          s1 = fma(e, e, s1);
          s2 = fma(cv, cv, s2);
        }
    }
    __shared__ double red[34];
    s1 = dev::block_sum(s1, red);
    s2 = dev::block_sum(s2, red);
    if (threadIdx.x == 0) {
      const int64_t cta = blockIdx.x + (int64_t)gridDim.x * blockIdx.y;
      p.out[2 * cta] = s1;
      p.out[2 * cta + 1] = s2;
    }
  }
}

// C(m, n) = alpha * sum_z part[z](m, n) + beta * C, z ascending.  Grid (row blocks, column n): no
// 64-bit divisions; the split loads of an element are issued together.
__global__ void k_splitk_reduce(const double* __restrict__ part, int splits, int M, int N, double alpha,
                                double beta, double* __restrict__ C, int64_t ldc, int lower) {
  const int64_t total = (int64_t)M * N;
  for (int64_t n = blockIdx.y; n < N; n += gridDim.y)
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
      if (lower && m / BM < n / BN) continue;      // tile above the diagonal: never computed
      const double* src = part + m + n * M;
      double s = 0.0;
#pragma unroll 8
      for (int z = 0; z < splits; ++z) s += __ldcs(src + (int64_t)z * total);
      double* cp = C + m + n * ldc;
      const double v = alpha * s;
      *cp = (beta == 0.0) ? v : fma(beta, *cp, v);
    }
}

__global__ void k_reduce_pairs(const double* part, int64_t count, double* out) {
  __shared__ double red[34];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    s1 += part[2 * i];
    s2 += part[2 * i + 1];
  }
  s1 = dev::block_sum(s1, red);
  s2 = dev::block_sum(s2, red);
  if (threadIdx.x == 0) { out[0] = s1; out[1] = s2; }
}

template <bool TA, bool TB, int MODE>
sk_status launch(sk_ctx* c, const Params& p, dim3 grid) {
  static bool attr_dev[kMaxDevices] = {};  // per template instance and device
  bool& attr_set = attr_dev[c->device % kMaxDevices];
  if (!attr_set) {
    SK_CUDA(c, cudaFuncSetAttribute(k_gemm<TA, TB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SMEM_BYTES));
    attr_set = true;
  }
  if (c->pdl) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = grid;
    lc.blockDim = dim3(NT);
    lc.dynamicSmemBytes = SMEM_BYTES;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at; lc.numAttrs = 1;
    SK_CUDA(c, cudaLaunchKernelEx(&lc, k_gemm<TA, TB, MODE>, p));
  } else {
    k_gemm<TA, TB, MODE><<<grid, NT, SMEM_BYTES, c->stream>>>(p);
  }
  return launched(c);
}

template <int MODE>
sk_status dispatch(sk_ctx* c, bool ta, bool tb, const Params& p, dim3 grid) {
  if (!ta && !tb) return launch<false, false, MODE>(c, p, grid);
  if (!ta && tb) return launch<false, true, MODE>(c, p, grid);
  if (ta && !tb) return launch<true, false, MODE>(c, p, grid);
  return launch<true, true, MODE>(c, p, grid);
}

}  // namespace

sk_status gemm(sk_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc) {
  if (M <= 0 || N <= 0) return SK_OK;
  if (K <= 0) {
    // C = beta*C
    Params p{};
    p.M = (int)M; p.N = (int)N; p.K = 0; p.A = A; p.B = B; p.C = C; p.Cin = C; p.ldc = ldc;
    p.alpha = 0.0; p.beta = beta; p.k_per_split = 1;
    p.lda = lda; p.ldb = ldb;
    dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN), 1);
    return dispatch<EPI_STORE>(c, false, false, p, grid);
  }
  Params p{};
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.Cin = C; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  const int64_t tiles = cdiv(M, BM) * cdiv(N, BN);
  // split K when the tile grid cannot fill the machine and K is long
  int splits = 1;
  const int64_t target = 2LL * c->num_sms * 3;  // ~3 CTAs per SM resident
  while (tiles * splits * 2 <= target && K / (splits * 2) >= 256) splits *= 2;
  p.k_per_split = (int)(cdiv(cdiv(K, splits), BK) * BK);
  splits = (int)cdiv(K, p.k_per_split);
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN), (unsigned)splits);
  if (splits == 1) return dispatch<EPI_STORE>(c, ta, tb, p, grid);
  DBuf part;
  SK_TRY(part.alloc(c, (size_t)splits * M * N * sizeof(double)));
  p.out = part.as<double>();
  SK_TRY(dispatch<EPI_PARTIAL>(c, ta, tb, p, grid));
  const dim3 rg((unsigned)std::min<int64_t>(cdiv(M, 256), 64), (unsigned)std::min<int64_t>(N, 65535));
  k_splitk_reduce<<<rg, 256, 0, c->stream>>>(part.as<double>(), splits, (int)M, (int)N, alpha, beta, C, ldc, 0);
  return launched(c);
}

sk_status gram_lower(sk_ctx* c, const double* Q, int64_t m, int64_t k, int64_t ldq, double* G, int64_t ldg) {
  // G = Q^T Q on the 64 x 64 tiles on or below the diagonal only (the consumers -- Cholesky, the
  // Newton-Schulz prep, the shift -- read the lower triangle): ~T(T+1)/2 of T^2 tiles
  if (k <= 0) return SK_OK;
  if (m <= 0) return gemm(c, true, false, k, k, m, 1.0, Q, ldq, Q, ldq, 0.0, G, ldg);
  Params p{};
  p.M = (int)k; p.N = (int)k; p.K = (int)m;
  p.A = Q; p.lda = ldq; p.B = Q; p.ldb = ldq; p.C = G; p.Cin = G; p.ldc = ldg;
  p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
  const int64_t T = cdiv(k, BM), tiles = T * (T + 1) / 2;
  int splits = 1;
  const int64_t target = 2LL * c->num_sms * 3;
  while (tiles * splits * 2 <= target && m / (splits * 2) >= 256) splits *= 2;
  p.k_per_split = (int)(cdiv(cdiv(m, splits), BK) * BK);
  splits = (int)cdiv(m, p.k_per_split);
  dim3 grid((unsigned)tiles, 1, (unsigned)splits);
  if (splits == 1) return dispatch<EPI_STORE>(c, true, false, p, grid);
  DBuf part;
  SK_TRY(part.alloc(c, (size_t)splits * k * k * sizeof(double)));
  p.out = part.as<double>();
  SK_TRY(dispatch<EPI_PARTIAL>(c, true, false, p, grid));
  const dim3 rg((unsigned)std::min<int64_t>(cdiv(k, 256), 64), (unsigned)std::min<int64_t>(k, 65535));
  k_splitk_reduce<<<rg, 256, 0, c->stream>>>(part.as<double>(), splits, (int)k, (int)k, 1.0, 0.0, G, ldg, 1);
  return launched(c);
}

sk_status gemm_sumsq(sk_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                     const double* C, int64_t ldc, double* sums) {
  Params p{};
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.Cin = C; p.C = nullptr; p.ldc = ldc;
  p.alpha = alpha; p.beta = beta;
  p.k_per_split = (int)std::max<int64_t>(K, 1);
  dim3 grid((unsigned)cdiv(M, BM), (unsigned)cdiv(N, BN), 1);
  const int64_t ctas = (int64_t)grid.x * grid.y;
  DBuf part;
  SK_TRY(part.alloc(c, (size_t)ctas * 2 * sizeof(double)));
  p.out = part.as<double>();
  SK_TRY(dispatch<EPI_SUMSQ>(c, ta, tb, p, grid));
  return reduce_pairs(c, part.as<double>(), ctas, sums);
}

sk_status reduce_pairs(sk_ctx* c, const double* partial, int64_t count, double* out) {
  k_reduce_pairs<<<1, 1024, 0, c->stream>>>(partial, count, out);
  return launched(c);
}

}  // namespace skel
