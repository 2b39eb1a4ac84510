// sketch.cu -- S0+S1 (dense Gaussian sketch) and S1' (sparse-sign sketch):  X = Gamma A.
//
// Paper: Algorithm 2 lines 1-2; embeddings P:176 (Gaussian)
// (sparse sign, zeta = min(l, 8)); costs Table 1.  Gamma is regenerated from the
// Philox counter (philox.cuh) on every call and never held in HBM as a whole.
//
// Dense: a DMMA GEMM with M = l (rows of Gamma), N = n, K = m, run over K-chunks of A's rows:
// per chunk k_omega_image generates that chunk's columns of Gamma (<= ~80 MB, an L2-resident
// slot reused chunk after chunk) in the layout the GEMM's bulk copies read, and k_sketch_pre
// (TMA + DMMA) accumulates Gamma(:, chunk) A(chunk, :) into X.  A fallback kernel for A that
// the tensor map cannot describe (odd lda, misaligned) generates each Gamma tile in shared memory.
//
// Sparse sign: X(r, j) = zeta^{-1/2} sum_{i : r in S_i} s_{i,r} A(i, j).  A CTA owns 32
// columns (lane = column) and all l rows; per chunk of 128 rows of A it stages the A tile
// in shared memory (coalesced along i), draws the chunk's zeta*128 nonzeros of Gamma,
// records them as per-output-row bit masks (hit / negative) and gathers
// X(r, j) +-= A(i, j) in registers in ascending i -- deterministic summation order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "dmma.cuh"
#include "internal.h"
#include "philox.cuh"
#include "sync.cuh"

namespace skel {
namespace {

// ============================================================ dense Gaussian sketch
constexpr int DBM = 32, DBN = 256, DBK = 16, DNT = 256, DST = 3;
constexpr int DSO = DBM + 4;   // Omega tile Os[k][r], stride 36 (= 4 mod 16)
constexpr int DSB = DBK + 4;   // A tile Bs[n][k], stride 20 (= 4 mod 16)
constexpr int D_O_ELEMS = DBK * DSO;
constexpr int D_B_ELEMS = DBN * DSB;
constexpr int D_STAGE = D_O_ELEMS + D_B_ELEMS;
constexpr size_t D_SMEM = (size_t)DST * D_STAGE * sizeof(double);

struct DenseParams {
  const double* A; int64_t lda;
  int64_t m, n; int l;
  uint2 key;
  double scale;          // 1/sqrt(l)
  double* X; int64_t ldx;
  double* part;          // split-K partials [splits][l][n] (row-major, ld n)
  int64_t k_per_split;
  int64_t k0;            // first row of A in this K-chunk (rows k0 .. m-1 of A; m = the chunk's end)
  int accum;             // 1: X += the chunk's product (chunks after the first), 0: X = it
  // MODE 4 (residual): E = Csub - product over each output tile, never stored; per-CTA
  // (sum E^2, sum Csub^2) into sums_part[2 * linear block]
  const double* Csub; int64_t ldcs;
  double* sums_part;
  // chained K-chunks (run_pre_chained): each CTA adds 1 here when its tile is in X (release); the
  // image kernel of the chunk that next overwrites this chunk's slot waits for the count
  unsigned* done;
  const unsigned* ready;  // chained chunks: generator CTAs done so far in this chunk's slot ...
  unsigned ready_need;    // ... must reach this before the GEMM reads the slot
  // chained chunks: CTAs [gen_lo, gen_lo + gen_n) of this GEMM also make the NEXT chunk's image (rows
  // [gen_i0, gen_i1) of A, gen_kt k tiles) in gen_img, once gen_gate reaches gen_need (the GEMM that
  // last read that slot is done), then count themselves in gen_ready
  double* gen_img;
  const double* gen_q; int64_t gen_ldq;       // packed from Q (Omega = Q^T) when non-null, else Philox
  int64_t gen_i0, gen_i1, gen_kt;
  unsigned gen_lo, gen_n;
  const unsigned* gen_gate; unsigned gen_need;
  unsigned* gen_ready;
  // chained chunks: tile_ord[tile] = chunks already added into X's tile; chunk chunk_idx adds after it
  // reaches chunk_idx, so every element of X sums its chunks in chunk order (deterministic)
  unsigned* tile_ord; unsigned chunk_idx;
};

template <bool VEC>
__device__ __forceinline__ void dense_load_a(const DenseParams& p, double* Bs, int64_t n0, int64_t k0,
                                             int64_t kend) {
  const int tid = threadIdx.x;
  if (VEC) {
    // 256 columns x 8 chunks of 16 B
#pragma unroll
    for (int r = 0; r < (DBN * DBK / 2) / DNT; ++r) {
      const int e = tid + r * DNT;
      const int col = e >> 3, ch = e & 7;
      const int64_t gn = n0 + col, gk = k0 + 2 * ch;
      int bytes = 0;
      if (gn < p.n) bytes = gk + 1 < kend ? 16 : (gk < kend ? 8 : 0);
      const double* src = bytes ? p.A + gk + gn * p.lda : p.A;
      dev::cp_async16(Bs + col * DSB + 2 * ch, src, bytes);
    }
  } else {
#pragma unroll 4
    for (int r = 0; r < (DBN * DBK) / DNT; ++r) {
      const int e = tid + r * DNT;
      const int col = e >> 4, kk = e & 15;
      const int64_t gn = n0 + col, gk = k0 + kk;
      const bool ok = gn < p.n && gk < kend;
      dev::cp_async8(Bs + col * DSB + kk, ok ? p.A + gk + gn * p.lda : p.A, ok);
    }
  }
}

// Gamma tile: rows r0..r0+31 (16 Box-Muller pairs) x columns k0..k0+15 of the virtual l x m Gamma.
__device__ __forceinline__ void dense_gen_omega(const DenseParams& p, double* Os, int r0, int64_t k0,
                                                int64_t kend) {
  const int tid = threadIdx.x;           // 256 threads = 16 pairs x 16 columns
  const int pr = tid & 15, kc = tid >> 4;
  const int64_t i = k0 + kc;
  const int row = r0 + 2 * pr;
  double z0 = 0.0, z1 = 0.0;
  if (i < kend && row < p.l) {
    dev::gauss_pair((uint64_t)i, (uint32_t)(row >> 1), p.key, z0, z1);
    if (row + 1 >= p.l) z1 = 0.0;
  }
  Os[kc * DSO + 2 * pr] = z0;
  Os[kc * DSO + 2 * pr + 1] = z1;
}

template <bool VEC, bool SPLIT>
__global__ void __launch_bounds__(DNT, 1) k_sketch_dense(DenseParams p) {
  extern __shared__ __align__(16) double sm[];
  const int r0 = blockIdx.x * DBM;
  const int64_t n0 = (int64_t)blockIdx.y * DBN;
  const int64_t kbeg = (int64_t)blockIdx.z * p.k_per_split;
  const int64_t kend = min(p.m, kbeg + p.k_per_split);
  const int ktiles = kend > kbeg ? (int)((kend - kbeg + DBK - 1) / DBK) : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int wn = warp * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < DST - 1; ++s) {
    if (s < ktiles) {
      double* st = sm + s * D_STAGE;
      dense_load_a<VEC>(p, st + D_O_ELEMS, n0, kbeg + s * DBK, kend);
      dense_gen_omega(p, st, r0, kbeg + s * DBK, kend);
    }
    dev::cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    dev::cp_async_wait<DST - 2>();
    __syncthreads();
    const int nx = kt + DST - 1;
    if (nx < ktiles) {
      double* st = sm + (nx % DST) * D_STAGE;
      dense_load_a<VEC>(p, st + D_O_ELEMS, n0, kbeg + (int64_t)nx * DBK, kend);
      dev::cp_async_commit();
      dense_gen_omega(p, st, r0, kbeg + (int64_t)nx * DBK, kend);   // overlaps the copy
    } else {
      dev::cp_async_commit();
    }
    const double* Os = sm + (kt % DST) * D_STAGE;
    const double* Bs = Os + D_O_ELEMS;
#pragma unroll
    for (int kk = 0; kk < DBK / 4; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Os[(kk * 4 + q) * DSO + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn + j * 8 + g) * DSB + kk * 4 + q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dev::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  dev::cp_async_wait<0>();

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + i * 8 + g;
    if (r >= p.l) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t cidx = n0 + wn + j * 8 + 2 * q;
      if (SPLIT) {
        double* dst = p.part + ((int64_t)blockIdx.z * p.l + r) * p.n;
        if (cidx < p.n) dst[cidx] = acc[i][j][0];
        if (cidx + 1 < p.n) dst[cidx + 1] = acc[i][j][1];
      } else {
        double* dst = p.X + (int64_t)r * p.ldx;
        if (cidx < p.n) dst[cidx] = acc[i][j][0] * p.scale;
        if (cidx + 1 < p.n) dst[cidx + 1] = acc[i][j][1] * p.scale;
      }
    }
  }
}

// X(r, col) = scale * sum_z part[z](r, col), z ascending (fixed order).  Grid (column blocks, row r):
// no 64-bit divisions, and the split loads of an element are independent of the running sum, so
// they are in flight together.
template <int U>
__global__ void k_sketch_splitk_reduce(const double* __restrict__ part, int splits, int l, int64_t n, double scale,
                                       double* __restrict__ X, int64_t ldx, int accum) {
  dev::griddep_wait();                                   // PDL: the partials are complete
  const int64_t total = (int64_t)l * n;
  for (int64_t r = blockIdx.y; r < l; r += gridDim.y)
    for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x * U + threadIdx.x; c0 < n; c0 += (int64_t)gridDim.x * blockDim.x * U) {
      double s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = 0.0;
#pragma unroll 4
      for (int z = 0; z < splits; ++z) {
        const double* src = part + (int64_t)z * total + r * n;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t col = c0 + (int64_t)u * blockDim.x;
          if (col < n) s[u] += __ldcs(src + col);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t col = c0 + (int64_t)u * blockDim.x;
        if (col < n) X[r * ldx + col] = accum ? X[r * ldx + col] + s[u] * scale : s[u] * scale;
      }
    }
}

// 4 columns per thread for wide X (whole 1024-column blocks, two CTAs per SM), else 1
inline sk_status splitk_reduce(sk_ctx* c, const double* part, int splits, int64_t l, int64_t n, double scale, double* X,
                               int64_t ldx, int accum = 0) {
  const unsigned gy = (unsigned)std::min<int64_t>(l, 65535);
  const bool wide = n >= 2048 && (int64_t)gy * cdiv(n, 1024) >= 2LL * c->num_sms;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)std::min<int64_t>(cdiv(n, wide ? 1024 : 256), 64), gy);
  lc.blockDim = dim3(256);
  lc.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;    // PDL behind the GEMM
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at; lc.numAttrs = 1;
  if (wide) SK_CUDA(c, cudaLaunchKernelEx(&lc, k_sketch_splitk_reduce<4>, part, splits, (int)l, n, scale, X, ldx, accum));
  else SK_CUDA(c, cudaLaunchKernelEx(&lc, k_sketch_splitk_reduce<1>, part, splits, (int)l, n, scale, X, ldx, accum));
  return launched(c);
}

// ============================================================ dense sketch helpers
constexpr int TBK = 16;                                       // k rows (of A) per pipeline stage

// B-fragment bank conflicts under the 128-byte swizzle are avoided by permuting the 8 logical MMA
// columns onto physical columns sig(g) = 2(g&3) + (g>>2) (half-warps then hit disjoint 16-byte
// chunks); the epilogue applies the same permutation.
__device__ __forceinline__ int sig8(int g) { return 2 * (g & 3) + (g >> 2); }

__device__ __forceinline__ void red_add_f64(double* addr, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(addr), "d"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive_local(unsigned addr) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}

// ------------------------------------------------------------ dense sketch, K-chunked Omega image
// Omega is generated once per call, one K-chunk at a time (k_omega_image, ~l*chunk/2 Box-Muller
// pairs per chunk), into a slot of at most kOmegaSlotBytes that stays in L2 and is reused by
// the next chunk -- the whole l x m Omega never exists in memory.  The slot is
// laid out exactly as the consumers read it: per (row tile rt, k tile kt) a [TBK][OS] block,
// OS = BM + 4 (= 4 mod 16: the 8x4 DMMA A-fragment loads are conflict-free).  k_sketch_pre is then
// a plain TMA-fed DMMA GEMM X = Omega A with no generation inside: per stage one 1-D bulk copy of
// the Omega block and TBN/64 2-D tensor loads of the A tile (16 x 64, 128-byte swizzle), one ring
// of full/empty mbarriers, NW consumer warps of 32 columns x BM rows, one elected thread issuing
// the copies up to a ring ahead.  Freed from the cluster-shared Box-Muller producers, the tile
// can be chosen for the wave (plan_pre): BM in {32, 48, 64} rows x 256 columns, split-K to fill
// the waves; C2 (l = 522) runs BM = 48 (1% padded rows instead of 10% at BM = 64) with 4 K-splits.
// Tile geometry: BM rows of X (WM warp rows of FI = BM / (8 WM) MMA row fragments) x TBNP columns
// (WN warp columns of FJ 8-column fragments), NW = WM * WN consumer warps, CPS CTAs per SM (the
// ring takes ~200 KB / CPS of shared memory).  The wide-n family is WM = 1, FJ = 4 (warp = BM x 32);
// the narrow-n family (C4's n = 784 = 7 x 112) is 2 x 2 warps of 40 x 56 at 2 CTAs per SM, which
// tiles l = 400 and n = 784 exactly and loads all four SM sub-partitions equally.
template <int BM_, int WM_, int WN_, int FJ_, int CPS_> struct PCfg {
  static constexpr int BM = BM_, WM = WM_, WN = WN_, FJ = FJ_, CPS = CPS_;
  static constexpr int NW = WM * WN;
  static constexpr int FI = BM / (8 * WM);
  static_assert(FI * 8 * WM == BM, "BM = 8 FI WM");
  static constexpr int OS = BM + 4;
  static constexpr int TBNP = WN * FJ * 8;
  static constexpr int PBOX = TBNP % 64 == 0 ? 64 : (TBNP % 32 == 0 ? 32 : 16);   // columns per tensor load (box 16 x PBOX)
  static constexpr int A_BYTES = TBNP * TBK * 8;
  static constexpr int O_BYTES = TBK * OS * 8;
  static constexpr int ST_BYTES = ((A_BYTES + O_BYTES) + 1023) & ~1023;
  static constexpr int TS = ((CPS == 1 ? (NW > 8 ? 220 : 200) : 216 / CPS - 4) * 1024) / ST_BYTES;   // ring depth
  static constexpr size_t SMEM = (size_t)TS * ST_BYTES + 2 * TS * 8 + 1024;
  static constexpr int NT = NW * 32;
  static_assert(TS >= 2, "ring depth");
};
// the wide-n family by (BM, warps)
template <int BM, int NW> using PCfgW = PCfg<BM, 1, NW, 4, 1>;

// One image block (row tile rt, k tile kt; tile = rt * KT + kt) of rows [i0, m) of A, generated by the
// calling CTA's threads (nthr of them): pair e of the block -> column kk = e / (OS/2), rows 2 pr, 2 pr + 1.
__device__ __forceinline__ void omega_tile(uint2 key, int l, int64_t i0, int64_t m, int BM, int OS, int64_t KT,
                                           int64_t tile, double* __restrict__ img, int tid, int nthr) {
  const int64_t rt = tile / KT, kt = tile - (tile / KT) * KT;
  const int hp = OS / 2, np = TBK * hp;
  double2* blk = reinterpret_cast<double2*>(img + tile * (int64_t)(TBK * OS));
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (int e = tid; e < np; e += nthr) {
    const int kk = e / hp, pr = e - kk * hp;
    const int64_t i = i0 + kt * TBK + kk;           // row of A (column of Omega); m = the chunk's end
    const int row = (int)(rt * BM) + 2 * pr;
    double z0 = 0.0, z1 = 0.0;
    if (2 * pr < BM && i < m && row < l) {
      dev::gauss_pair((uint64_t)i, (uint32_t)(row >> 1), key, z0, z1);
      if (row + 1 >= l) z1 = 0.0;
    }
    // the slot is re-read by every column tile of A: keep it in L2 (evict_last)
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(blk + e), "d"(z0), "d"(z1), "l"(pol)
                 : "memory");
  }
}

// Chained K-chunks: the image kernel of chunk c overwrites the slot chunk c - 2's GEMM read, so it
// first waits (thread 0, bounded) until that GEMM's CTAs have all counted themselves done, then lets
// the chunk's GEMM be scheduled (the GEMM's griddepcontrol.wait still waits for this image).
__device__ __forceinline__ void wait_count(const unsigned* gate, unsigned need) {
  if (gate) {
    if (threadIdx.x == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gate) : "memory");
        if (v >= need) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20ull * 1000 * 1000 * 1000) __trap();   // 20 s: a scheduling bug, not a hang
        __nanosleep(256);
      }
    }
    __syncthreads();
  }
}
__device__ __forceinline__ void count_done(unsigned* ctr) {
  if (ctr) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
  }
}

// One CTA per image block: blockIdx.x = rt * KT + kt.
__global__ void __launch_bounds__(128) k_omega_image(uint2 key, int l, int64_t i0, int64_t m, int BM, int OS, int64_t KT,
                                                     double* __restrict__ img) {
  omega_tile(key, l, i0, m, BM, OS, KT, blockIdx.x, img, threadIdx.x, 128);
}

// The same image from a GIVEN Omega: Omega(r, i) = Q(i, r), Q m x l column-major (ld ldq), e.g. an
// orthonormal basis for W = Q^T A in the residual.  One CTA per image block; thread -> (kk, r) with
// kk fastest, so a warp reads 128-byte column segments of Q.
__device__ __forceinline__ void pack_tile(const double* __restrict__ Q, int64_t ldq, int l, int64_t i0, int64_t m, int BM,
                                          int OS, int64_t KT, int64_t tile, double* __restrict__ img, int tid, int nthr) {
  const int64_t rt = tile / KT, kt = tile - (tile / KT) * KT;
  double* blk = img + tile * (int64_t)(TBK * OS);
  for (int e = tid; e < TBK * OS; e += nthr) {
    const int kk = e % TBK, r = e / TBK;
    const int64_t i = i0 + kt * TBK + kk;
    const int64_t row = rt * BM + r;
    blk[kk * OS + r] = (r < BM && row < l && i < m) ? Q[i + row * ldq] : 0.0;
  }
}
__global__ void __launch_bounds__(128) k_omega_pack(const double* __restrict__ Q, int64_t ldq, int l, int64_t i0, int64_t m,
                                                    int BM, int OS, int64_t KT, double* __restrict__ img) {
  pack_tile(Q, ldq, l, i0, m, BM, OS, KT, blockIdx.x, img, threadIdx.x, 128);
}

// The image of a GIVEN row operand Q (M x K, column-major, ld ldq) for the GEMM E = C - Q B: block
// (row tile rt of M, k tile kt of K) = [TBK][OS] with img(kk, r) = Q(rt*BM + r, kt*TBK + kk); one CTA
// per block, threads along r (contiguous in Q's columns).
__global__ void __launch_bounds__(128) k_pack_rows(const double* __restrict__ Q, int64_t ldq, int64_t M, int64_t K,
                                                   int BM, int OS, int64_t KT, double* __restrict__ img) {
  const int64_t tile = blockIdx.x;
  const int64_t rt = tile / KT, kt = tile - (tile / KT) * KT;
  double* blk = img + tile * (int64_t)(TBK * OS);
  for (int e = threadIdx.x; e < TBK * OS; e += 128) {
    const int kk = e / OS, r = e - kk * OS;
    const int64_t row = rt * BM + r, kq = kt * TBK + kk;
    blk[e] = (r < BM && row < M && kq < K) ? Q[row + kq * ldq] : 0.0;
  }
}

__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_load_hint(unsigned dst, const void* src, unsigned bytes, unsigned mbar,
                                               unsigned long long policy) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar), "l"(policy) : "memory");
}
#ifndef SKEL_SKETCH_HINTS
#define SKEL_SKETCH_HINTS 1
#endif
// L2 policy of the sketch GEMM's loads: the Omega image slot is re-read by every column tile of A
// (keep: evict_last), a tile of A by the l / BM row-tile CTAs co-scheduled with it (evict_first)

// MODE 0: one K range, X written directly; 1: K-split partials to HBM (+ k_sketch_splitk_reduce);
// 2: the gridDim.z K-splits of a tile form one cluster and are summed through distributed shared
// memory in rank order (deterministic), each rank writing 1/S of the tile's rows.
template <class C, int MODE>
__global__ void __launch_bounds__(C::NT, C::CPS) k_sketch_pre(const __grid_constant__ CUtensorMap tmA, DenseParams p,
                                                               const double* __restrict__ img, int64_t KT) {
  constexpr int TS = C::TS, BM = C::BM, NW = C::NW, FI = C::FI, FJ = C::FJ;
  if (MODE == 0 && p.done) {
    // chained chunks: this chunk's image was made by generator CTAs of the previous GEMM -- wait for
    // them, not for that whole GEMM (whose last wave this grid's CTAs fill); let the next GEMM be
    // scheduled; generator CTAs then make the next chunk's image before their own tile
    if (p.ready) wait_count(p.ready, p.ready_need);
    else dev::griddep_wait();                            // chunk 0: its image is the preceding kernel
    dev::griddep_launch();
    const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (p.gen_img && lin - p.gen_lo < p.gen_n) {
      wait_count(p.gen_gate, p.gen_need);
      const int64_t tiles = (int64_t)((p.l + BM - 1) / BM) * p.gen_kt;
      for (int64_t t = lin - p.gen_lo; t < tiles; t += p.gen_n) {
        if (p.gen_q) pack_tile(p.gen_q, p.gen_ldq, p.l, p.gen_i0, p.gen_i1, BM, C::OS, p.gen_kt, t, p.gen_img, threadIdx.x, C::NT);
        else omega_tile(p.key, p.l, p.gen_i0, p.gen_i1, BM, C::OS, p.gen_kt, t, p.gen_img, threadIdx.x, C::NT);
      }
      count_done(p.gen_ready);
    }
  } else {
    dev::griddep_wait();                                 // PDL: the Omega image is complete
  }
  extern __shared__ __align__(1024) unsigned char psm_raw[];
  unsigned char* base = psm_raw + ((1024u - (dev::smem_addr(psm_raw) & 1023u)) & 1023u);
  const unsigned base_u = dev::smem_addr(base);
  const unsigned fullB = base_u + TS * C::ST_BYTES, emptyB = fullB + 8 * TS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rt = blockIdx.x;
  const int64_t n0 = (int64_t)blockIdx.y * C::TBNP;
  const int64_t kbeg = p.k0 + (int64_t)blockIdx.z * p.k_per_split;
  const int64_t kend = min(p.m, kbeg + p.k_per_split);
  const int ktiles = (int)((kend - kbeg + TBK - 1) / TBK);
  const int64_t kt0 = (kbeg - p.k0) / TBK;              // k tile within the chunk's Omega image
  if (tid == 0) {
    for (int s = 0; s < TS; ++s) {
      dev::mbar_init(fullB + 8 * s, 1);
      dev::mbar_init(emptyB + 8 * s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    dev::prefetch_tmap(&tmA);
  }
  __syncthreads();
  const double* img_rt = img + ((int64_t)rt * KT) * (TBK * C::OS);
  // number of 64-column tensor loads with any column inside A (the rest of the tile stays stale)
  constexpr int PBOX = C::PBOX;
  const int64_t nbox_all = (p.n - n0 + PBOX - 1) / PBOX;
  const int nbox = (int)(nbox_all < C::TBNP / PBOX ? nbox_all : C::TBNP / PBOX);
  int issued = 0;
  const unsigned long long pol_a = SKEL_SKETCH_HINTS ? dev::policy_evict_first() : 0ull;
  const unsigned long long pol_o = SKEL_SKETCH_HINTS ? dev::policy_evict_last() : 0ull;
  auto issue = [&](int upto, bool block) {
    while (issued < upto && issued < ktiles) {
      const int kq = issued, sq = kq % TS;
      if (kq >= TS) {
        const unsigned par = ((unsigned)(kq / TS) & 1u) ^ 1u;
        if (block) dev::mbar_wait(emptyB + 8 * sq, par);
        else if (!dev::mbar_test(emptyB + 8 * sq, par)) break;
      }
      const unsigned st = base_u + sq * C::ST_BYTES;
      dev::mbar_arm(fullB + 8 * sq, (unsigned)(nbox * PBOX * TBK * 8 + C::O_BYTES));
      if (SKEL_SKETCH_HINTS) {
        bulk_load_hint(st + C::A_BYTES, img_rt + (kt0 + kq) * (TBK * C::OS), (unsigned)C::O_BYTES, fullB + 8 * sq, pol_o);
        for (int b = 0; b < nbox; ++b)
          dev::tma_load_2d_hint(st + b * PBOX * TBK * 8, &tmA, (int)(kbeg + (int64_t)kq * TBK), (int)(n0 + b * PBOX),
                                fullB + 8 * sq, pol_a);
      } else {
        bulk_load(st + C::A_BYTES, img_rt + (kt0 + kq) * (TBK * C::OS), (unsigned)C::O_BYTES, fullB + 8 * sq);
        for (int b = 0; b < nbox; ++b)
          dev::tma_load_2d(st + b * PBOX * TBK * 8, &tmA, (int)(kbeg + (int64_t)kq * TBK), (int)(n0 + b * PBOX), fullB + 8 * sq);
      }
      ++issued;
    }
  };
  const int g = lane >> 2, q = lane & 3;
  const int wm = warp % C::WM;                             // warp row (FI fragments of 8 rows)
  const int wr = wm * FI * 8;                              // first row of the warp within the tile
  const int wn = (warp / C::WM) * FJ * 8;                  // first column of the warp within the tile
  const int sg = sig8(g);
  double acc[FI][FJ][2];
#pragma unroll
  for (int i = 0; i < FI; ++i)
#pragma unroll
    for (int j = 0; j < FJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const bool lead = tid == 0;
  const bool active = n0 + wn < p.n;                       // warp has columns inside A
  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % TS;
    if (lead) {
      issue(kt + 1, true);
      issue(kt + TS, false);
    }
    __syncwarp();
    dev::mbar_wait(fullB + 8 * s, (unsigned)(kt / TS) & 1u);
    if (active) {
      const unsigned char* st = base + (size_t)s * C::ST_BYTES;
      const double* Os = reinterpret_cast<const double*>(st + C::A_BYTES) + q * C::OS + g + wr;
      const unsigned char* At = st + (size_t)(wn + sg) * 128 + ((q & 1) << 3);
#pragma unroll
      for (int kk = 0; kk < TBK / 4; ++kk) {
        double a[FI], b[FJ];
#pragma unroll
        for (int i = 0; i < FI; ++i) a[i] = Os[kk * 4 * C::OS + i * 8];
        const int inrow = ((2 * kk + (q >> 1)) ^ sg) << 4;
#pragma unroll
        for (int j = 0; j < FJ; ++j) b[j] = *reinterpret_cast<const double*>(At + j * 8 * 128 + inrow);
#pragma unroll
        for (int i = 0; i < FI; ++i)
#pragma unroll
          for (int j = 0; j < FJ; ++j) dev::dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_local(emptyB + 8 * s);
  }
  const int c0 = sig8(2 * q), c1 = sig8(2 * q + 1);
  if (MODE == 4) {
    // residual epilogue (S6): e = Csub(r, col) - acc, squared and summed with Csub^2; Csub (the
    // m x n A, column-major) is read once, streamed; nothing of the m x n residual is written
    double se = 0.0, sc = 0.0;
    if (active) {
#pragma unroll
      for (int i = 0; i < FI; ++i) {
        const int64_t r = (int64_t)rt * BM + wr + i * 8 + g;
        if (r >= p.l) continue;
#pragma unroll
        for (int j = 0; j < FJ; ++j) {
          const int64_t cb = n0 + wn + j * 8;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t col = cb + (h ? c1 : c0);
            if (col < p.n) {
              const double a = __ldcs(p.Csub + r + col * p.ldcs);
              const double e = a - acc[i][j][h];
              se = fma(e, e, se);
              sc = fma(a, a, sc);
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      se += __shfl_xor_sync(0xffffffffu, se, o);
      sc += __shfl_xor_sync(0xffffffffu, sc, o);
    }
    __shared__ double wred[2 * NW];
    if (lane == 0) { wred[2 * warp] = se; wred[2 * warp + 1] = sc; }
    __syncthreads();
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < NW; ++w) { a += wred[2 * w]; b += wred[2 * w + 1]; }
      const int64_t lin = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
      p.sums_part[2 * lin] = a;
      p.sums_part[2 * lin + 1] = b;
    }
    return;
  }
  if (MODE == 2) {
    constexpr int TST = C::TBNP + 1;                        // tile row stride (odd: fewer conflicts)
    static_assert((size_t)BM * TST * 8 <= (size_t)TS * C::ST_BYTES, "tile fits the ring");
    __syncthreads();                                        // every stage consumed: the ring is free
    double* T = reinterpret_cast<double*>(base);
#pragma unroll
    for (int i = 0; i < FI; ++i)
#pragma unroll
      for (int j = 0; j < FJ; ++j) {
        T[(wr + i * 8 + g) * TST + wn + j * 8 + c0] = acc[i][j][0];
        T[(wr + i * 8 + g) * TST + wn + j * 8 + c1] = acc[i][j][1];
      }
    dev::cluster_arrive();
    dev::cluster_wait();
    const unsigned S = gridDim.z, rank = dev::cluster_ctarank();
    const int rows = BM / (int)S;
    for (int e = tid; e < rows * C::TBNP; e += C::NT) {
      const int rl = (int)rank * rows + e / C::TBNP, col = e % C::TBNP;
      const unsigned a = dev::smem_addr(T + rl * TST + col);
      double sum = 0.0;
      for (unsigned r = 0; r < S; ++r) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(dev::mapa(a, r)));
        sum += v;
      }
      const int r = rt * BM + rl;
      const int64_t cn = n0 + col;
      if (r < p.l && cn < p.n) {
        double* dst = p.X + (int64_t)r * p.ldx + cn;
        *dst = p.accum ? *dst + sum * p.scale : sum * p.scale;
      }
    }
    dev::cluster_arrive();                                  // no CTA leaves while peers read it
    dev::cluster_wait();
    return;
  }
  if (MODE == 0 && p.tile_ord) {                        // chained chunks: the previous chunk's adds first
    const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    wait_count(p.tile_ord + lin, p.chunk_idx);
  }
  if (active) {
#pragma unroll
  for (int i = 0; i < FI; ++i) {
    const int r = rt * BM + wr + i * 8 + g;
    if (r >= p.l) continue;
#pragma unroll
    for (int j = 0; j < FJ; ++j) {
      const int64_t cb = n0 + wn + j * 8;
      if (MODE == 1) {
        double* dst = p.part + ((int64_t)blockIdx.z * p.l + r) * p.n;
        if (cb + c0 < p.n) dst[cb + c0] = acc[i][j][0];
        if (cb + c1 < p.n) dst[cb + c1] = acc[i][j][1];
      } else {
        double* dst = p.X + (int64_t)r * p.ldx;
        if (p.accum) {
          // later K-chunks add into X with fire-and-forget reductions (no load round trip holding the
          // SM); each element gets one add per chunk and the chunks are stream-ordered, so the
          // summation order -- hence X -- is deterministic
          if (cb + c0 < p.n) red_add_f64(dst + cb + c0, acc[i][j][0] * p.scale);
          if (cb + c1 < p.n) red_add_f64(dst + cb + c1, acc[i][j][1] * p.scale);
        } else {
          if (cb + c0 < p.n) dst[cb + c0] = acc[i][j][0] * p.scale;
          if (cb + c1 < p.n) dst[cb + c1] = acc[i][j][1] * p.scale;
        }
      }
    }
  }
  }
  if (MODE == 0 && p.done) {                              // chained chunks: this tile is in X
    __syncthreads();
    if (tid == 0) {
      if (p.tile_ord) {
        const unsigned lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.tile_ord + lin) : "memory");
      }
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.done) : "memory");
    }
  }
}

// ============================================================ sparse-sign sketch
constexpr int SCH = 128;          // rows of A per chunk (4 mask words)
constexpr int SMW = SCH / 32;
constexpr int SCOLS = 32;         // columns per CTA (lane = column)
constexpr int SNT = 512;          // 16 warps
constexpr int SNW = SNT / 32;
constexpr int SAS = SCH + 1;      // A tile stride (odd -> conflict-free lane-strided reads)

struct SparseParams {
  const double* A; int64_t lda;
  int64_t m, n; int l; int zeta;
  uint2 key;
  double scale;                   // 1/sqrt(zeta)
  double* X; int64_t ldx;
};

// Each warp owns output rows r = warp + SNW*j, j < J (J = ceil(l / SNW) <= JMAX).
// Per chunk the nonzeros of Gamma(:, i0:i0+SCH) are recorded as two bit masks per
// output row (hit, negative) built with atomicOr -- order independent -- and the
// gather walks the set bits in ascending i, so the summation order is fixed.
template <int JMAX>
__global__ void __launch_bounds__(SNT, 1) k_sketch_sparse(SparseParams p) {
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                                                // [SCOLS][SAS]
  uint32_t* hit = reinterpret_cast<uint32_t*>(As + SCOLS * SAS);  // [l][SMW]
  uint32_t* neg = hit + (size_t)p.l * SMW;                        // [l][SMW]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * SCOLS;
  const int J = (p.l + SNW - 1) / SNW;
  double acc[JMAX];
#pragma unroll
  for (int j = 0; j < JMAX; ++j) acc[j] = 0.0;

  for (int64_t i0 = 0; i0 < p.m; i0 += SCH) {
    const int rows_here = (int)((p.m - i0) < SCH ? (p.m - i0) : SCH);
    // (1) stage A(i0:i0+SCH, n0:n0+32); consecutive threads -> consecutive i (coalesced)
    for (int e = threadIdx.x; e < SCOLS * SCH; e += SNT) {
      const int col = e / SCH, ii = e % SCH;
      const int64_t gn = n0 + col;
      As[col * SAS + ii] = (ii < rows_here && gn < p.n) ? p.A[(i0 + ii) + gn * p.lda] : 0.0;
    }
    for (int e = threadIdx.x; e < p.l * SMW; e += SNT) { hit[e] = 0u; neg[e] = 0u; }
    __syncthreads();
    // (2) draw the chunk's nonzeros of Gamma, one column i of Gamma per thread
    if (threadIdx.x < rows_here) {
      const int ii = threadIdx.x;
      int rows[64];
      const uint64_t sbits = dev::sparse_col((uint64_t)(i0 + ii), p.l, p.zeta, p.key, rows);
      const uint32_t bit = 1u << (ii & 31);
      for (int j = 0; j < p.zeta; ++j) {
        atomicOr(&hit[rows[j] * SMW + (ii >> 5)], bit);
        if ((sbits >> j) & 1ull) atomicOr(&neg[rows[j] * SMW + (ii >> 5)], bit);
      }
    }
    __syncthreads();
    // (3) gather: lane = column, warp = row subset; ascending i within each row
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      if (j >= J) break;
      const int r = warp + SNW * j;
      if (r < p.l) {
        double s = acc[j];
#pragma unroll
        for (int w = 0; w < SMW; ++w) {
          uint32_t bits = hit[r * SMW + w];
          const uint32_t nb = neg[r * SMW + w];
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const double v = As[lane * SAS + w * 32 + b];
            s = ((nb >> b) & 1u) ? s - v : s + v;
          }
        }
        acc[j] = s;
      }
    }
    __syncthreads();
  }
  const int64_t col = n0 + lane;
  if (col < p.n) {
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      if (j >= J) break;
      const int r = warp + SNW * j;
      if (r < p.l) p.X[(int64_t)r * p.ldx + col] = acc[j] * p.scale;
    }
  }
}

// ------------------------------------------------------------ sparse-sign sketch, warp-specialised
// CW consumer warps (lane = column of a 32-column block, warp w owns output rows r = w + CW jj held
// in registers) + 1 producer warp that builds the Omega structure of each 128-row chunk of A as
// per-output-row bit masks (hit / negative; Floyd rows and sign bits from Philox, R1/R4) into a
// 4-deep mask ring (full/empty mbarriers).  The consumers stream A through a 3-stage shared ring
// with software-pipelined coalesced loads (one chunk in registers, one in flight), and walk the
// mask bits of their rows in ascending i: X(r, j) += +-A(i, j) -- a fixed summation order.
constexpr int S2_R = 128, S2_W = 32;
constexpr int S2_AS = S2_R + 1, S2_NA = 3, S2_NM = 4, S2_MW = S2_R / 32;

__host__ __device__ constexpr size_t s2_smem(int l) {
  return (size_t)S2_NA * S2_W * S2_AS * 8 + (size_t)S2_NM * l * S2_MW * 2 * 4 + 2 * S2_NM * 8 + 16;
}

template <int S2_CW, int J>
__global__ void __launch_bounds__((S2_CW + 1) * 32, 1) k_sketch_sparse2(SparseParams p) {
  // (CW + 1 warps: registers are allocated as for a multiple of 4 warps, so CW = 7 or 15)
  constexpr int S2_LD = (S2_R * S2_W + S2_CW * 32 - 1) / (S2_CW * 32);   // A doubles per consumer thread per chunk
  extern __shared__ __align__(16) unsigned char s2raw[];
  double* As = reinterpret_cast<double*>(s2raw);                                        // [NA][W][AS]
  uint32_t* masks = reinterpret_cast<uint32_t*>(As + (size_t)S2_NA * S2_W * S2_AS);     // [NM][2][l][MW]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(masks + (size_t)S2_NM * p.l * S2_MW * 2);
  const unsigned mfull = dev::smem_addr(bars), mempty = mfull + 8 * S2_NM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * S2_W;
  const int nchunks = (int)((p.m + S2_R - 1) / S2_R);
  const size_t mstage = (size_t)p.l * S2_MW * 2;
  if (tid == 0) {
    for (int s = 0; s < S2_NM; ++s) {
      dev::mbar_init(mfull + 8 * s, 1);
      dev::mbar_init(mempty + 8 * s, S2_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == S2_CW) {
    // ---------------------------------------------------------------- producer: Omega masks
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % S2_NM;
      if (c >= S2_NM) dev::mbar_wait(mempty + 8 * s, ((unsigned)(c / S2_NM) & 1u) ^ 1u);
      uint32_t* hit = masks + (size_t)s * mstage;
      uint32_t* neg = hit + (size_t)p.l * S2_MW;
      uint4* z4 = reinterpret_cast<uint4*>(hit);
      for (int e = lane; e < (int)(mstage / 4); e += 32) z4[e] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
      for (int ii = lane; ii < S2_R; ii += 32) {
        const int64_t i = (int64_t)c * S2_R + ii;
        if (i < p.m) {
          int rows[64];
          const uint64_t sb = dev::sparse_col((uint64_t)i, p.l, p.zeta, p.key, rows);
          const uint32_t bit = 1u << (ii & 31);
          const int w = ii >> 5;
          for (int j = 0; j < p.zeta; ++j) {
            atomicOr(&hit[rows[j] * S2_MW + w], bit);
            if ((sb >> j) & 1ull) atomicOr(&neg[rows[j] * S2_MW + w], bit);
          }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mfull + 8 * s) : "memory");
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  double acc[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) acc[jj] = 0.0;
  double pre[S2_LD];
  auto load_chunk = [&](int c) {
#pragma unroll
    for (int q = 0; q < S2_LD; ++q) {
      const int e = tid + q * (S2_CW * 32);
      const int col = e / S2_R, ii = e % S2_R;
      const int64_t i = (int64_t)c * S2_R + ii, j = n0 + col;
      pre[q] = (e < S2_R * S2_W && i < p.m && j < p.n) ? __ldcs(p.A + i + j * p.lda) : 0.0;   // streamed once
    }
  };
  auto store_chunk = [&](int c) {
    double* dst = As + (size_t)(c % S2_NA) * S2_W * S2_AS;
#pragma unroll
    for (int q = 0; q < S2_LD; ++q) {
      const int e = tid + q * (S2_CW * 32);
      if (e < S2_R * S2_W) dst[(e / S2_R) * S2_AS + (e % S2_R)] = pre[q];
    }
  };
  load_chunk(0);
  store_chunk(0);
  if (nchunks > 1) load_chunk(1);
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) store_chunk(c + 1);
    if (c + 2 < nchunks) load_chunk(c + 2);
    asm volatile("bar.sync 1, %0;" ::"n"(S2_CW * 32) : "memory");
    const int s = c % S2_NM;
    dev::mbar_wait(mfull + 8 * s, (unsigned)(c / S2_NM) & 1u);
    const uint32_t* hit = masks + (size_t)s * mstage;
    const uint32_t* neg = hit + (size_t)p.l * S2_MW;
    const double* At = As + (size_t)(c % S2_NA) * S2_W * S2_AS + lane * S2_AS;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int r = warp + S2_CW * jj;
      if (r < p.l) {
        const uint4 h = *reinterpret_cast<const uint4*>(hit + r * S2_MW);
        const uint4 g = *reinterpret_cast<const uint4*>(neg + r * S2_MW);
        double a = acc[jj];
        unsigned long long hb = ((unsigned long long)h.y << 32) | h.x, nb = ((unsigned long long)g.y << 32) | g.x;
        while (hb) {
          const int b = __ffsll((long long)hb) - 1;
          hb &= hb - 1;
          const long long sgn = (long long)((nb >> b) & 1ull) << 63;
          a += __longlong_as_double(__double_as_longlong(At[b]) ^ sgn);
        }
        hb = ((unsigned long long)h.w << 32) | h.z;
        nb = ((unsigned long long)g.w << 32) | g.z;
        while (hb) {
          const int b = __ffsll((long long)hb) - 1;
          hb &= hb - 1;
          const long long sgn = (long long)((nb >> b) & 1ull) << 63;
          a += __longlong_as_double(__double_as_longlong(At[64 + b]) ^ sgn);
        }
        acc[jj] = a;
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(mempty + 8 * s) : "memory");
  }
  const int64_t col = n0 + lane;
  if (col < p.n) {
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int r = warp + S2_CW * jj;
      if (r < p.l) p.X[(int64_t)r * p.ldx + col] = acc[jj] * p.scale;
    }
  }
}


// ------------------------------------------------------------ sparse-sign sketch v4: precomputed CSR
// Omega's structure is the same for every column tile, so it is built ONCE per call by
// k_sparse_csr into a small L2-resident table (Omega's values +-1/sqrt(zeta) are never stored):
// per 256-row chunk of A, for every output row r the list of its nonzeros in the chunk, ascending
// i, as 32-bit entries (byte offset of i in a tile column | sign << 31), padded to an even count
// with entries that point at a zero element; row r's header = (first 8-byte pair, #pairs).
// k_sketch_sparse4 has no producer and no cluster: all 16 warps are consumers (lane = column of a
// 32-column tile, warp w owns the contiguous output rows [w J, w J + J) in registers); A streams
// by 8-byte cp.async into a padded double-buffered tile and the chunk's CSR rides in the same
// cp.async group.  A row's walk is one 8-byte load per 2 entries and 2 independent shared loads,
// sign flips and adds (pairs pad 11 % of the entries where groups of 4 padded 37 %: C3 1.22 -> 1.11 ms).  Summation order is fixed (chunk by chunk, ascending i) -- deterministic.
// Two i-halves per column tile (split = 2) fill the last wave; their partials meet in X by atomic
// add from zero, which is order independent for two terms (fl(fl(0 + a) + b) = fl(a + b)).
constexpr int S4_R = 256, S4_W = 32, S4_AS = S4_R + 1;
struct S4Geom {
  int rows_pad;   // S4_NW * J: rows with headers (rows >= l have empty lists)
  int groups;     // 8-byte entry pairs per chunk (upper bound, even)
  int bytes;      // bytes per chunk record = 4 rows_pad + 8 groups (a multiple of 16)
};
__host__ __device__ inline S4Geom s4_geom(int J, int NW, int zeta) {
  S4Geom g;
  g.rows_pad = NW * J;
  g.groups = ((S4_R * zeta + g.rows_pad + 1) / 2 + 1) & ~1;
  g.bytes = 4 * g.rows_pad + 8 * g.groups;
  return g;
}
__host__ __device__ inline size_t s4_smem(const S4Geom& g) {
  return (size_t)2 * S4_W * S4_AS * 8 + (size_t)2 * g.bytes;
}

__global__ void __launch_bounds__(S4_R) k_sparse_csr(SparseParams p, unsigned char* __restrict__ csr, S4Geom geo) {
  extern __shared__ __align__(16) int s4c[];
  const int nr = geo.rows_pad;
  int* cnt = s4c;                                                     // [nr]: count, then fill cursor
  int* gst = cnt + nr;                                                // [nr]: first group of the row
  uint32_t* ent = reinterpret_cast<uint32_t*>(gst + nr);              // [4 groups]
  const int tid = threadIdx.x;
  const int64_t c = blockIdx.x;
  const int64_t i = c * S4_R + tid;
  const bool valid = i < p.m;
  for (int r = tid; r < nr; r += S4_R) cnt[r] = 0;
  for (int e = tid; e < 2 * geo.groups; e += S4_R) ent[e] = (uint32_t)(S4_R * 8);   // padding -> zero element
  __syncthreads();
  int rows[8];
  const uint64_t sb = dev::sparse_col8((uint64_t)(valid ? i : 0), p.l, p.zeta, p.key, rows);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (valid && rows[j] >= 0) atomicAdd(&cnt[rows[j]], 1);
  __syncthreads();
  // exclusive scan of the padded group counts: each thread a contiguous row segment + warp scans
  const int seg = (nr + S4_R - 1) / S4_R;
  const int r0 = min(nr, tid * seg), r1 = min(nr, r0 + seg);
  int local = 0;
  for (int r = r0; r < r1; ++r) local += (cnt[r] + 1) >> 1;
  __shared__ int wsum[S4_R / 32];
  int incl = local;
  const int lane = tid & 31, w = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  int run = incl - local;
  for (int q = 0; q < w; ++q) run += wsum[q];
  uint32_t* hdr = reinterpret_cast<uint32_t*>(csr + c * geo.bytes);
  for (int r = r0; r < r1; ++r) {
    const int ng = (cnt[r] + 1) >> 1;
    gst[r] = run;
    hdr[r] = (uint32_t)run | ((uint32_t)ng << 16);
    run += ng;
    cnt[r] = 2 * gst[r];                                                 // fill cursor (entry index)
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (valid && rows[j] >= 0) {
      const int pos = atomicAdd(&cnt[rows[j]], 1);
      ent[pos] = (uint32_t)(tid * 8) | ((uint32_t)((sb >> j) & 1ull) << 31);
    }
  __syncthreads();
  for (int r = tid; r < nr; r += S4_R) {                               // ascending i within the row
    const int e0 = 2 * gst[r], e1 = cnt[r];
    for (int x = e0 + 1; x < e1; ++x) {
      const uint32_t v = ent[x];
      int y = x - 1;
      while (y >= e0 && (ent[y] & 0xffffu) > (v & 0xffffu)) { ent[y + 1] = ent[y]; --y; }
      ent[y + 1] = v;
    }
  }
  __syncthreads();
  uint32_t* out = hdr + nr;
  for (int e = tid; e < 2 * geo.groups; e += S4_R) out[e] = ent[e];
}

template <int J, int S4_NW>
__global__ void __launch_bounds__(S4_NW * 32, 1) k_sketch_sparse4(SparseParams p, const unsigned char* __restrict__ csr,
                                                                   S4Geom geo, int nchunks, int split) {
  extern __shared__ __align__(16) unsigned char s4raw[];
  double* As = reinterpret_cast<double*>(s4raw);                                   // [2][W][AS]
  unsigned char* Cs = s4raw + (size_t)2 * S4_W * S4_AS * 8;                       // [2][bytes]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * S4_W;
  const int cper = (nchunks + split - 1) / split;
  const int cb = blockIdx.y * cper, ce = min(nchunks, cb + cper);
  const int r0 = warp * J;
  static_assert(S4_R * S4_W % (S4_NW * 32) == 0 && S4_NW * 32 % S4_R == 0, "tile loads");
  if (tid < 2 * S4_W) As[(tid >> 5) * S4_W * S4_AS + (tid & 31) * S4_AS + S4_R] = 0.0;   // the zero element
  double acc[J];
#pragma unroll
  for (int jj = 0; jj < J; ++jj) acc[jj] = 0.0;
  // A tile loads: thread covers row ii = tid % R of the chunk and columns colt + 2q (q < 16)
  constexpr int NQ = S4_R * S4_W / (S4_NW * 32);
  constexpr int CSTEP = S4_NW * 32 / S4_R;            // columns covered by one pass of the CTA
  const int ii = tid % S4_R, colt = tid / S4_R;
  const int64_t lda = p.lda;
  const double* abase = p.A + (n0 + colt) * lda + ii;
  uint32_t jmask = 0u;
#pragma unroll
  for (int q = 0; q < NQ; ++q) jmask |= (n0 + colt + CSTEP * q < p.n ? 1u : 0u) << q;
  auto issue = [&](int c) {
    const int st = c & 1;
    double* dst = As + st * S4_W * S4_AS + colt * S4_AS + ii;
    const bool iok = (int64_t)c * S4_R + ii < p.m;
    const double* src = abase + (int64_t)c * S4_R;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const bool ok = iok && ((jmask >> q) & 1u);
      dev::cp_async8(dst + CSTEP * q * S4_AS, ok ? src + CSTEP * q * lda : p.A, ok);
    }
    const unsigned char* csrc = csr + (int64_t)c * geo.bytes;
    unsigned char* cd = Cs + st * geo.bytes;
    for (int e = tid; e < geo.bytes / 16; e += S4_NW * 32) dev::cp_async16(cd + 16 * e, csrc + 16 * e, 16);
    dev::cp_async_commit();
  };
  if (cb < ce) issue(cb);
  for (int c = cb; c < ce; ++c) {
    dev::cp_async_wait<0>();
    __syncthreads();                                      // chunk c landed; stage c+1 free (consumed at c-1)
    if (c + 1 < ce) issue(c + 1);
    const int st = c & 1;
    const uint32_t* hdr = reinterpret_cast<const uint32_t*>(Cs + st * geo.bytes);
    const uint2* grp = reinterpret_cast<const uint2*>(hdr + geo.rows_pad);
    const char* At = reinterpret_cast<const char*>(As + st * S4_W * S4_AS + lane * S4_AS);
    uint4 h4;
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      if (jj % 4 == 0) h4 = reinterpret_cast<const uint4*>(hdr + r0)[jj / 4];   // 4 row headers per broadcast load
      const uint32_t h = jj % 4 == 0 ? h4.x : jj % 4 == 1 ? h4.y : jj % 4 == 2 ? h4.z : h4.w;
      const int g0 = (int)(h & 0xffffu), g1 = g0 + (int)(h >> 16);
      double a = acc[jj];
#pragma unroll 1
      for (int g = g0; g < g1; ++g) {
        const uint2 w2 = grp[g];
        const uint32_t wv[2] = {w2.x, w2.y};
        double x[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double v = *reinterpret_cast<const double*>(At + (wv[q] & 0xffffu));
          x[q] = __hiloint2double(__double2hiint(v) ^ (int)(wv[q] & 0x80000000u), __double2loint(v));
        }
        a += x[0];
        a += x[1];
      }
      acc[jj] = a;
    }
  }
  const int64_t col = n0 + lane;
  if (col < p.n) {
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      const int r = r0 + jj;
      if (r < p.l) {
        double* dst = p.X + (int64_t)r * p.ldx + col;
        if (split == 1) *dst = acc[jj] * p.scale;
        else atomicAdd(dst, acc[jj] * p.scale);
      }
    }
  }
}

template <int J, int NW>
sk_status launch_sparse4(sk_ctx* c, const SparseParams& p) {
  const int nchunks = (int)cdiv(p.m, S4_R);
  const S4Geom geo = s4_geom(J, NW, p.zeta);
  DBuf csr;
  SK_TRY(csr.alloc(c, (size_t)nchunks * geo.bytes));
  const size_t csmem = (size_t)geo.rows_pad * 8 + (size_t)geo.groups * 8;
  SK_CUDA(c, cudaFuncSetAttribute(k_sparse_csr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
  k_sparse_csr<<<(unsigned)nchunks, S4_R, csmem, c->stream>>>(p, csr.as<unsigned char>(), geo);
  SK_TRY(launched(c));
  // i-split for the last wave: 2 halves when it raises the filled fraction of the waves by > 5%
  const int64_t tiles = cdiv(p.n, S4_W);
  auto eff = [&](int64_t u) { return (double)u / (double)(cdiv(u, c->num_sms) * c->num_sms); };
  const int split = (nchunks >= 2 && eff(2 * tiles) > eff(tiles) + 0.05) ? 2 : 1;
  if (split > 1)
    SK_CUDA(c, cudaMemset2DAsync(p.X, p.ldx * sizeof(double), 0, p.n * sizeof(double), p.l, c->stream));
  const size_t smem = s4_smem(geo);
  SK_CUDA(c, cudaFuncSetAttribute(k_sketch_sparse4<J, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_sketch_sparse4<J, NW><<<dim3((unsigned)tiles, (unsigned)split), NW * 32, smem, c->stream>>>(
      p, csr.as<unsigned char>(), geo, nchunks, split);
  return launched(c);
}

template <int CW, int J>
sk_status launch_sparse2(sk_ctx* c, const SparseParams& p) {
  const size_t smem = s2_smem(p.l);
  SK_CUDA(c, cudaFuncSetAttribute(k_sketch_sparse2<CW, J>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_sketch_sparse2<CW, J><<<(unsigned)cdiv(p.n, S2_W), (CW + 1) * 32, smem, c->stream>>>(p);
  return launched(c);
}

template <int JMAX>
sk_status launch_sparse(sk_ctx* c, const SparseParams& p) {
  const size_t smem = (size_t)SCOLS * SAS * sizeof(double) + 2 * sizeof(uint32_t) * (size_t)p.l * SMW;
  SK_CUDA(c, cudaFuncSetAttribute(k_sketch_sparse<JMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  const dim3 grid((unsigned)cdiv(p.n, SCOLS));
  k_sketch_sparse<JMAX><<<grid, SNT, smem, c->stream>>>(p);
  return launched(c);
}

}  // namespace

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q{};
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    cudaGetLastError();
  }
  return fn;
}

struct PrePlan {
  int geo = 0, bm = 0, nw = 0, splits = 1;
  bool cluster = true;     // K-splits reduced in-cluster when eligible (<= 8, dividing BM)
  int64_t chunk = 0;       // rows of A per K-chunk (the Omega image slot holds one chunk)
  double cost = 1e300;
};
// An Omega image slot at most this large stays (mostly) in the 126 MB L2 next to the streaming A
// tiles.  Measured at C5 (131072 x 8192 block, l = 1100): 40 MB slots (32 chunks) 84.9% of the
// DMMA ceiling, 80 MB (16 chunks) 86.3%, one 1.2 GB image 87.7% (profiles/round2/sketch_chunks.txt):
// the per-chunk cost is the launch tail and the X read-modify-write, not L2 misses on the slot.
constexpr double kOmegaSlotBytes = 80.0 * (1 << 20);

// The tile geometries of k_sketch_pre the planner chooses from (G_W56 only on request).
enum PreGeo { G_W48 = 0, G_W64, G_W32, G_W40, G_W40_7, G_W48_7, G_W56, G_N80, G_N40, G_T80, G_T48, G_T96, G_COUNT };
struct GeoDesc { int bm, nw, tbn, cps; };
constexpr GeoDesc kGeo[G_COUNT] = {{48, 8, 256, 1}, {64, 8, 256, 1}, {32, 8, 256, 1}, {40, 8, 256, 1},
                                   {40, 7, 224, 1}, {48, 7, 224, 1}, {56, 8, 256, 1}, {80, 4, 112, 2},
                                   {40, 2, 112, 4}, {80, 12, 192, 1}, {48, 12, 384, 1}, {96, 8, 128, 1}};
using CfgW48 = PCfgW<48, 8>;
using CfgW64 = PCfgW<64, 8>;
using CfgW32 = PCfgW<32, 8>;
using CfgW40 = PCfgW<40, 8>;
using CfgW40_7 = PCfgW<40, 7>;
using CfgW48_7 = PCfgW<48, 7>;
using CfgW56 = PCfgW<56, 8>;
using CfgN80 = PCfg<80, 2, 2, 7, 2>;     // 80 x 112: 2 x 2 warps of 40 x 56, 2 CTAs per SM
using CfgN40 = PCfg<40, 1, 2, 7, 4>;     // 40 x 112: 2 warps of 40 x 56, 4 CTAs per SM
using CfgT80 = PCfg<80, 2, 6, 4, 1>;     // 80 x 192: 2 x 6 warps of 40 x 32 (3 warps per SM sub-partition)
using CfgT48 = PCfg<48, 1, 12, 4, 1>;    // 48 x 384: 12 warps of 48 x 32
using CfgT96 = PCfg<96, 2, 4, 4, 1>;     // 96 x 128: 2 x 4 warps of 48 x 32
// Calls f(C{}) with the geometry's config type.
template <class F> auto with_geo(int g, F&& f) {
  switch (g) {
    case G_W64: return f(CfgW64{});
    case G_W32: return f(CfgW32{});
    case G_W40: return f(CfgW40{});
    case G_W40_7: return f(CfgW40_7{});
    case G_W48_7: return f(CfgW48_7{});
    case G_W56: return f(CfgW56{});
    case G_N80: return f(CfgN80{});
    case G_N40: return f(CfgN40{});
    case G_T80: return f(CfgT80{});
    case G_T48: return f(CfgT48{});
    case G_T96: return f(CfgT96{});
    default: return f(CfgW48{});
  }
}

// co-resident CTAs of k_sketch_pre<C> launched in clusters of S along z (cached per process)
template <class C> int pre_max_ctas(int S) {
  static int cached[9] = {0};
  if (S < 1 || S > 8) return 0;
  if (cached[S] == 0) {
    auto kern = S > 1 ? k_sketch_pre<C, 2> : k_sketch_pre<C, 0>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(1, 1, (unsigned)S);
    lc.blockDim = dim3(C::NT);
    lc.dynamicSmemBytes = C::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = (unsigned)S;
    lc.attrs = at; lc.numAttrs = 1;
    int ncl = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kern, &lc);
    cudaGetLastError();
    cached[S] = (e == cudaSuccess && ncl > 0) ? ncl * S : -1;
  }
  return cached[S];
}
int pre_capacity(int geo, int S) {
  return with_geo(geo, [&](auto cfg) { return pre_max_ctas<decltype(cfg)>(S); });
}

// rows of A per K-chunk for a row-tile height bm: the largest multiple of 1024 whose Omega image
// fits kOmegaSlotBytes (at least 1024), or all of m
int64_t chunk_rows(int64_t m, int64_t l, int bm, int64_t forced, int64_t col_tiles) {
  if (forced > 0) return std::min<int64_t>(m, cdiv(forced, TBK) * TBK);
  const double per_row = (double)cdiv(l, bm) * (bm + 4) * 8.0;
  // (one whole image for few column tiles -- C4 k=200's 210 MB -- measured 1.6 % faster but would put
  // the whole of Omega in HBM, which S0 excludes: not done)
  (void)col_tiles;
  const int64_t ch = std::max<int64_t>(1024, (int64_t)(kOmegaSlotBytes / per_row) / 1024 * 1024);
  return ch >= m ? m : ch;
}

// (geometry, K-splits per chunk) by a cost model: whole waves of the co-resident CTA count x per-CTA
// DMMA work (padded tiles included) x the CTAs sharing an SM x the load of the busiest SM
// sub-partition (warps are dealt to the 4 sub-partitions round-robin: 7 warps leave one with half
// the work) + split-K overhead, summed over the K-chunks; a candidate must beat the incumbent by 1%
// (fewer splits, less partial traffic, win ties).  Checked against a measured sweep of every plan
// (tools/sweep_pre.py).  The context's tuning (sk_set_sketch_tuning) can pin BM, the warp count, the
// split count and the chunk height.
PrePlan plan_pre(sk_ctx* c, int64_t m, int64_t n, int64_t l) {
  PrePlan best;
  // 8 warps = 256-column tiles; 7 warps = 224; the narrow family 112 (C4's n = 784 = 7 x 112)
  // (BM = 56 is a tuning value only: measured 85.2 % at C5 vs 88.1 % for BM = 48)
  // the automatic candidates; an exact (bm, warps) pin may name any geometry (G_W56, G_T96 are
  // reachable through sk_set_sketch_tuning only)
  const int cand[] = {G_W48, G_W64, G_W32, G_W40, G_W40_7, G_W48_7, G_N80, G_N40, G_T48, G_T80};
  const int ncand = (int)(sizeof(cand) / sizeof(cand[0]));
  const bool pin = c->tune_sketch_bm && c->tune_sketch_nw;
  PrePlan pinned;
  if (pin)
    for (int g = 0; g < G_COUNT; ++g)
      if (kGeo[g].bm == c->tune_sketch_bm && kGeo[g].nw == c->tune_sketch_nw) pinned.geo = g;
  for (int ci = 0; ci < (pin ? 1 : ncand); ++ci) {
    const int geo = pin ? pinned.geo : cand[ci];
    const int bm = kGeo[geo].bm, nw = kGeo[geo].nw, tbn = kGeo[geo].tbn;
    if (c->tune_sketch_bm && c->tune_sketch_bm != bm) continue;
    if (c->tune_sketch_nw && c->tune_sketch_nw != nw) continue;
    const int64_t mb = cdiv(l, bm), nb = cdiv(n, tbn);
    const int64_t ch = chunk_rows(m, l, bm, c->tune_sketch_chunk, cdiv(n, tbn));
    const int64_t nch = cdiv(m, ch);
    // K-splits per chunk 1..8 (any count: 5 fills the waves at C2 k=512), then powers of two up to 64
    for (int splits = 1; splits <= 64; splits = splits < 8 ? splits + 1 : splits * 2) {
      if (c->tune_sketch_splits && splits != c->tune_sketch_splits) continue;
      if (splits > 1 && ch / splits < 512 && !c->tune_sketch_splits) break;
      const int64_t kps = cdiv(cdiv(ch, splits), TBK) * TBK;
      const int64_t sp = cdiv(ch, kps);
      for (int clus = 0; clus < 2; ++clus) {
        if (clus && !(sp > 1 && sp <= 8 && bm % sp == 0)) continue;
        // several CTAs per SM: the in-cluster reduction measured far slower (C4 k=200 N80: 41 % vs
        // 75 % of the DMMA ceiling through HBM partials) -- planned through partials only
        if (clus && kGeo[geo].cps > 1 && !c->tune_sketch_path) continue;
        if ((c->tune_sketch_path == 2 && clus) || (c->tune_sketch_path == 3 && !clus && sp > 1)) continue;
        const int cap = pre_capacity(geo, clus ? (int)sp : 1);   // clusters of 4/8 strand SMs per GPC
        if (cap <= 0) continue;
        const double per_sm = std::max(1.0, (double)cap / c->num_sms);      // CTAs sharing an SM
        const double wps = per_sm * nw;                                     // warps per SM
        const double smsp = std::ceil(wps / 4.0) * 4.0 / wps;                // busiest sub-partition
        // two warps per sub-partition leave DMMA issue gaps that a third fills (C5's full width:
        // 48 x 384 tiles, 12 warps, 93.4 % of the ceiling vs 89.4 % for 48 x 256, 8 warps)
        const double tlp = wps >= 12.0 ? 1.0 : 1.045;
        const double stage = (double)bm * tbn * TBK;
        // one chunk of `rows` rows of A: whole waves x the per-CTA k tiles, + the split-K overhead:
        // summed in-cluster through DSMEM (~0.05 FMA-equivalents per partial element) or through HBM
        // partials + a reduce launch.  (Adding the splits into X in split order through per-tile flags
        // was measured slower: C2 k=512 0.594 -> 0.688 ms, k=16 0.06 -> 0.16 ms -- the splits of a tile
        // then serialise.)  The ragged last chunk is costed at its own height.
        // Chained chunks (>= 3 chunks in one K range each, run_pre) fill each chunk's last wave with the
        // next chunk's CTAs: their waves count fractionally -- when a chunk has at least one full wave
        // (a grid smaller than the GPU leaves it idle however the chunks overlap: C4 k=200 at one split
        // per chunk, 35 CTAs, measured 8.0 ms vs 1.47 ms with 8 splits)
        const bool chained = nch >= 3 && sp == 1 && !clus && mb * nb >= cap;
        auto chunk_cost = [&](int64_t rows) {
          const int64_t kr = cdiv(cdiv(rows, splits), TBK) * TBK;
          const int64_t spr = cdiv(rows, kr);
          const double waves = chained ? (double)(mb * nb * spr) / cap : (double)cdiv(mb * nb * spr, cap);
          double cc = waves * (double)cdiv(kr, TBK) * stage * per_sm * smsp * tlp;
          if (spr > 1) cc += clus ? 0.05 * (double)spr * l * n : 0.3 * (double)spr * l * n + 3.6e5;
          return cc;
        };
        // chunks after the first add X into X
        double cost = (nch - 1) * chunk_cost(ch) + chunk_cost(m - (nch - 1) * ch) +
                      (nch - 1) * (0.3 * (double)l * n + 3.6e5);
        if (cost < 0.99 * best.cost) {
          best.geo = geo; best.bm = bm; best.nw = nw; best.splits = (int)sp; best.cluster = clus != 0;
          best.cost = cost; best.chunk = ch;
        }
      }
    }
  }
  return best;
}

// Omega(:, j0:j1) as a plain column-major l x (j1 - j0) block (ld l): Omega(r, j) = z_r(j) / sqrt(l)
// from the same counter layout as Gamma (R1, over the column index j of A).
__global__ void __launch_bounds__(128) k_omega_plain(uint2 key, int l, int64_t j0, int64_t j1, double scale,
                                                     double* __restrict__ out) {
  const int hp = (l + 1) / 2;
  const int64_t total = (j1 - j0) * hp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jj = e / hp;
    const int pr = (int)(e - jj * hp);
    double z0, z1;
    dev::gauss_pair((uint64_t)(j0 + jj), (uint32_t)pr, key, z0, z1);
    double* col = out + jj * l;
    col[2 * pr] = z0 * scale;
    if (2 * pr + 1 < l) col[2 * pr + 1] = z1 * scale;
  }
}

// The tensor map of a column-major m x n A (box 16 rows x 64 columns, 128-byte swizzle).
sk_status make_tmap(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, CUtensorMap* tm, int pbox) {
  const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)lda * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)TBK, (cuuint32_t)pbox};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = tmap_encoder()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, SK_E_CUDA, "cuTensorMapEncodeTiled failed for A");
  return SK_OK;
}

// The Omega image of rows [i0, i1) of A (from Philox, or packed from Q when Qom != nullptr).
template <class C>
sk_status omega_chunk_image(sk_ctx* c, uint2 key, const double* Qom, int64_t ldq, int64_t l, int64_t i0, int64_t i1,
                            double* img) {
  constexpr int BM = C::BM;
  const int64_t mb = cdiv(l, BM), KT = cdiv(i1 - i0, TBK);
  if (Qom) k_omega_pack<<<(unsigned)(mb * KT), 128, 0, c->stream>>>(Qom, ldq, (int)l, i0, i1, BM, C::OS, KT, img);
  else k_omega_image<<<(unsigned)(mb * KT), 128, 0, c->stream>>>(key, (int)l, i0, i1, BM, C::OS, KT, img);
  return launched(c);
}

// Waits (one thread, bounded) until both slot counters reach their totals: every CTA of every chained
// chunk GEMM has added its tile into X.  Launched normally after the chain, it restores plain stream
// order for what follows (the chain's image kernels do not wait for their predecessors).
__global__ void k_chain_join(const unsigned* done, unsigned need0, unsigned need1) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int s = 0; s < 2; ++s) {
    const unsigned need = s ? need1 : need0;
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + s) : "memory");
      if (v >= need) break;
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20ull * 1000 * 1000 * 1000) __trap();
      __nanosleep(256);
    }
  }
}

// One K-chunk's GEMM: X (+)= Omega(:, p.k0:p.m) A(p.k0:p.m, :) with the chunk's image, K-split
// `splits_req` ways (partials through `part` or cluster DSMEM); p.accum selects = or +=.
template <class C>
sk_status pre_gemm_chunk(sk_ctx* c, const CUtensorMap& tm, DenseParams p, int64_t l, int64_t n, int splits_req,
                         bool cl_allowed, const double* img, double* part) {
  constexpr int BM = C::BM;
  const int64_t mb = cdiv(l, BM), nb = cdiv(n, C::TBNP), KT = cdiv(p.m - p.k0, TBK);
  p.k_per_split = cdiv(cdiv(p.m - p.k0, splits_req), TBK) * TBK;
  const int splits = (int)cdiv(p.m - p.k0, p.k_per_split);
  const bool clu = cl_allowed && splits > 1 && splits <= 8 && BM % splits == 0;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)mb, (unsigned)nb, (unsigned)splits);
  lc.blockDim = dim3(C::NT);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = c->stream;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (clu) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = (unsigned)splits;
    ++na;
  }
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL behind the image kernel
  at[na].val.programmaticStreamSerializationAllowed = 1;
  ++na;
  lc.attrs = at; lc.numAttrs = na;
  if (splits == 1 || clu) {
    auto kern = clu ? k_sketch_pre<C, 2> : k_sketch_pre<C, 0>;
    SK_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
    SK_CUDA(c, cudaLaunchKernelEx(&lc, kern, tm, p, img, KT));
    return launched(c);
  }
  p.part = part;
  auto kern = k_sketch_pre<C, 1>;
  SK_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  SK_CUDA(c, cudaLaunchKernelEx(&lc, kern, tm, p, img, KT));
  SK_TRY(launched(c));
  return splitk_reduce(c, p.part, splits, l, n, p.scale, p.X, p.ldx, p.accum);
}

// X = Omega A chunk by chunk: per K-chunk, the chunk's Omega image (generated from Philox, or packed
// from a given Q when Qom != nullptr) then the TMA + DMMA GEMM accumulating into X.
template <class C>
sk_status run_pre(sk_ctx* c, const DenseParams& p0, int64_t m, int64_t n, int64_t l, const PrePlan& pl,
                  const double* Qom = nullptr, int64_t ldq = 0) {
  constexpr int BM = C::BM;
  DenseParams p = p0;
  CUtensorMap tm;
  SK_TRY(make_tmap(c, p.A, m, n, p.lda, &tm, C::PBOX));
  const int64_t mb = cdiv(l, BM);
  const int64_t chunk = pl.chunk > 0 ? pl.chunk : m;
  DBuf img, part;
  SK_TRY(img.alloc(c, (size_t)mb * cdiv(chunk, TBK) * TBK * C::OS * sizeof(double)));   // one chunk's Omega: the slot
  const int64_t kps_max = cdiv(cdiv(chunk, pl.splits), TBK) * TBK;
  const int sp_max = (int)cdiv(chunk, kps_max);
  const bool cl = pl.cluster && sp_max > 1 && sp_max <= 8 && BM % sp_max == 0;
  const int64_t nch = cdiv(m, chunk);
  // a ragged last chunk splits into fewer K ranges; when that count cannot form the cluster it goes
  // through HBM partials, so those are allocated too
  const int64_t last = m - (nch - 1) * chunk;
  const int sp_last = (int)cdiv(last, cdiv(cdiv(last, pl.splits), TBK) * TBK);
  if ((sp_max > 1 && !cl) || (sp_last > 1 && (!cl || sp_last != sp_max)))
    SK_TRY(part.alloc(c, (size_t)sp_max * l * n * sizeof(double)));
  if (nch == 1) {
    SK_TRY((omega_chunk_image<C>(c, p.key, Qom, ldq, l, 0, m, img.as<double>())));
    p.k0 = 0;
    p.m = m;
    p.accum = 0;
    return pre_gemm_chunk<C>(c, tm, p, l, n, pl.splits, cl, img.as<double>(), part.as<double>());
  }
  // Several chunks in one K range each (no split): the chunk GEMMs form ONE programmatic chain on the
  // context stream, each letting its successor be scheduled once all its CTAs are resident, so the
  // next chunk's CTAs take the SMs the last wave frees (no idle tail per chunk).  The next chunk's Omega
  // image is made inside the current GEMM by kGenCtas CTAs starting kGenAt CTAs into the grid (well
  // past the previous GEMM's tail); device counters carry the ordering the chain cannot: a GEMM waits
  // for its image's generator CTAs (ready), generators wait for the GEMM that last read their slot
  // (done) before overwriting it, k_chain_join waits for every GEMM CTA.  X is zeroed and every chunk
  // adds (red.add) its product.
  if (nch >= 3 && sp_max == 1 && sp_last == 1 && c->tune_sketch_path != 2 && c->tune_sketch_path != 3 &&
      cdiv(l, BM) * cdiv(n, C::TBNP) >= c->num_sms &&          // at least a wave per chunk (and generators)
      !(dist_on(c) && dist_view(c).exchange == 1)) {
    // (on a distributed context with the per-step exchange the chain measured slower at world size 1,
    // 784 vs 565 ms per C5 sketch -- cause not isolated; the replicate exchange, the default, gains
    // 545 -> 535 ms: profiles/round2/chain/dist_world1.txt)
    const unsigned ctas = (unsigned)(cdiv(l, BM) * cdiv(n, C::TBNP));
    DBuf img2, cnt;
    SK_TRY(img2.alloc(c, img.bytes));
    SK_TRY(cnt.alloc(c, (4 + (size_t)ctas) * sizeof(unsigned)));
    SK_CUDA(c, cudaMemsetAsync(cnt.p, 0, (4 + (size_t)ctas) * sizeof(unsigned), c->stream));
    SK_CUDA(c, cudaMemset2DAsync(p.X, p.ldx * sizeof(double), 0, n * sizeof(double), l, c->stream));
    double* slot[2] = {img.as<double>(), img2.as<double>()};
    unsigned* done = cnt.as<unsigned>();
    unsigned* ready = done + 2;
    unsigned* tile_ord = done + 4;
    const unsigned gen_n = std::min<unsigned>(ctas / 2, (unsigned)c->num_sms);
    const unsigned gen_lo = std::min<unsigned>(ctas - gen_n, 3u * (unsigned)c->num_sms);
    SK_TRY((omega_chunk_image<C>(c, p.key, Qom, ldq, l, 0, std::min(m, chunk), slot[0])));   // chunk 0's image
    for (int64_t ci = 0; ci < nch; ++ci) {
      const int64_t i0 = ci * chunk, i1 = std::min(m, i0 + chunk);
      const int s = (int)(ci & 1);
      DenseParams q = p;
      q.k0 = i0;
      q.m = i1;
      q.accum = 1;
      q.done = done + s;
      q.tile_ord = tile_ord;
      q.chunk_idx = (unsigned)ci;
      q.ready = ci >= 1 ? ready + s : nullptr;              // chunk 0's image: a plain kernel before
      q.ready_need = (unsigned)((ci + 1) / 2) * gen_n;      // generator CTAs of the chunks ci-1, ci-3, ...
      if (ci + 1 < nch) {
        const int64_t j0 = i1, j1 = std::min(m, j0 + chunk);
        q.gen_img = slot[s ^ 1];
        q.gen_q = Qom; q.gen_ldq = ldq;
        q.gen_i0 = j0; q.gen_i1 = j1; q.gen_kt = cdiv(j1 - j0, TBK);
        q.gen_lo = gen_lo; q.gen_n = gen_n;
        q.gen_gate = ci >= 1 ? done + (s ^ 1) : nullptr;    // chunk ci-1's GEMM read slot s^1
        q.gen_need = (unsigned)((ci + 1) / 2) * ctas;       // GEMMs ci-1, ci-3, ... used slot s^1
        q.gen_ready = ready + (s ^ 1);
      }
      SK_TRY(pre_gemm_chunk<C>(c, tm, q, l, n, 1, false, slot[s], nullptr));
    }
    k_chain_join<<<1, 32, 0, c->stream>>>(done, (unsigned)((nch + 1) / 2) * ctas, (unsigned)(nch / 2) * ctas);
    return launched(c);
  }
  // Several chunks: two image slots; the image of chunk c + 1 is generated on the image stream while
  // the GEMM of chunk c runs (its small CTAs fit beside a GEMM CTA on an SM), into the slot the GEMM of
  // chunk c - 1 has finished reading.  Events order slot reuse and image -> GEMM.
  DBuf img2;
  SK_TRY(img2.alloc(c, img.bytes));
  if (!c->img) SK_CUDA(c, cudaStreamCreateWithFlags(&c->img, cudaStreamNonBlocking));
  double* slot[2] = {img.as<double>(), img2.as<double>()};
  cudaEvent_t ev[5] = {};
  sk_status rs = SK_OK;
  for (int e = 0; e < 5 && rs == SK_OK; ++e)
    if (cudaEventCreateWithFlags(&ev[e], cudaEventDisableTiming) != cudaSuccess) rs = fail(c, SK_E_CUDA, "sketch: event");
  cudaEvent_t* made = ev;         // [2] image of the chunk in slot s complete (helper stream)
  cudaEvent_t* read = ev + 2;     // [2] GEMM that read slot s complete (context stream)
  if (rs == SK_OK && (cudaEventRecord(ev[4], c->stream) != cudaSuccess || cudaStreamWaitEvent(c->img, ev[4], 0) != cudaSuccess))
    rs = fail(c, SK_E_CUDA, "sketch: event");
  if (rs == SK_OK) rs = omega_chunk_image<C>(c, p.key, Qom, ldq, l, 0, std::min(m, chunk), slot[0]);
  for (int64_t ci = 0; ci < nch && rs == SK_OK; ++ci) {
    const int64_t i0 = ci * chunk, i1 = std::min(m, i0 + chunk);
    if (ci + 1 < nch) {           // next image on the helper stream, into the other slot
      const int s = (int)((ci + 1) & 1);
      cudaStream_t main_stream = c->stream;
      if (ci >= 1 && cudaStreamWaitEvent(c->img, read[s], 0) != cudaSuccess) { rs = fail(c, SK_E_CUDA, "sketch: event"); break; }
      c->stream = c->img;
      rs = omega_chunk_image<C>(c, p.key, Qom, ldq, l, i1, std::min(m, i1 + chunk), slot[s]);
      c->stream = main_stream;
      if (rs == SK_OK && cudaEventRecord(made[s], c->img) != cudaSuccess) rs = fail(c, SK_E_CUDA, "sketch: event");
      if (rs != SK_OK) break;
    }
    if (ci >= 1 && cudaStreamWaitEvent(c->stream, made[ci & 1], 0) != cudaSuccess) { rs = fail(c, SK_E_CUDA, "sketch: event"); break; }
    p.k0 = i0;
    p.m = i1;
    p.accum = ci > 0;
    const int64_t kps = cdiv(cdiv(i1 - i0, pl.splits), TBK) * TBK;
    const bool clu = cl && cdiv(i1 - i0, kps) == sp_max;
    rs = pre_gemm_chunk<C>(c, tm, p, l, n, pl.splits, clu, slot[ci & 1], part.as<double>());
    if (rs == SK_OK && cudaEventRecord(read[ci & 1], c->stream) != cudaSuccess) rs = fail(c, SK_E_CUDA, "sketch: event");
  }
  // the context stream has waited for every image, so the slots are freed after their last use
  for (int e = 0; e < 5; ++e)
    if (ev[e]) cudaEventDestroy(ev[e]);
  return rs;
}


sk_status sketch_dense_pre(sk_ctx* c, const DenseParams& p, int64_t m, int64_t n, int64_t l, const PrePlan& pl,
                           const double* Qom = nullptr, int64_t ldq = 0) {
  if (pl.bm <= 0) return fail(c, SK_E_ARG, "sketch: no tensor-core plan for this shape");
  return with_geo(pl.geo, [&](auto cfg) { return run_pre<decltype(cfg)>(c, p, m, n, l, pl, Qom, ldq); });
}

bool tma_ok_for(const double* A, int64_t m, int64_t n, int64_t lda) {
  return (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && tmap_encoder() != nullptr &&
         m < (1LL << 31) && n < (1LL << 31);
}

}  // namespace

sk_status sketch_dense(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                       uint64_t seed, double* X, int64_t ldx) {
  if (n == 0) return SK_OK;
  DenseParams p{};
  p.A = A; p.lda = lda; p.m = m; p.n = n; p.l = (int)l;
  p.key = dev::seed_key(seed);
  p.scale = 1.0 / std::sqrt((double)l);
  p.X = X; p.ldx = ldx;
  // TMA path: A 16-byte aligned with a 16-byte multiple column stride (the tensor-map rules)
  if (tma_ok_for(A, m, n, lda) && c->tune_sketch_path != 1) {
    const PrePlan pl = plan_pre(c, m, n, l);
    if (pl.bm > 0) return sketch_dense_pre(c, p, m, n, l, pl);
  }
  // fallback (A the tensor map cannot describe): each CTA generates its Omega tiles in shared memory
  const int64_t mb = cdiv(l, DBM), nb = cdiv(n, DBN);
  int splits = 1;
  while (mb * nb * splits < c->num_sms && m / (splits * 2) >= 1024 && splits < 64) splits *= 2;
  p.k_per_split = cdiv(cdiv(m, splits), DBK) * DBK;
  splits = (int)cdiv(m, p.k_per_split);
  const bool vec = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const dim3 grid((unsigned)mb, (unsigned)nb, (unsigned)splits);
  DBuf part;
  if (splits > 1) {
    SK_TRY(part.alloc(c, (size_t)splits * l * n * sizeof(double)));
    p.part = part.as<double>();
  }
  auto go = [&](auto kern) -> sk_status {
    SK_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)D_SMEM));
    kern<<<grid, DNT, D_SMEM, c->stream>>>(p);
    return launched(c);
  };
  if (splits == 1) {
    SK_TRY(vec ? go(k_sketch_dense<true, false>) : go(k_sketch_dense<false, false>));
    return SK_OK;
  }
  SK_TRY(vec ? go(k_sketch_dense<true, true>) : go(k_sketch_dense<false, true>));
  return splitk_reduce(c, p.part, splits, l, n, p.scale, X, ldx);
}


namespace {
// sums[0] = ||A - Q W||_F^2, sums[1] = ||A||_F^2 on the TMA + DMMA pipeline: rows of the output = the
// M = m rows of Q (packed once into the row-operand image), K = k, the column operand W (k x n,
// column-major) streamed by TMA, MODE 4 epilogue against A.
template <class C>
sk_status run_sumsq(sk_ctx* c, const double* Q, int64_t ldq, const double* W, int64_t ldw, const double* A, int64_t lda,
                    int64_t m, int64_t n, int64_t k, double* sums) {
  constexpr int BM = C::BM;
  CUtensorMap tm;
  SK_TRY(make_tmap(c, W, k, n, ldw, &tm, C::PBOX));
  const int64_t mb = cdiv(m, BM), nb = cdiv(n, C::TBNP), KT = cdiv(k, TBK);
  DBuf img, part;
  SK_TRY(img.alloc(c, (size_t)mb * KT * TBK * C::OS * sizeof(double)));
  SK_TRY(part.alloc(c, (size_t)2 * mb * nb * sizeof(double)));
  k_pack_rows<<<(unsigned)(mb * KT), 128, 0, c->stream>>>(Q, ldq, m, k, BM, C::OS, KT, img.as<double>());
  SK_TRY(launched(c));
  DenseParams p{};
  p.A = W; p.lda = ldw; p.m = k; p.n = n; p.l = (int)std::min<int64_t>(m, INT32_MAX);
  p.scale = 1.0; p.k0 = 0; p.k_per_split = cdiv(k, TBK) * TBK;
  p.Csub = A; p.ldcs = lda; p.sums_part = part.as<double>();
  auto kern = k_sketch_pre<C, 4>;
  SK_CUDA(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)mb, (unsigned)nb, 1);
  lc.blockDim = dim3(C::NT);
  lc.dynamicSmemBytes = C::SMEM;
  lc.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;     // PDL behind the pack kernel
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at; lc.numAttrs = 1;
  SK_CUDA(c, cudaLaunchKernelEx(&lc, kern, tm, p, (const double*)img.as<double>(), KT));
  SK_TRY(launched(c));
  return reduce_pairs(c, part.as<double>(), mb * nb, sums);
}
}  // namespace

sk_status residual_sumsq_tma(sk_ctx* c, const double* Q, int64_t ldq, const double* W, int64_t ldw, const double* A,
                             int64_t lda, int64_t m, int64_t n, int64_t k, double* sums) {
  if (!tma_ok_for(W, k, n, ldw) || m >= (1LL << 31)) return fail(c, SK_E_ARG, "residual_sumsq_tma: layout");
  // narrow n (C4's 784 = 7 x 112): the 112-column tiles fill the columns exactly where 256-column
  // tiles would leave a quarter of the last one idle
  auto fill = [&](int64_t tbn) { return (double)n / (double)(cdiv(n, tbn) * tbn); };
  if (fill(112) > fill(256) + 0.05) return run_sumsq<CfgN80>(c, Q, ldq, W, ldw, A, lda, m, n, k, sums);
  // 12-warp 48 x 384 tiles where their column fill and wave count keep up with 48 x 256 (the third
  // warp per SM sub-partition is worth ~4 %, see plan_pre)
  auto waves = [&](int64_t tbn) {
    const int64_t ctas = cdiv(m, 48) * cdiv(n, tbn);
    return (double)ctas / (double)(cdiv(ctas, c->num_sms) * c->num_sms);
  };
  if (fill(384) * waves(384) * 1.045 > fill(256) * waves(256))
    return run_sumsq<CfgT48>(c, Q, ldq, W, ldw, A, lda, m, n, k, sums);
  return run_sumsq<CfgW48>(c, Q, ldq, W, ldw, A, lda, m, n, k, sums);
}

sk_status gemm_qta(sk_ctx* c, const double* Q, int64_t ldq, const double* A, int64_t m, int64_t n, int64_t lda,
                   int64_t l, double* X, int64_t ldx) {
  if (n == 0 || l == 0) return SK_OK;
  if (!tma_ok_for(A, m, n, lda)) {   // X^T (n x l col-major, ld ldx) = A^T Q
    return gemm(c, true, false, n, l, m, 1.0, A, lda, Q, ldq, 0.0, X, ldx);
  }
  DenseParams p{};
  p.A = A; p.lda = lda; p.m = m; p.n = n; p.l = (int)l;
  p.scale = 1.0;
  p.X = X; p.ldx = ldx;
  return sketch_dense_pre(c, p, m, n, l, plan_pre(c, m, n, l), Q, ldq);
}

namespace {
// Y (m x l, ldy) (+)= A Omega(:, col0 : col0 + n)^T for the Gaussian Omega (l x n_total over A's
// columns), one pass over A: Omega is generated one block of A's columns at a time into an L2-sized
// slot and each block's product is accumulated into Y by the DMMA GEMM -- no transpose of A.
sk_status cols_sketch_gaussian(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                               uint64_t seed, double* Y, int64_t ldy, int64_t col0 = 0, bool accumulate = false) {
  const int64_t nc = std::max<int64_t>(256, std::min<int64_t>(n, (int64_t)(kOmegaSlotBytes / (8.0 * l)) / 256 * 256));
  DBuf om;
  SK_TRY(om.alloc(c, (size_t)l * std::min(nc, n) * sizeof(double)));
  const uint2 key = dev::seed_key(seed);
  const double scale = 1.0 / std::sqrt((double)l);
  for (int64_t j0 = 0; j0 < n; j0 += nc) {
    const int64_t j1 = std::min(n, j0 + nc);
    const int64_t work = (j1 - j0) * ((l + 1) / 2);
    k_omega_plain<<<(unsigned)std::min<int64_t>(cdiv(work, 128), 16LL * c->num_sms), 128, 0, c->stream>>>(
        key, (int)l, col0 + j0, col0 + j1, scale, om.as<double>());
    SK_TRY(launched(c));
    SK_TRY(gemm(c, false, true, m, l, j1 - j0, 1.0, A + j0 * lda, lda, om.as<double>(), l,
                (j0 > 0 || accumulate) ? 1.0 : 0.0, Y, ldy));
  }
  return SK_OK;
}
}  // namespace

sk_status sketch_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                      int zeta, uint64_t seed, double* Y, int64_t ldy) {
  if (emb == SK_EMB_GAUSSIAN) return cols_sketch_gaussian(c, A, m, n, lda, l, seed, Y, ldy);
  // sparse sign / SRTT: Y = A Omega^T (m x l col-major) = (Omega A^T)^T, the row sketch of A^T written
  // with row stride ldy (one transpose pass of A, then the row-sketch kernels)
  DBuf At;
  SK_TRY(At.alloc(c, (size_t)n * m * sizeof(double)));
  SK_TRY(transpose(c, A, m, n, lda, At.as<double>(), n));
  if (emb == SK_EMB_SRTT) return sketch_srtt(c, At.as<double>(), n, m, n, l, seed, Y, ldy);
  return sketch_sparse(c, At.as<double>(), n, m, n, l, zeta, seed, Y, ldy);
}

sk_status sketch_power(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                       int zeta, uint64_t seed, int q, double* X, int64_t ldx) {
  // X = Omega (A^T A)^q = ((Omega A^T) A) ... : T = Omega A^T (kept as T^T = A Omega^T, m x l), then
  // alternately X^T = A^T T^T (the TMA + DMMA sketch GEMM with Omega := T^T) and T^T = A X^T.
  DBuf Tt, Xt;
  SK_TRY(Tt.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(sketch_cols(c, A, m, n, lda, l, emb, zeta, seed, Tt.as<double>(), m));
  double* Xout = X;
  int64_t ldo = ldx;
  for (int it = 0; it < q; ++it) {
    if (it > 0) {
      SK_TRY(gemm(c, false, false, m, l, n, 1.0, A, lda, Xout, ldo, 0.0, Tt.as<double>(), m));      // T^T = A X^T
    }
    SK_TRY(gemm_qta(c, Tt.as<double>(), m, A, m, n, lda, l, Xout, ldo));                         // X = T A
  }
  return SK_OK;
}

// Algorithm 3 line 2: X = Gamma A and Y = A Omega^T "in a single pass through A".  The pass
// that matters is the one over the STREAM A arrives on: with A in host memory its column blocks cross
// PCIe once, through the ring of for_host_blocks, and each block feeds both products -- X(:, block)
// completely (the TMA + DMMA sketch of the block) and its term A_block Omega(:, block)^T of Y.  With
// A already in HBM the two products run as two full-efficiency passes (FP64-bound: an L2-blocked
// single pass was measured 1.1-3.3x slower, its partial-sum traffic exceeding A's).
sk_status sketch_dual(sk_ctx* c, const double* A, bool a_on_host, int64_t m, int64_t n, int64_t lda, int64_t lx,
                      int64_t ly, uint64_t seed_x, uint64_t seed_y, double* X, int64_t ldx, double* Y, int64_t ldy) {
  if (n == 0 || m == 0) return SK_OK;
  if (!a_on_host) {
    SK_TRY(sketch_dense(c, A, m, n, lda, lx, seed_x, X, ldx));
    return cols_sketch_gaussian(c, A, m, n, lda, ly, seed_y, Y, ldy);
  }
  return for_host_blocks(c, A, m, n, lda, [&](const double* blk, int64_t j0, int64_t jw) {
    SK_TRY(sketch_dense(c, blk, m, jw, m, lx, seed_x, X + j0, ldx));
    return cols_sketch_gaussian(c, blk, m, jw, m, ly, seed_y, Y, ldy, j0, j0 > 0);
  });
}

sk_status sketch_power_ortho(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                             int zeta, uint64_t seed, int q, double* X, int64_t ldx, int64_t* status_dev) {
  // eq:ortho_power_iter: Y1 = A Omega^T; Y_i = ortho(A ortho(A^T Y_{i-1})); X = ortho(Y_q)^T A.
  // ortho = this library's LUPP basis + CholeskyQR2 (shifted CholeskyQR3 for very tall panels).
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  DBuf Y, Q, Z, Qz;
  SK_TRY(Y.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(Q.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(sketch_cols(c, A, m, n, lda, l, emb, zeta, seed, Y.as<double>(), m));
  SK_TRY(orthonormal_basis(c, Y.as<double>(), m, l, Q.as<double>(), status_dev));
  if (q > 1) {
    SK_TRY(Z.alloc(c, (size_t)n * l * sizeof(double)));
    SK_TRY(Qz.alloc(c, (size_t)n * l * sizeof(double)));
  }
  for (int i = 2; i <= q; ++i) {
    SK_TRY(gemm_qta(c, Q.as<double>(), m, A, m, n, lda, l, Z.as<double>(), n));             // A^T Q (n x l col-major)
    SK_TRY(orthonormal_basis(c, Z.as<double>(), n, l, Qz.as<double>(), status_dev));
    SK_TRY(gemm(c, false, false, m, l, n, 1.0, A, lda, Qz.as<double>(), n, 0.0, Y.as<double>(), m));   // A ortho(.)
    SK_TRY(orthonormal_basis(c, Y.as<double>(), m, l, Q.as<double>(), status_dev));
  }
  return gemm_qta(c, Q.as<double>(), m, A, m, n, lda, l, X, ldx);                            // ortho(Y_q)^T A
}

sk_status sketch_sparse(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                        int zeta, uint64_t seed, double* X, int64_t ldx) {
  if (n == 0) return SK_OK;
  SparseParams p{};
  p.A = A; p.lda = lda; p.m = m; p.n = n; p.l = (int)l; p.zeta = zeta;
  p.key = dev::seed_key(seed);
  p.scale = 1.0 / std::sqrt((double)zeta);
  p.X = X; p.ldx = ldx;
  if (zeta <= 8 && l <= 48 * 16 && s4_smem(s4_geom(48, 16, zeta)) <= (size_t)c->max_smem_optin) {
    if (l <= 16 * 32) return l <= 8 * 32 ? launch_sparse4<8, 32>(c, p) : launch_sparse4<16, 32>(c, p);
    if (l <= 8 * 16) return launch_sparse4<8, 16>(c, p);
    if (l <= 16 * 16) return launch_sparse4<16, 16>(c, p);
    if (l <= 32 * 16) return launch_sparse4<32, 16>(c, p);
    return launch_sparse4<48, 16>(c, p);
  }
  if (s2_smem((int)l) <= (size_t)c->max_smem_optin) {
    if (l <= 7 * 16) return launch_sparse2<7, 16>(c, p);
    if (l <= 15 * 16) return launch_sparse2<15, 16>(c, p);
    if (l <= 15 * 35) return launch_sparse2<15, 35>(c, p);
  }
  const int64_t J = cdiv(l, SNW);
  if (J <= 8) return launch_sparse<8>(c, p);
  if (J <= 16) return launch_sparse<16>(c, p);
  if (J <= 32) return launch_sparse<32>(c, p);
  if (J <= 64) return launch_sparse<64>(c, p);
  if (J <= 128) return launch_sparse<128>(c, p);
  return fail(c, SK_E_ARG, "sparse sketch supports l <= 2048");
}

}  // namespace skel
