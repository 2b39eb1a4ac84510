// srtt.cu -- SRTT embedding: X = Gamma A with
//     Gamma = sqrt(m/l) Pi_{m->l} T Phi Pi_{m->m}           (Table 1)
// T the unitary discrete Hartley transform, T(k, i) = cas(2 pi i k / m) / sqrt(m).
// Readings (R18, R19): Pi_{m->m}, Pi_{m->l} are keyed Feistel bijections of the
// b = log2(m)-bit indices and Phi(i) = -1 iff bit 0 of Philox(i, 0, 0, 'SIGN') is set
// (philox.cuh); m must be a power of two.  Nothing of Gamma is stored in HBM.
//
// One CTA per column at a time (grid-stride over columns; 1 CTA per SM, shared memory bound):
//   1. y = Phi Pi x: x = A(:, j) is read coalesced and scattered into shared memory at the
//      inverse-permuted position q = Pi^{-1}(i) with sign Phi(q) (inverse permutation and signs
//      are tabulated once per CTA), packed as N = m/2 complex z_n = y_2n + i y_2n+1 in
//      bit-reversed order;
//   2. DIT FFT of length N in shared memory: radix-8 passes in registers (one table twiddle per
//      8-point group, the others by squaring and constant rotations), padded storage;
//   3. for the l selected indices k = Pi_{m->l}(r): the real-input DFT
//      Y_k = E_k + e^{-2 pi i k/m} O_k with E = (Z_k + conj Z_{N-k})/2, O = (Z_k - conj Z_{N-k})/(2i),
//      then the Hartley value H_k = Re Y_k - Im Y_k and X(r, j) = H_k / sqrt(l)
//      (sqrt(m/l) * 1/sqrt(m)).
// Work O(m log m) per column; the bound is reading A once (8mn bytes).
#include <cmath>

#include "common.cuh"
#include "internal.h"
#include "philox.cuh"

namespace skel {
namespace {

constexpr int RNT = 512;

struct SrttParams {
  const double* A; int64_t lda;
  int64_t m, n; int l; int b;     // m = 2^b
  uint2 key;
  double* X; int64_t ldx;
};

__host__ __device__ inline size_t srtt_smem(int64_t m, int l) {
  const int64_t N = m / 2;
  return (size_t)(N + N / 8 + 1) * 16 /* z, one pad slot per 8 */ + (size_t)(64 + (N / 128 + 1)) * 16 /* twiddles */ +
         (size_t)m * 2 /* inv perm */ + (size_t)((m + 31) / 32) * 4 /* sign bits */ + (size_t)l * 2 /* selection */ +
         (size_t)l * 16 + 16 /* e^{-2 pi i k/m} per selected k */;
}

// z is stored with one padding slot per 8 complex values: slot(i) = i + i / 8, so the 8 consecutive
// points of a first-pass radix-8 group (16-byte lanes 144 bytes apart) and the strided points of
// the later passes hit distinct banks.
__device__ __forceinline__ int slot(int i) { return i + (i >> 3); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One radix-2^R pass of the DIT FFT = radix-2 stages s .. s+R-1 (1-based, half distance h = 2^(s-1)),
// done in registers on groups of 2^R points z[base + q h].  Only one twiddle is looked up per
// group, w = W_{2^R h}^{pos}; the stage-(s+u) twiddles are w^(2^(R-1-u)) times the constants
// W_{2^(u+1)}^{j} (1, -i, e^{-i pi/4}, e^{-3 i pi/4}).
template <int R>
__device__ __forceinline__ void fft_pass(double2* z, int N, int s, const double2* twA, const double2* twB, int tid,
                                         int nthreads) {
  constexpr int P = 1 << R;
  const int h = 1 << (s - 1);
  const double r2 = 0.70710678118654752440;
  for (int o = tid; o < (N >> R); o += nthreads) {
    const int pos = o & (h - 1);
    const int base = (o >> (s - 1)) * (P * h) + pos;
    double2 x[P];
#pragma unroll
    for (int q = 0; q < P; ++q) x[q] = z[slot(base + q * h)];
    const int ti = pos * (N >> (s - 1 + R));                   // W_{P h}^{pos} = tw(ti), ti < N / 2
    double2 w[R];
    w[R - 1] = cmul(twA[ti & 63], twB[ti >> 6]);
#pragma unroll
    for (int u = R - 2; u >= 0; --u) w[u] = cmul(w[u + 1], w[u + 1]);
#pragma unroll
    for (int u = 0; u < R; ++u) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        if (q & (1 << u)) continue;
        const int j = q & ((1 << u) - 1);
        double2 t = w[u];
        if (u == 1 && j == 1) t = make_double2(t.y, -t.x);                                   // * (-i)
        if (u == 2 && j == 1) t = make_double2(r2 * (t.x + t.y), r2 * (t.y - t.x));          // * e^{-i pi/4}
        if (u == 2 && j == 2) t = make_double2(t.y, -t.x);                                   // * (-i)
        if (u == 2 && j == 3) t = make_double2(r2 * (t.y - t.x), -r2 * (t.x + t.y));         // * e^{-3 i pi/4}
        const double2 a = x[q], b = cmul(x[q + (1 << u)], t);
        x[q] = make_double2(a.x + b.x, a.y + b.y);
        x[q + (1 << u)] = make_double2(a.x - b.x, a.y - b.y);
      }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) z[slot(base + q * h)] = x[q];
  }
}

__device__ __forceinline__ uint32_t bitrev(uint32_t x, int bits) { return __brev(x) >> (32 - bits); }

__global__ void __launch_bounds__(RNT, 1) k_sketch_srtt(SrttParams p) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int64_t m = p.m, N = m / 2;
  const int lgN = p.b - 1;
  double2* z = reinterpret_cast<double2*>(rsm);                               // [N]
  // twiddle e^{-2 pi i t/N} = twA[t & 63] * twB[t >> 6]: two small tables, no bank-conflicting
  // strided lookups (a single table indexed by pos * (N >> s) is a 32-way conflict mid-transform)
  double2* twA = z + N + N / 8 + 1;                                            // [64]
  double2* twB = twA + 64;                                                     // [N/128 + 1]
  uint16_t* pinv = reinterpret_cast<uint16_t*>(twB + (N / 128 + 1));          // [m]   (m <= 65536)
  uint32_t* sgn = reinterpret_cast<uint32_t*>(pinv + m);                       // [m/32]
  uint16_t* sel = reinterpret_cast<uint16_t*>(sgn + (m + 31) / 32);           // [l]
  double2* selw = reinterpret_cast<double2*>(
      (reinterpret_cast<uintptr_t>(sel + p.l) + 15) & ~uintptr_t(15));          // [l]
  const int tid = threadIdx.x;
  // ---- per-CTA tables (Gamma's structure, regenerated, never in HBM)
  for (int64_t t = tid; t < 64 + N / 128 + 1; t += RNT) {
    const double ang = t < 64 ? 2.0 * (double)t / (double)N : 2.0 * (double)((t - 64) * 64) / (double)N;
    double s, c;
    dev::bm_sincospi(ang, s, c);
    twA[t] = make_double2(c, -s);                       // (twB follows twA contiguously)
  }
  for (int64_t i = tid; i < m; i += RNT) pinv[i] = (uint16_t)dev::feistel_inv((uint32_t)i, p.b, dev::kTagPerm, p.key);
  for (int64_t w = tid; w < (m + 31) / 32; w += RNT) {
    uint32_t bits = 0u;
    for (int q = 0; q < 32 && w * 32 + q < m; ++q) {
      const uint32_t i = (uint32_t)(w * 32 + q);
      bits |= (dev::philox4x32_10(make_uint4(i, 0u, 0u, dev::kTagSign), p.key).x & 1u) << q;
    }
    sgn[w] = bits;
  }
  for (int r = tid; r < p.l; r += RNT) {
    const uint32_t k = dev::feistel((uint32_t)r, p.b, dev::kTagSubs, p.key);
    sel[r] = (uint16_t)k;
    double sn, cs;
    dev::bm_sincospi(2.0 * (double)k / (double)m, sn, cs);        // e^{-2 pi i k/m} = cs - i sn
    selw[r] = make_double2(cs, sn);
  }
  __syncthreads();
  const double inv_sqrt_l = 1.0 / sqrt((double)p.l);

  // the column is held in registers (m / RNT <= 32 per thread) and the next column's loads are
  // issued before the current column's FFT, so HBM latency overlaps the transform
  constexpr int XPT = 32;
  double xv[XPT];
  auto load_col = [&](int64_t j) {
    const double* col = p.A + j * p.lda;
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int64_t i = tid + (int64_t)q * RNT;
      xv[q] = (j < p.n && i < m) ? __ldcs(col + i) : 0.0;
    }
  };
  load_col(blockIdx.x);
  for (int64_t j = blockIdx.x; j < p.n; j += gridDim.x) {
    // 1. scatter y_q = Phi(q) x_{Pi(q)} into bit-reversed complex slots
#pragma unroll
    for (int qq = 0; qq < XPT; ++qq) {
      const int64_t i = tid + (int64_t)qq * RNT;
      if (i < m) {
        const uint32_t q = pinv[i];
        const double x = xv[qq];
        const double y = ((sgn[q >> 5] >> (q & 31)) & 1u) ? -x : x;
        double* zd = reinterpret_cast<double*>(z + slot((int)bitrev(q >> 1, lgN)));
        zd[q & 1u] = y;
      }
    }
    __syncthreads();
    load_col(j + gridDim.x);
    // 2. DIT FFT of length N: radix-8 passes (3 stages each), then one radix-4 or radix-2 pass
    {
      int st = 1;
      for (; st + 2 <= lgN; st += 3) {
        fft_pass<3>(z, (int)N, st, twA, twB, tid, RNT);
        __syncthreads();
      }
      if (lgN - st + 1 == 2) { fft_pass<2>(z, (int)N, st, twA, twB, tid, RNT); __syncthreads(); }
      else if (lgN - st + 1 == 1) { fft_pass<1>(z, (int)N, st, twA, twB, tid, RNT); __syncthreads(); }
    }
    // 3. selected Hartley outputs
    for (int r = tid; r < p.l; r += RNT) {
      const int64_t k = sel[r];
      const int64_t k1 = k & (N - 1), k2 = (N - k1) & (N - 1);
      const double2 Zk = z[slot((int)k1)], Zk2 = z[slot((int)k2)];
      const double2 Zc = make_double2(Zk2.x, -Zk2.y);
      const double2 E = make_double2(0.5 * (Zk.x + Zc.x), 0.5 * (Zk.y + Zc.y));
      const double2 D = make_double2(0.5 * (Zk.x - Zc.x), 0.5 * (Zk.y - Zc.y));
      const double2 O = make_double2(D.y, -D.x);                      // D / i
      const double2 ws = selw[r];
      const double s = ws.y, c = ws.x;                                // e^{-2 pi i k/m} = c - i s
      const double yr = E.x + (O.x * c + O.y * s);
      const double yi = E.y + (O.y * c - O.x * s);
      p.X[(int64_t)r * p.ldx + j] = (yr - yi) * inv_sqrt_l;
    }
    __syncthreads();
  }
}

}  // namespace

sk_status sketch_srtt(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                      double* X, int64_t ldx) {
  if (n == 0) return SK_OK;
  int b = 0;
  while ((1ll << b) < m) ++b;
  if ((1ll << b) != m || m < 8) return fail(c, SK_E_ARG, "sk_sketch: SRTT needs m a power of two >= 8 (R19)");
  const size_t smem = srtt_smem(m, (int)l);
  if (m > 32 * RNT || smem > (size_t)c->max_smem_optin)
    return fail(c, SK_E_ARG, "sk_sketch: SRTT column transform exceeds shared memory (m <= 16384)");
  SrttParams p{};
  p.A = A; p.lda = lda; p.m = m; p.n = n; p.l = (int)l; p.b = b;
  p.key = dev::seed_key(seed);
  p.X = X; p.ldx = ldx;
  SK_CUDA(c, cudaFuncSetAttribute(k_sketch_srtt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)std::min<int64_t>(n, c->num_sms);
  k_sketch_srtt<<<grid, RNT, smem, c->stream>>>(p);
  return launched(c);
}

}  // namespace skel
