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
// Work O(m log m) per column; the bound is reading A once (8mn bytes).  This path holds m <= 16384
// (one column's transform in one CTA's shared memory); larger m (to 131072) take the four-step
// cluster kernel k_sketch_srtt_big below.
#include <cooperative_groups.h>

#include <cmath>

#include "common.cuh"
#include "internal.h"
#include "philox.cuh"

namespace skel {
namespace {

namespace cg = cooperative_groups;
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

// output row r takes transform index k = Pi_{m->l}(r) (the Feistel bijection on b bits)
__global__ void k_srtt_select(uint32_t* sel, int l, int b, uint2 key) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < l) sel[r] = dev::feistel((uint32_t)r, b, dev::kTagSubs, key);
}

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

// ------------------------------------------------------------------ m > 16384: four-step, one cluster per column
// N = m/2 = N1 N2 with N2 = 8192 (the shared-memory transform) and N1 = N / N2 <= 8 (the cluster):
//   Z_kappa = sum_{n1} W_N^{n1 kappa} FFT_{N2}( z_{n1 + N1 n2} )[kappa mod N2]
// (n = n1 + N1 n2, kappa = kappa2 + N2 kappa1, W_N^{n1 kappa2} W_{N1}^{n1 kappa1} = W_N^{n1 kappa}).  CTA
// n1 of the cluster gathers its N2 complex inputs z_n = y_{2n} + i y_{2n+1}, y_q = Phi(q) x_{Pi(q)},
// through a per-call table of (Pi(q), sign), transforms them, and turns each selected output r into
// its partial Hartley value (a real-linear function of Z_k, Z_{N-k}, so the N1 partials add); the
// partials meet in distributed shared memory and are summed in rank order (deterministic).
// The table is laid out in the order of the bit-reversed FFT slots (entry 2s + parity holds input
// n2 = bitrev(s)), so a warp's shared-memory stores hit consecutive slots (conflict-free) and its
// table loads are coalesced; the column's gathered values for the next column are in flight in
// registers during the current column's transform.
constexpr int BN2 = 8192, BLG2 = 13, BXPT = 2 * BN2 / RNT;   // 32 inputs per thread

struct SrttBigParams {
  const double* A; int64_t lda;
  int64_t m, n; int l; int N1;
  const uint32_t* gl;     // [N1][2 N2]: Pi(q) | sign << 31, entry 2 s + par <-> q = 2 (n1 + N1 bitrev(s)) + par
  const uint32_t* selk;   // [l] transform index k of output row r
  double* X; int64_t ldx;
};

// W_m^t = e^{-2 pi i t/m} (t < m) as tA[t & 511] * tB[t >> 9]: 512 + m/512 (<= 256) entries
__host__ __device__ inline size_t srtt_big_smem(int l) {
  return (size_t)(BN2 + BN2 / 8 + 1) * 16 + (size_t)(64 + BN2 / 128 + 1) * 16 + (size_t)(512 + 256) * 16 +
         (size_t)l * (8 + 4) + 64;
}

__global__ void k_srtt_table(uint32_t* gl, int64_t m, int b, int N1, uint2 key) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n1 = e / (2 * BN2), rem = e - n1 * 2 * BN2;
    const int64_t n2 = bitrev((uint32_t)(rem >> 1), BLG2), par = rem & 1;
    const uint32_t q = (uint32_t)(2 * (n1 + N1 * n2) + par);
    const uint32_t i = dev::feistel(q, b, dev::kTagPerm, key);
    const uint32_t sg = dev::philox4x32_10(make_uint4(q, 0u, 0u, dev::kTagSign), key).x & 1u;
    gl[e] = i | (sg << 31);
  }
}

__global__ void __launch_bounds__(RNT, 1) k_sketch_srtt_big(SrttBigParams p) {
  extern __shared__ __align__(16) unsigned char rsm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int n1 = (int)cluster.block_rank(), N1 = p.N1;
  const int64_t m = p.m, N = m / 2;
  double2* z = reinterpret_cast<double2*>(rsm);                                // [BN2] (+pad)
  double2* twA = z + BN2 + BN2 / 8 + 1;                                        // [64]
  double2* twB = twA + 64;                                                     // [BN2/128 + 1]
  double2* tA = twB + (BN2 / 128 + 1);                                          // [512]: W_m^t, t < 512
  double2* tB = tA + 512;                                                      // [m/512]: W_m^{512 t}
  double* part = reinterpret_cast<double*>(tB + 256);                          // [l]: this CTA's partial outputs
  uint32_t* sel = reinterpret_cast<uint32_t*>(part + p.l);                     // [l]
  const int tid = threadIdx.x;
  for (int t = tid; t < 64 + BN2 / 128 + 1; t += RNT) {
    const double ang = t < 64 ? 2.0 * (double)t / (double)BN2 : 2.0 * (double)((t - 64) * 64) / (double)BN2;
    double sn, cs;
    dev::bm_sincospi(ang, sn, cs);
    twA[t] = make_double2(cs, -sn);
  }
  for (int64_t t = tid; t < 512 + m / 512; t += RNT) {
    const double ang = t < 512 ? 2.0 * (double)t / (double)m : 2.0 * (double)((t - 512) * 512) / (double)m;
    double sn, cs;
    dev::bm_sincospi(ang, sn, cs);
    tA[t] = make_double2(cs, -sn);                                             // (tB follows tA contiguously)
  }
  for (int r = tid; r < p.l; r += RNT) sel[r] = p.selk[r];
  __syncthreads();
  auto wm = [&](int64_t t) { return cmul(tA[t & 511], tB[t >> 9]); };       // W_m^t, 0 <= t < m
  const double inv_sqrt_l = 1.0 / sqrt((double)p.l);
  const uint32_t* gln = p.gl + (int64_t)n1 * 2 * BN2;
  double xv[BXPT];
  uint32_t sg = 0u;
  auto load_col = [&](int64_t j) {
    if (j >= p.n) return;
    const double* col = p.A + j * p.lda;
    uint32_t t[BXPT];
#pragma unroll
    for (int q = 0; q < BXPT; ++q) t[q] = __ldg(gln + tid + q * RNT);
    sg = 0u;
#pragma unroll
    for (int q = 0; q < BXPT; ++q) {
      xv[q] = col[t[q] & 0x7fffffffu];
      sg |= (t[q] >> 31) << q;
    }
  };
  load_col(blockIdx.y);
  for (int64_t j = blockIdx.y; j < p.n; j += gridDim.y) {
    // 1. y_q into the bit-reversed complex slots (entry e = tid + q RNT -> slot e / 2, part e & 1)
#pragma unroll
    for (int q = 0; q < BXPT; ++q) {
      const int e = tid + q * RNT;
      const double x = xv[q];
      reinterpret_cast<double*>(z + slot(e >> 1))[e & 1] = ((sg >> q) & 1u) ? -x : x;
    }
    __syncthreads();
    load_col(j + gridDim.y);
    // 2. DIT FFT of length BN2 = 2^13: four radix-8 passes + one radix-2
    {
      int st = 1;
      for (; st + 2 <= BLG2; st += 3) {
        fft_pass<3>(z, BN2, st, twA, twB, tid, RNT);
        __syncthreads();
      }
      if (BLG2 - st + 1 == 2) { fft_pass<2>(z, BN2, st, twA, twB, tid, RNT); __syncthreads(); }
      else if (BLG2 - st + 1 == 1) { fft_pass<1>(z, BN2, st, twA, twB, tid, RNT); __syncthreads(); }
    }
    // 3. partial Hartley outputs: Z_kappa's share W_N^{n1 kappa} FFT[kappa mod N2], W_N^t = W_m^{2t}
    for (int r = tid; r < p.l; r += RNT) {
      const int64_t k = sel[r];
      const int64_t k1 = k & (N - 1), k2 = (N - k1) & (N - 1);
      const double2 Zk = cmul(wm((2 * n1 * k1) & (m - 1)), z[slot((int)(k1 & (BN2 - 1)))]);
      const double2 Zk2 = cmul(wm((2 * n1 * k2) & (m - 1)), z[slot((int)(k2 & (BN2 - 1)))]);
      const double2 Zc = make_double2(Zk2.x, -Zk2.y);
      const double2 E = make_double2(0.5 * (Zk.x + Zc.x), 0.5 * (Zk.y + Zc.y));
      const double2 D = make_double2(0.5 * (Zk.x - Zc.x), 0.5 * (Zk.y - Zc.y));
      const double2 O = make_double2(D.y, -D.x);
      const double2 ws = wm(k);                                 // e^{-2 pi i k/m} = cw - i sw
      const double cw = ws.x, sw = -ws.y;
      const double yr = E.x + (O.x * cw + O.y * sw);
      const double yi = E.y + (O.y * cw - O.x * sw);
      part[r] = (yr - yi) * inv_sqrt_l;
    }
    cluster.sync();                                           // every CTA's partials are in place
    for (int r = n1 + N1 * tid; r < p.l; r += N1 * RNT) {       // rows r = n1 (mod N1): sum in rank order
      double s = 0.0;
      for (int q = 0; q < N1; ++q) s += cluster.map_shared_rank(part, q)[r];
      p.X[(int64_t)r * p.ldx + j] = s;
    }
    cluster.sync();                                           // partials and z free for the next column
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
  if (m > 32 * RNT || smem > (size_t)c->max_smem_optin) {
    // m > 16384: four-step transform, one cluster of N1 = m / 16384 CTAs per column (N1 <= 8)
    const int N1 = (int)(m / (2 * BN2));
    const size_t bsm = srtt_big_smem((int)l);
    if (N1 < 1 || N1 > 8 || N1 * 2 * BN2 != m || bsm > (size_t)c->max_smem_optin)
      return fail(c, SK_E_ARG, "sk_sketch: SRTT supports m a power of two <= 131072 (and l <= 5800 beyond m = 16384)");
    DBuf gl, sel;
    SK_TRY(gl.alloc(c, (size_t)m * sizeof(uint32_t)));
    SK_TRY(sel.alloc(c, (size_t)l * sizeof(uint32_t)));
    const uint2 key = dev::seed_key(seed);
    k_srtt_table<<<(unsigned)std::min<int64_t>(cdiv(m, 256), 4LL * c->num_sms), 256, 0, c->stream>>>(
        gl.as<uint32_t>(), m, b, N1, key);
    SK_TRY(launched(c));
    k_srtt_select<<<(unsigned)cdiv(l, 256), 256, 0, c->stream>>>(sel.as<uint32_t>(), (int)l, b, key);
    SK_TRY(launched(c));
    SrttBigParams q{};
    q.A = A; q.lda = lda; q.m = m; q.n = n; q.l = (int)l; q.N1 = N1;
    q.gl = gl.as<uint32_t>(); q.selk = sel.as<uint32_t>(); q.X = X; q.ldx = ldx;
    SK_CUDA(c, cudaFuncSetAttribute(k_sketch_srtt_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    cudaLaunchConfig_t lc{};
    lc.blockDim = dim3(RNT);
    lc.dynamicSmemBytes = bsm;
    lc.stream = c->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)N1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    // every cluster loops over columns, so the grid is exactly the clusters that are co-resident
    // (a second wave would start only when the first has finished all of its columns)
    lc.gridDim = dim3((unsigned)N1, (unsigned)std::max(1, c->num_sms / N1), 1);
    int resident = 0;
    SK_CUDA(c, cudaOccupancyMaxActiveClusters(&resident, k_sketch_srtt_big, &lc));
    lc.gridDim.y = (unsigned)std::min<int64_t>(n, std::max(1, resident));
    SK_CUDA(c, cudaLaunchKernelEx(&lc, k_sketch_srtt_big, q));
    return launched(c);
  }
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
