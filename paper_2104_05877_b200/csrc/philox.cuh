// philox.cuh -- device-side counter-based generation of the embedding Gamma.
//
// Gamma is never held in HBM as a whole: every kernel that needs Gamma(r, i) regenerates it from
// (seed, r, i) -- the dense sketch one K-chunk at a time into an L2-sized slot (sketch.cu).  Counter layout = DESIGN.md readings R1/R2 (the paper
// only fixes the distributions, P:176 Gaussian N(0,1/l), P:182 sparse sign):
//   Gaussian pair p of column i:  Philox4x32-10(ctr = (i lo, i hi, p, 'GAUS'), key = seed)
//       u1 = U53(w0, w1), u2 = U53(w2, w3);  z_{2p} = r cos(2 pi u2), z_{2p+1} = r sin(2 pi u2),
//       r = sqrt(-2 ln u1)  (Box-Muller).  Gamma(r, i) = z_r / sqrt(l).
//   Sparse sign, column i, call c: Philox4x32-10(ctr = (i lo, i hi, c, 'SPAR'), key = seed)
//       rows by Floyd's subset sampling from words 0..zeta-1 (word j = call j/4, lane j%4),
//       signs from the bits of call ceil(zeta/4) + j/128, word (j/32)%4, bit j%32.
#pragma once
#include <cstdint>

namespace skel {
namespace dev {

constexpr uint32_t kTagGauss = 0x47415553u;   // "GAUS"
constexpr uint32_t kTagSparse = 0x53504152u;  // "SPAR"
constexpr uint32_t kTagPerm = 0x5045524Du;    // "PERM"  SRTT Pi_{m->m}
constexpr uint32_t kTagSubs = 0x53554253u;    // "SUBS"  SRTT Pi_{m->l}
constexpr uint32_t kTagSign = 0x5349474Eu;    // "SIGN"  SRTT Phi

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

__host__ __device__ __forceinline__ uint2 seed_key(uint64_t seed) {
  return make_uint2((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
}

// U53 (R2): u = RN(N + 0.5) * 2^-53 with N = (w_hi >> 5) * 2^26 + (w_lo >> 6) < 2^53.
// Built without an int->double conversion (the conversion unit is slow next to the DMMA-bound
// sketch): for N < 2^52, N + 0.5 is exact and equals as_double(0x4330...0 + N) - (2^52 - 0.5);
// for N >= 2^52 the spacing is 1 and round-half-even gives K = N + (N & 1) (even, <= 2^53),
// = 2 * (as_double(0x4330...0 + K/2) - 2^52).  Every DADD/DMUL below is exact.
__device__ __forceinline__ double u53(uint32_t w_hi, uint32_t w_lo) {
  const uint64_t N = ((uint64_t)(w_hi >> 5) << 26) | (uint64_t)(w_lo >> 6);
  const bool big = (N >> 52) != 0;
  const uint64_t K = big ? (N + (N & 1ull)) >> 1 : N;
  const double off = big ? 4503599627370496.0 : 4503599627370495.5;
  const double scale = big ? 1.0 / 4503599627370496.0 : 1.0 / 9007199254740992.0;
  return __dmul_rn(__dsub_rn(__longlong_as_double((long long)(0x4330000000000000ull + K)), off), scale);
}

// ---- branch-free FP64 elementary functions for Box-Muller -------------------------------
// CUDA's log / sqrt / sincospi contain divergent slow paths (BSSY/BSYNC regions), which keeps
// the compiler from interleaving independent Box-Muller chains; the sketch's producer warps
// run several chains per thread, so these straight-line versions (restated textbook
// algorithms, accurate to a few ulp on the ranges used) are what lets them overlap.

// log(u) for u in [2^-54, 1] (normal, positive): fdlibm's reduction u = 2^e m,
// m in (sqrt2/2, sqrt2], f = m - 1, s = f / (2 + f), log m = 2 atanh s with the
// Remez polynomial R(s^2) of fdlibm's e_log.c (|error| < 2^-58.45 on the reduced range).
__device__ __forceinline__ double bm_log(double u) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(u);
  int e = (int)(bits >> 52) - 1023;
  double m = __longlong_as_double((long long)((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
  const bool big = m > 1.4142135623730951;
  m = big ? 0.5 * m : m;
  e = big ? e + 1 : e;
  const double f = m - 1.0;                       // exact
  const double d = 2.0 + f;
  float rf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rf) : "f"((float)d));
  double r = (double)rf;                          // 1/d to ~2^-23, then two Newton steps
  r = fma(r, fma(-d, r, 1.0), r);
  r = fma(r, fma(-d, r, 1.0), r);
  double sq = f * r;
  sq = fma(fma(-d, sq, f), r, sq);                // s = f / d to ~0.5 ulp
  const double z = sq * sq, w = z * z;
  const double t1 = w * (3.999999999940941908e-01 + w * (2.222219843214978396e-01 + w * 1.531383769920937332e-01));
  const double t2 = z * (6.666666666666735130e-01 +
                         w * (2.857142874366239149e-01 + w * (1.818357216161805012e-01 + w * 1.479819860511658591e-01)));
  const double R = t2 + t1;
  const double hfsq = 0.5 * f * f;
  const double de = (double)e;
  return de * 6.93147180369123816490e-01 - ((hfsq - (sq * (hfsq + R) + de * 1.90821492927058770002e-10)) - f);
}

// sqrt(x) for x in [0, 80]: float rsqrt seed, two Newton steps, one Markstein correction.
__device__ __forceinline__ double bm_sqrt(double x) {
  const double xs = fmax(x, 1e-300);
  float yf;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"((float)xs));
  double y = (double)yf;
  y = fma(0.5 * y, fma(-xs * y, y, 1.0), y);
  y = fma(0.5 * y, fma(-xs * y, y, 1.0), y);
  double s = xs * y;
  s = fma(0.5 * y, fma(-s, s, xs), s);
  return x > 0.0 ? s : 0.0;
}

// sin(pi t), cos(pi t) for t in [0, 2]: t = n/2 + r exactly (|r| <= 1/4), x = pi r with a
// two-term pi, Taylor polynomials of sin to x^17 and cos to x^16 (truncation < 1e-17 for
// |x| <= pi/4), quadrant n mod 4 by selects.
__device__ __forceinline__ void bm_sincospi(double t, double& sn, double& cs) {
  const double n = rint(2.0 * t);
  const double r = fma(n, -0.5, t);               // exact
  const double x = fma(r, 3.141592653589793116, r * 1.2246467991473532e-16);
  const double z = x * x;
  double ps = 2.8114572543455206e-15;             // 1/17!
  ps = fma(z, ps, -7.6471637318198164e-13);       // -1/15!
  ps = fma(z, ps, 1.6059043836821613e-10);        // 1/13!
  ps = fma(z, ps, -2.5052108385441720e-08);       // -1/11!
  ps = fma(z, ps, 2.7557319223985893e-06);        // 1/9!
  ps = fma(z, ps, -1.9841269841269841e-04);       // -1/7!
  ps = fma(z, ps, 8.3333333333333332e-03);        // 1/5!
  ps = fma(z, ps, -1.6666666666666666e-01);       // -1/3!
  const double s = fma(x * z, ps, x);
  double pc = 4.7794773323873853e-14;             // 1/16!
  pc = fma(z, pc, -1.1470745597729725e-11);       // -1/14!
  pc = fma(z, pc, 2.0876756987868100e-09);        // 1/12!
  pc = fma(z, pc, -2.7557319223985888e-07);       // -1/10!
  pc = fma(z, pc, 2.4801587301587302e-05);        // 1/8!
  pc = fma(z, pc, -1.3888888888888889e-03);       // -1/6!
  pc = fma(z, pc, 4.1666666666666664e-02);        // 1/4!
  pc = fma(z, pc, -0.5);                          // -1/2!
  const double c = fma(z, pc, 1.0);
  const int q = (int)n & 3;                       // quadrant: (s, c) -> (c, -s) -> (-s, -c) -> (-c, s)
  const bool odd = (q & 1) != 0;
  const double a = odd ? c : s, b = odd ? s : c;
  const unsigned long long sa = (unsigned long long)(q & 2) << 62, sb = (unsigned long long)((q + 1) & 2) << 62;
  sn = __longlong_as_double(__double_as_longlong(a) ^ (long long)sa);
  cs = __longlong_as_double(__double_as_longlong(b) ^ (long long)sb);
}

// Standard normals z_{2p}, z_{2p+1} of column i (before the 1/sqrt(l) scale), Box-Muller (R2).
__device__ __forceinline__ void gauss_pair(uint64_t i, uint32_t p, uint2 key, double& z0, double& z1) {
  const uint4 w = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), p, kTagGauss), key);
  const double u1 = u53(w.x, w.y), u2 = u53(w.z, w.w);
  const double rad = bm_sqrt(-2.0 * bm_log(u1));
  double s, c;
  bm_sincospi(2.0 * u2, s, c);
  z0 = rad * c;
  z1 = rad * s;
}

// Rows (distinct, in [0,l)) of the zeta nonzeros of column i, in draw order j = 0..zeta-1,
// and their sign bits (bit j set = negative).  zeta <= 64.
__device__ __forceinline__ uint64_t sparse_col(uint64_t i, int l, int zeta, uint2 key, int* rows) {
  const uint32_t ilo = (uint32_t)i, ihi = (uint32_t)(i >> 32);
  const int nrc = (zeta + 3) >> 2;
  const uint4 sw = philox4x32_10(make_uint4(ilo, ihi, (uint32_t)nrc, kTagSparse), key);
  uint4 w = make_uint4(0, 0, 0, 0);
  for (int j = 0; j < zeta; ++j) {
    if ((j & 3) == 0) w = philox4x32_10(make_uint4(ilo, ihi, (uint32_t)(j >> 2), kTagSparse), key);
    const uint32_t word = (j & 3) == 0 ? w.x : (j & 3) == 1 ? w.y : (j & 3) == 2 ? w.z : w.w;
    const uint32_t nrange = (uint32_t)(l - zeta + j + 1);
    int t = (int)(((uint64_t)word * nrange) >> 32);
    bool taken = false;
    for (int q = 0; q < j; ++q) taken |= (rows[q] == t);
    if (taken) t = (int)nrange - 1;
    rows[j] = t;
  }
  return (uint64_t)sw.x | ((uint64_t)sw.y << 32);   // bit j of word (j/32) -> bit j
}

// SRTT (R18): keyed 4-round Feistel bijection of [0, 2^b); round r XORs one half with
// the first Philox word of (other half, r, 0, tag).  feistel_inv runs the rounds backwards.
__device__ __forceinline__ uint32_t feistel(uint32_t x, int b, uint32_t tag, uint2 key) {
  const int hb = b >> 1, lb = b - hb;
  uint32_t lo = x & ((1u << lb) - 1u), hi = x >> lb;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if ((r & 1) == 0) hi ^= philox4x32_10(make_uint4(lo, (uint32_t)r, 0u, tag), key).x & ((1u << hb) - 1u);
    else lo ^= philox4x32_10(make_uint4(hi, (uint32_t)r, 0u, tag), key).x & ((1u << lb) - 1u);
  }
  return (hi << lb) | lo;
}
__device__ __forceinline__ uint32_t feistel_inv(uint32_t x, int b, uint32_t tag, uint2 key) {
  const int hb = b >> 1, lb = b - hb;
  uint32_t lo = x & ((1u << lb) - 1u), hi = x >> lb;
#pragma unroll
  for (int r = 3; r >= 0; --r) {
    if ((r & 1) == 0) hi ^= philox4x32_10(make_uint4(lo, (uint32_t)r, 0u, tag), key).x & ((1u << hb) - 1u);
    else lo ^= philox4x32_10(make_uint4(hi, (uint32_t)r, 0u, tag), key).x & ((1u << lb) - 1u);
  }
  return (hi << lb) | lo;
}

// Register-resident variant of sparse_col for zeta <= 8 (identical draws; unrolled so rows[]
// stays in registers).
__device__ __forceinline__ uint64_t sparse_col8(uint64_t i, int l, int zeta, uint2 key, int (&rows)[8]) {
  const uint32_t ilo = (uint32_t)i, ihi = (uint32_t)(i >> 32);
  const int nrc = (zeta + 3) >> 2;
  const uint4 sw = philox4x32_10(make_uint4(ilo, ihi, (uint32_t)nrc, kTagSparse), key);
  const uint4 w0 = philox4x32_10(make_uint4(ilo, ihi, 0u, kTagSparse), key);
  const uint4 w1 = zeta > 4 ? philox4x32_10(make_uint4(ilo, ihi, 1u, kTagSparse), key) : make_uint4(0, 0, 0, 0);
  const uint32_t words[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    rows[j] = -1;
    if (j < zeta) {
      const uint32_t nrange = (uint32_t)(l - zeta + j + 1);
      int t = (int)(((uint64_t)words[j] * nrange) >> 32);
      bool taken = false;
#pragma unroll
      for (int q = 0; q < j; ++q) taken |= (rows[q] == t);
      rows[j] = taken ? (int)nrange - 1 : t;
    }
  }
  return (uint64_t)sw.x | ((uint64_t)sw.y << 32);
}

}  // namespace dev
}  // namespace skel
