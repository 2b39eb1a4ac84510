// philox.cuh -- device-side counter-based generation of the embedding Gamma.
//
// Gamma is never stored in HBM: every kernel that needs Gamma(r, i) regenerates
// it from (seed, r, i).  Counter layout = DESIGN.md readings R1/R2 (the paper
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

// U53 (R2): u = (N + 0.5) * 2^-53 with N = (w_hi >> 5) * 2^26 + (w_lo >> 6) < 2^53,
// the sum N + 0.5 rounded to nearest-even in double.  Computed as RN(2N + 1) * 2^-54: the
// integer 2N+1 (< 2^54) is formed exactly on the integer pipe and converted once, which
// rounds identically (same real value, same 53-bit RN), and the power-of-two scale is exact.
__device__ __forceinline__ double u53(uint32_t w_hi, uint32_t w_lo) {
  const uint64_t N = ((uint64_t)(w_hi >> 5) << 26) | (uint64_t)(w_lo >> 6);
  return __dmul_rn(__ull2double_rn(2ull * N + 1ull), 1.0 / 18014398509481984.0);
}

// Standard normals z_{2p}, z_{2p+1} of column i (before the 1/sqrt(l) scale).
__device__ __forceinline__ void gauss_pair(uint64_t i, uint32_t p, uint2 key, double& z0, double& z1) {
  const uint4 w = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), p, kTagGauss), key);
  const double u1 = u53(w.x, w.y), u2 = u53(w.z, w.w);
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
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

}  // namespace dev
}  // namespace skel
