// rng_probe.cu -- TEST-ONLY probe library (tests/librngprobe.so).
// Exposes (1) cuRAND's device Philox4x32-10 (an independent implementation, the KAT for the
// library's generator) and (2) the library's own device generators from csrc/philox.cuh, so
// the tests can compare them with the oracle element by element.
#include <cuda_runtime.h>
#include <curand_kernel.h>
#include <cstdint>

#include "../../paper_2104_05877_b200/csrc/philox.cuh"

namespace {
__global__ void k_curand(const uint32_t* in, uint32_t* out, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t* v = in + 6 * t;
  uint4 r = curand_Philox4x32_10(make_uint4(v[0], v[1], v[2], v[3]), make_uint2(v[4], v[5]));
  out[4 * t] = r.x; out[4 * t + 1] = r.y; out[4 * t + 2] = r.z; out[4 * t + 3] = r.w;
}
__global__ void k_skel(const uint32_t* in, uint32_t* out, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t* v = in + 6 * t;
  uint4 r = skel::dev::philox4x32_10(make_uint4(v[0], v[1], v[2], v[3]), make_uint2(v[4], v[5]));
  out[4 * t] = r.x; out[4 * t + 1] = r.y; out[4 * t + 2] = r.z; out[4 * t + 3] = r.w;
}
__global__ void k_gauss(uint64_t seed, int l, int64_t m, double* z) {   // z: l x m row-major (unscaled)
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int np = (l + 1) / 2;
  if (e >= (int64_t)np * m) return;
  const int p = (int)(e / m);
  const int64_t i = e % m;
  double z0, z1;
  skel::dev::gauss_pair((uint64_t)i, (uint32_t)p, skel::dev::seed_key(seed), z0, z1);
  z[(int64_t)(2 * p) * m + i] = z0;
  if (2 * p + 1 < l) z[(int64_t)(2 * p + 1) * m + i] = z1;
}
__global__ void k_sparse(uint64_t seed, int l, int64_t m, int zeta, int* rows, unsigned long long* sbits) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  int r[64];
  sbits[i] = skel::dev::sparse_col((uint64_t)i, l, zeta, skel::dev::seed_key(seed), r);
  for (int j = 0; j < zeta; ++j) rows[i * zeta + j] = r[j];
}
}  // namespace

extern "C" {
int probe_philox(int which, const uint32_t* in_host, uint32_t* out_host, int n) {
  uint32_t *din, *dout;
  cudaMalloc(&din, 24 * n);
  cudaMalloc(&dout, 16 * n);
  cudaMemcpy(din, in_host, 24 * n, cudaMemcpyHostToDevice);
  if (which == 0) k_curand<<<(n + 127) / 128, 128>>>(din, dout, n);
  else k_skel<<<(n + 127) / 128, 128>>>(din, dout, n);
  cudaMemcpy(out_host, dout, 16 * n, cudaMemcpyDeviceToHost);
  cudaFree(din); cudaFree(dout);
  return (int)cudaGetLastError();
}
int probe_gauss(uint64_t seed, int l, int64_t m, double* z_host) {
  double* d;
  cudaMalloc(&d, sizeof(double) * l * m);
  const int64_t tot = (int64_t)((l + 1) / 2) * m;
  k_gauss<<<(unsigned)((tot + 255) / 256), 256>>>(seed, l, m, d);
  cudaMemcpy(z_host, d, sizeof(double) * l * m, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)cudaGetLastError();
}
int probe_sparse(uint64_t seed, int l, int64_t m, int zeta, int* rows_host, unsigned long long* sbits_host) {
  int* dr; unsigned long long* ds;
  cudaMalloc(&dr, sizeof(int) * m * zeta);
  cudaMalloc(&ds, sizeof(unsigned long long) * m);
  k_sparse<<<(unsigned)((m + 127) / 128), 128>>>(seed, l, m, zeta, dr, ds);
  cudaMemcpy(rows_host, dr, sizeof(int) * m * zeta, cudaMemcpyDeviceToHost);
  cudaMemcpy(sbits_host, ds, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost);
  cudaFree(dr); cudaFree(ds);
  return (int)cudaGetLastError();
}
}
