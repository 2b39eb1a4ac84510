// Microbenchmarks that fix the B200 FP64 roofline denominators used in DESIGN.md:
//   (1) DMMA (mma.sync m8n8k4 f64) throughput, (2) DFMA throughput,
//   (3) DMMA + DFMA interleaved (are they separate pipes?),
//   (4) Box-Muller (FP64 log + sqrt + sincospi) throughput,
//   (5) flag-based grid-barrier latency for a persistent 148-CTA kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NACC>
__global__ void k_dmma(double* out, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(c[i][0], c[i][1], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dfma(double* out, int iters, double a, double b) {
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// interleave: per iteration 8 DMMA (2048 FMA / warp) and NF DFMA per thread (32*NF FMA / warp)
template <int NF>
__global__ void k_mixed(double* out, int iters, double a, double b) {
  double c[8][2];
  double f[NF];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < NF; ++i) f[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
#pragma unroll
    for (int i = 0; i < NF; ++i) f[i] = fma(f[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_boxmuller(double* out, int iters) {
  double s = 0;
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t y = x ^ (x >> 13);
    double u1 = ((double)(x >> 5) * 67108864.0 + (double)(y >> 6) + 0.5) * (1.0 / 9007199254740992.0);
    double u2 = ((double)(y >> 5) * 67108864.0 + (double)(x >> 6) + 0.5) * (1.0 / 9007199254740992.0);
    double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    s += r * cs + r * sn;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Flag-based grid barrier: each CTA publishes (value, step) then waits for all.
__global__ void k_gridbar(unsigned long long* flags, double* vals, int steps, double* out) {
  const int G = gridDim.x;
  __shared__ double best;
  double acc = 0;
  for (int t = 1; t <= steps; ++t) {
    if (threadIdx.x == 0) {
      vals[blockIdx.x] = (double)((blockIdx.x * 7919 + t) % 1009);
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(flags + blockIdx.x * 16), "l"((unsigned long long)t) : "memory");
    }
    double v = -1;
    for (int j = threadIdx.x; j < G; j += blockDim.x) {
      unsigned long long f;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(flags + j * 16) : "memory");
      } while (f < (unsigned long long)t);
      v = fmax(v, vals[j]);
    }
    // block max
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffff, v, o));
    __shared__ double wm[32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = -1;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, wm[w]);
      best = m;
    }
    __syncthreads();
    acc += best;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs %d, clock %d kHz\n", nsm, clk);
  double* out;
  CK(cudaMalloc(&out, 1 << 26));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int threads = 256;
  for (int occ : {1, 2, 4}) {
    int blocks = nsm * occ;
    int iters = 4000;
    k_dmma<8><<<blocks, threads>>>(out, 10, 1.0, 1.0);
    cudaEventRecord(e0);
    k_dmma<8><<<blocks, threads>>>(out, iters, 1.0000001, 0.9999999);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * 8 * iters * (threads / 32) * (double)blocks;
    printf("DMMA  occ %d: %.2f TFLOP/s (%.3f ms)\n", occ, flops / ms / 1e9, ms);
    k_dfma<8><<<blocks, threads>>>(out, 10, 1.0, 1.0);
    cudaEventRecord(e0);
    k_dfma<8><<<blocks, threads>>>(out, iters * 8, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 8 * iters * 8 * threads * (double)blocks;
    printf("DFMA  occ %d: %.2f TFLOP/s (%.3f ms)\n", occ, flops / ms / 1e9, ms);
  }
  {
    int blocks = nsm * 2, iters = 4000;
    // DMMA-only reference at same shape
    cudaEventRecord(e0);
    k_mixed<1><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed 8 DMMA + 1 DFMA/iter : %.3f ms\n", ms);
    cudaEventRecord(e0);
    k_mixed<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed 8 DMMA + 8 DFMA/iter : %.3f ms\n", ms);
    cudaEventRecord(e0);
    k_mixed<32><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed 8 DMMA + 32 DFMA/iter: %.3f ms\n", ms);
    cudaEventRecord(e0);
    k_mixed<64><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed 8 DMMA + 64 DFMA/iter: %.3f ms\n", ms);
  }
  {
    int blocks = nsm * 4, iters = 2000;
    k_boxmuller<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    k_boxmuller<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double pairs = (double)iters * threads * blocks;
    printf("Box-Muller: %.2f Gpairs/s => %.1f pairs/clk/SM\n", pairs / ms / 1e6,
           pairs / (ms * 1e-3) / nsm / (clk * 1e3));
  }
  for (int G : {32, 74, 148}) {
    unsigned long long* flags; double* vals;
    CK(cudaMalloc(&flags, 148 * 16 * 8)); CK(cudaMemset(flags, 0, 148 * 16 * 8));
    CK(cudaMalloc(&vals, 148 * 8));
    int steps = 2000;
    k_gridbar<<<G, 256>>>(flags, vals, 10, out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemset(flags, 0, 148 * 16 * 8));
    cudaEventRecord(e0);
    k_gridbar<<<G, 256>>>(flags, vals, steps, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("grid barrier G=%d: %.3f us/step\n", G, ms * 1e3 / steps);
    cudaFree(flags); cudaFree(vals);
  }
  return 0;
}
