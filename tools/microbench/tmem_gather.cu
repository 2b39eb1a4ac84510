// Microbenchmark: warp-uniform random 8-byte gathers from tensor memory (tcgen05.ld 32x32b.x2,
// lane = column of an A tile) vs from shared memory (LDS.64, lane = column, padded stride 257).
// This is the inner operation of the sparse-sign sketch (X(r, j) += +-A(i, j) for a warp-uniform i).
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_gather tmem_gather.cu && ./tmem_gather
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NT = 512, ITERS = 4096, G = 16;   // loads per wait

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(NT, 1) k_tmem(double* out, long long* cyc, int mode) {
  __shared__ uint32_t taddr_s;
  extern __shared__ double sm[];                 // [32][257] for the LDS variant
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  for (int e = tid; e < 32 * 257; e += NT) sm[e] = (double)(e % 97) * 0.5;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16);
  // fill: every warp of a quadrant writes all 512 columns of its lanes (values = lane + col)
  if (warp < 4) {
    for (int c = 0; c < 512; c += 2) {
      const double v = (double)(lane + c);
      const uint32_t lo = (uint32_t)__double_as_longlong(v), hi = (uint32_t)(__double_as_longlong(v) >> 32);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(base + c), "r"(lo), "r"(hi));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  uint32_t x = 12345u + warp * 7919u;
  const long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < ITERS; ++it) {
      uint32_t r[2 * G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t col = ((x + (uint32_t)g * 97u) & 255u) * 2;   // warp-uniform, 0..510
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                     : "=r"(r[2 * g]), "=r"(r[2 * g + 1]) : "r"(base + col));
      }
      x += 776u;
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int g = 0; g < G; g += 4) {
        acc0 += __hiloint2double((int)r[2 * g + 1], (int)r[2 * g]);
        acc1 += __hiloint2double((int)r[2 * g + 3], (int)r[2 * g + 2]);
        acc2 += __hiloint2double((int)r[2 * g + 5], (int)r[2 * g + 4]);
        acc3 += __hiloint2double((int)r[2 * g + 7], (int)r[2 * g + 6]);
      }
    }
  } else {
    const char* At = reinterpret_cast<const char*>(sm + lane * 257);
    for (int it = 0; it < ITERS; ++it) {
      double v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t i = (x + (uint32_t)g * 97u) & 255u;
        v[g] = *reinterpret_cast<const volatile double*>(At + 8 * i);
      }
      x += 776u;
#pragma unroll
      for (int g = 0; g < G; g += 4) { acc0 += v[g]; acc1 += v[g + 1]; acc2 += v[g + 2]; acc3 += v[g + 3]; }
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(taddr_s));
  out[blockIdx.x * NT + tid] = acc0 + acc1 + acc2 + acc3;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * NT);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  const size_t smem = 32 * 257 * 8;
  cudaFuncSetAttribute(k_tmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k_tmem<<<sms, NT, smem>>>(out, cyc, mode);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
      const double loads = (double)NT / 32 * ITERS * G;                 // warp-loads per SM
      printf("%s: %.3f ms, %lld cycles/SM, %.3f cycles per warp-load (8 B x 32 lanes), %.1f B/clk/SM\n",
             mode == 0 ? "tmem tcgen05.ld 32x32b.x2" : "smem LDS.64          ", ms, c0, c0 / loads,
             loads * 256.0 / c0);
    }
  }
  return 0;
}
