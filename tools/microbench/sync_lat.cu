// Latency of the exchange primitives available to the LUPP pivot chain on B200:
//   cluster.sync() for cluster sizes 2..16, DSMEM remote load, and a flag-based
//   grid barrier (LL-style flag+value words, no fences) over G CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_lat sync_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void k_cluster_sync(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}

// barrier.cluster arrive(relaxed)+wait only by warp 0 after __syncthreads -- the cheapest form
__global__ void k_cluster_sync_w0(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x < 32) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}

__global__ void k_dsmem_lat(int iters, long long* out) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 64; i += blockDim.x) buf[i] = i;
  cl.sync();
  const int peer = (cl.block_rank() + cl.num_blocks() / 2) % cl.num_blocks();
  double* rp = cl.map_shared_rank(buf, peer);
  double acc = 0;
  int idx = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { acc += rp[idx]; idx = ((int)acc) & 31; }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && cl.block_rank() == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)acc; }
}

// Each CTA publishes {value, step} packed in 2x u64 via one 16-byte st.relaxed? Use two LL words.
__global__ void k_grid_ll(unsigned long long* slots, int steps, long long* out) {
  const int G = gridDim.x;
  __shared__ unsigned long long best;
  long long t0 = clock64();
  for (int t = 1; t <= steps; ++t) {
    if (threadIdx.x == 0) {
      unsigned int v = (blockIdx.x * 7919u + t) % 1009u;
      unsigned long long w = ((unsigned long long)t << 32) | v;
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(slots + blockIdx.x * 8 + (t & 1) * G * 8), "l"(w) : "memory");
    }
    unsigned long long m = 0;
    if (threadIdx.x < 32) {
      for (int j = threadIdx.x; j < G; j += 32) {
        unsigned long long w;
        do {
          asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(slots + j * 8 + (t & 1) * G * 8) : "memory");
        } while ((w >> 32) < (unsigned long long)t);
        m = max(m, w & 0xffffffffull);
      }
      for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (threadIdx.x == 0) best = m;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = (t1 - t0) / steps; out[1] = best; }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  long long* d; cudaMalloc(&d, 64);
  long long h[2];
  cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_cluster_sync_w0, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_dsmem_lat, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) {
    for (int nt : {128, 512}) {
      cudaLaunchConfig_t lc{}; lc.gridDim = dim3(cs); lc.blockDim = dim3(nt);
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.attrs = at; lc.numAttrs = 1;
      cudaLaunchKernelEx(&lc, k_cluster_sync, 2000, d); cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      long long a = h[0];
      long long b = -1;   // barrier.cluster needs every thread of the cluster (k_cluster_sync_w0 deadlocks)
      cudaLaunchKernelEx(&lc, k_dsmem_lat, 2000, d); cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("cluster %2d threads %3d: cluster.sync %lld cyc, warp0-barrier+2xsyncthreads %lld cyc, DSMEM load %lld cyc (%s)\n",
             cs, nt, a, b, h[0], cudaGetErrorString(e));
    }
  }
  for (int G : {16, 32, 74, 148}) {
    unsigned long long* slots; cudaMalloc(&slots, 2 * 148 * 64); cudaMemset(slots, 0, 2 * 148 * 64);
    k_grid_ll<<<G, 128>>>(slots, 4000, d); cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("LL grid exchange G=%3d: %lld cyc/step (%.2f us @1.965GHz)\n", G, h[0], h[0] / 1965.0);
    cudaFree(slots);
  }
  return 0;
}
