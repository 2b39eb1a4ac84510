// Latency of a cluster all-to-all "mailbox" exchange: every CTA of a cluster st.async's a
// message of B 16-byte chunks into every CTA's double-buffered mailbox (completing bytes on the
// receiver's mbarrier) and waits for all CS messages -- the per-pivot exchange of the LUPP panel.
// Also: 2-CTA ping-pong of one 16-byte message (one-way latency = half the round trip).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mailbox_lat mailbox_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void st_async(unsigned ra, unsigned long long x, unsigned long long y, unsigned rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra), "l"(x),
               "l"(y), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void arm(unsigned b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(unsigned b, unsigned par) {
  unsigned done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(b), "r"(par)
                 : "memory");
  } while (!done);
}

template <int CHUNKS>
__global__ void k_alltoall(int steps, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned cs = cl.num_blocks(), rank = cl.block_rank();
  __shared__ __align__(16) unsigned long long box[2][16][CHUNKS * 2];
  __shared__ __align__(8) unsigned long long bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl.sync();
  long long t0 = clock64();
  unsigned long long acc = 0;
  for (int s = 0; s < steps; ++s) {
    const int par = s & 1;
    if (threadIdx.x == 0) arm(smem_u32(&bar[par]), cs * CHUNKS * 16);
    // warp w sends to CTAs w, w+8; lane j sends chunk j
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (unsigned d = w; d < cs; d += blockDim.x >> 5)
      for (int j = lane; j < CHUNKS; j += 32)
        st_async(mapa(smem_u32(&box[par][rank][2 * j]), d), acc + s, rank, mapa(smem_u32(&bar[par]), d));
    wait(smem_u32(&bar[par]), (s >> 1) & 1);
    acc += box[par][(rank + 1) % cs][0];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) {
    out[0] = (t1 - t0) / steps;
    out[1] = (long long)acc;
  }
  cl.sync();
}

__global__ void k_pingpong(int steps, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  __shared__ __align__(16) unsigned long long box[2][2];
  __shared__ __align__(8) unsigned long long bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cl.sync();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int s = 0; s < steps; ++s) {
      const int par = s & 1;
      arm(smem_u32(&bar[par]), 16);
      if (rank == 0) {
        st_async(mapa(smem_u32(&box[par][0]), 1), s, 0, mapa(smem_u32(&bar[par]), 1));
        wait(smem_u32(&bar[par]), (s >> 1) & 1);
      } else {
        wait(smem_u32(&bar[par]), (s >> 1) & 1);
        st_async(mapa(smem_u32(&box[par][0]), 0), s, 0, mapa(smem_u32(&bar[par]), 0));
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[2] = (t1 - t0) / steps;
  __syncthreads();
  cl.sync();
}

template <int CHUNKS>
void run(int cs, long long* d, long long* h) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(cs);
  lc.blockDim = dim3(256);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  lc.attrs = at; lc.numAttrs = 1;
  cudaFuncSetAttribute(k_alltoall<CHUNKS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchKernelEx(&lc, k_alltoall<CHUNKS>, 2000, d);
  cudaMemcpy(h, d, 3 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("all-to-all cluster %2d, %2d x 16 B per message: %lld cyc/step (%.3f us @1.965GHz)  [%s]\n", cs, CHUNKS, h[0],
         h[0] / 1965.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long *d, h[3];
  cudaMalloc(&d, 3 * sizeof(long long));
  for (int cs : {2, 4, 8, 16}) {
    run<1>(cs, d, h);
    run<34>(cs, d, h);
  }
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(2);
  lc.blockDim = dim3(32);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  lc.attrs = at; lc.numAttrs = 1;
  cudaLaunchKernelEx(&lc, k_pingpong, 2000, d);
  cudaMemcpy(h, d, 3 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("ping-pong round trip (2 CTAs, 16 B): %lld cyc (%.3f us)  [%s]\n", h[2], h[2] / 1965.0,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
