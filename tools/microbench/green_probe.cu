// Feasibility probe: can a 16-CTA thread-block cluster run in a green-context SM partition while a
// long kernel occupies the rest of the GPU?  (Would let the LUPP panel start on the first sketch rows.)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o green_probe green_probe.cu -lcuda
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x)                                                                                  \
  do {                                                                                         \
    CUresult r_ = (x);                                                                         \
    if (r_ != CUDA_SUCCESS) {                                                                  \
      const char* s_ = nullptr;                                                                \
      cuGetErrorString(r_, &s_);                                                               \
      std::printf("FAIL %s: %s (line %d)\n", #x, s_ ? s_ : "?", __LINE__);                     \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)
#define RK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      std::printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__);            \
      std::exit(1);                                                                            \
    }                                                                                          \
  } while (0)

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

// every CTA spins for `ns`; records min start / max end and the SMs it ran on
__global__ void k_spin(unsigned long long ns, unsigned long long* t, unsigned* sms) {
  const unsigned long long t0 = gtime();
  while (gtime() - t0 < ns) {
  }
  if (threadIdx.x == 0) {
    atomicMin(&t[0], t0);
    atomicMax(&t[1], gtime());
    atomicOr(&sms[smid() / 32], 1u << (smid() % 32));
  }
}

// a cluster of 16 CTAs: one cluster barrier, then spin
__global__ void __cluster_dims__(16, 1, 1) k_cluster(unsigned long long ns, unsigned long long* t, unsigned* sms) {
  cg::this_cluster().sync();
  const unsigned long long t0 = gtime();
  while (gtime() - t0 < ns) {
  }
  cg::this_cluster().sync();
  if (threadIdx.x == 0) {
    atomicMin(&t[0], t0);
    atomicMax(&t[1], gtime());
    atomicOr(&sms[smid() / 32], 1u << (smid() % 32));
  }
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  RK(cudaSetDevice(0));
  RK(cudaFree(0));  // primary context
  CUcontext prim;
  CK(cuCtxGetCurrent(&prim));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  std::printf("device SMs: %u\n", all.sm.smCount);
  for (unsigned flags : {0u, (unsigned)CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE}) {
    for (unsigned minc : {16u, 24u, 32u}) {
      CUdevResource grp[1], rest;
      unsigned nb = 1;
      CUresult r = cuDevSmResourceSplitByCount(grp, &nb, &all, &rest, flags, minc);
      std::printf("split flags=%u minCount=%u -> r=%d groups=%u group SMs=%u rest SMs=%u\n", flags, minc, (int)r, nb,
                  nb ? grp[0].sm.smCount : 0, rest.sm.smCount);
    }
  }
  CUdevResource grp[1], rest;
  unsigned nb = 1;
  CK(cuDevSmResourceSplitByCount(grp, &nb, &all, &rest, CU_DEV_SM_RESOURCE_SPLIT_MAX_POTENTIAL_CLUSTER_SIZE, 16));
  CUdevResourceDesc dl, ds;
  CK(cuDevResourceGenerateDesc(&dl, &grp[0], 1));
  CK(cuDevResourceGenerateDesc(&ds, &rest, 1));
  CUgreenCtx gl, gs;
  CK(cuGreenCtxCreate(&gl, dl, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CK(cuGreenCtxCreate(&gs, ds, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sl, ss;
  CK(cuGreenCtxStreamCreate(&sl, gl, CU_STREAM_NON_BLOCKING, 0));
  CK(cuGreenCtxStreamCreate(&ss, gs, CU_STREAM_NON_BLOCKING, 0));
  CUcontext cl, cs;
  CK(cuCtxFromGreenCtx(&cl, gl));
  CK(cuCtxFromGreenCtx(&cs, gs));

  unsigned long long* t;
  unsigned* sms;
  RK(cudaMalloc(&t, 4 * sizeof(unsigned long long)));
  RK(cudaMalloc(&sms, 16 * sizeof(unsigned)));
  unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  RK(cudaMemcpy(t, init, sizeof(init), cudaMemcpyHostToDevice));
  RK(cudaMemset(sms, 0, 16 * sizeof(unsigned)));

  // occupancy of the cluster kernel in each partition (16-CTA clusters are non-portable: opt in per context)
  for (int which = 0; which < 2; ++which) {
    CK(cuCtxSetCurrent(which ? cs : cl));
    RK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(16);
    lc.blockDim = dim3(256);
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_cluster, &lc);
    std::printf("%s partition: max active 16-CTA clusters = %d (%s)\n", which ? "sketch" : "lupp", ncl,
                cudaGetErrorString(e));
  }
  // long spin in the big partition (4 CTAs per SM of it, 200 ms), cluster kernel in the small one
  CK(cuCtxSetCurrent(cs));
  k_spin<<<rest.sm.smCount * 4, 256, 0, (cudaStream_t)ss>>>(200000000ull, t, sms);
  RK(cudaGetLastError());
  CK(cuCtxSetCurrent(cl));
  k_cluster<<<16, 256, 0, (cudaStream_t)sl>>>(20000000ull, t + 2, sms + 8);
  RK(cudaGetLastError());
  CK(cuCtxSetCurrent(prim));
  RK(cudaDeviceSynchronize());
  unsigned long long h[4];
  unsigned hs[16];
  RK(cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost));
  RK(cudaMemcpy(hs, sms, sizeof(hs), cudaMemcpyDeviceToHost));
  const unsigned long long base = h[0] < h[2] ? h[0] : h[2];
  std::printf("spin (big partition):   start %.3f ms end %.3f ms\n", (h[0] - base) * 1e-6, (h[1] - base) * 1e-6);
  std::printf("cluster (small part.):  start %.3f ms end %.3f ms  -> %s\n", (h[2] - base) * 1e-6, (h[3] - base) * 1e-6,
              h[2] < h[1] ? "CONCURRENT" : "serialised");
  int nspin = 0, ncl = 0, both = 0;
  for (int w = 0; w < 8; ++w) {
    nspin += __builtin_popcount(hs[w]);
    ncl += __builtin_popcount(hs[8 + w]);
    both += __builtin_popcount(hs[w] & hs[8 + w]);
  }
  std::printf("SMs used: spin %d, cluster %d, overlap %d\n", nspin, ncl, both);
  return 0;
}
