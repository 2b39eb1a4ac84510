// dmma.cuh -- FP64 tensor-core MMA and cp.async primitives (sm_100a).
//
// On sm_100a the only FP64 MMA is the warp-level mma.sync m8n8k4 (SASS DMMA.8x8x4);
// tcgen05.mma has no f64 kind.  Measured on B200 (tools/microbench):
// DMMA 37.1 TFLOP/s, DFMA 34.1 TFLOP/s, and the two share the FP64 pipe.
//
// Fragment layout of mma.m8n8k4.row.col.f64 (lane = 4*g + q):
//   A (8x4):  a  = A[g][q]
//   B (4x8):  b  = B[q][g]
//   C (8x8):  c0 = C[g][2q], c1 = C[g][2q+1]
#pragma once
#include <cstdint>

namespace skel {
namespace dev {

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy global->shared; src_bytes = 0 zero-fills.
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(valid ? 8 : 0));
}
// 16-byte async copy (L2-only caching); src_bytes in {0, 8, 16}.
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(sdst)), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace dev
}  // namespace skel
