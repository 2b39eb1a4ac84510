// common.cuh -- context, errors, stream-ordered workspace, small device helpers.
// Part of libskel.so (see include/skel.h).  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/skel.h"

#ifndef __CUDA_ARCH_LIST__
#endif

namespace skel { struct DistState; }

struct sk_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;
  int num_sms = 148;
  int max_smem_optin = 0;
  std::string err;
  int64_t launches = 0;
  int64_t ws_hwm = 0;       // high-water mark of pooled bytes
  // pinned host scratch for small device->host results (info, scalars)
  void* host_scratch = nullptr;
  // dense-sketch tuning (sk_set_sketch_tuning; 0 = automatic): path 1 = the fallback kernel that
  // generates Omega tiles in shared memory; row-tile height, warps (x 32 columns), K-splits per chunk,
  // rows per K-chunk
  int tune_sketch_path = 0, tune_sketch_bm = 0, tune_sketch_nw = 0, tune_sketch_splits = 0;
  int64_t tune_sketch_chunk = 0;
  // lowest-priority helper stream + events for look-ahead overlap (LUPP trailing updates)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // helper stream of the K-chunked dense sketch (next chunk's Omega image beside the current GEMM);
  // separate from aux, which carries the host -> device copies of the host-A ring
  cudaStream_t img = nullptr;
  // column-sharded (distributed) context, sk_create_dist: this rank's block of A's columns and the
  // library-owned NCCL communicator (dist.cu); nullptr for a single-GPU context
  skel::DistState* dist = nullptr;
  // launches made while set carry programmatic stream serialization (PDL): the kernel may start
  // while its predecessor drains; every such kernel calls griddep_wait() before touching memory
  bool pdl = false;
};

namespace skel {

constexpr int kMaxDevices = 64;   // per-device caches of function attributes / library handles

// ---- status helpers --------------------------------------------------------
inline sk_status fail(sk_ctx* c, sk_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

#define SK_CUDA(ctx, expr)                                                          \
  do {                                                                             \
    cudaError_t e__ = (expr);                                                      \
    if (e__ != cudaSuccess)                                                        \
      return ::skel::fail((ctx), SK_E_CUDA,                                        \
                          std::string(#expr " -> ") + cudaGetErrorString(e__));    \
  } while (0)

#define SK_TRY(expr)                    \
  do {                                  \
    sk_status s__ = (expr);             \
    if (s__ != SK_OK) return s__;       \
  } while (0)

#define SK_ARG(ctx, cond, msg)                                         \
  do {                                                                \
    if (!(cond)) return ::skel::fail((ctx), SK_E_ARG, (msg));         \
  } while (0)

// Count of kernels launched through a context (reported by the bench).
inline sk_status launched(sk_ctx* c, int n = 1) {
  c->launches += n;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, SK_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  return SK_OK;
}

// ---- stream-ordered device buffers from the context's pool -------------------
// cudaMallocFromPoolAsync with release threshold = max: after warm-up no call
// reaches the OS allocator; buffers are freed in stream order when they go out
// of scope, so a later call on the same stream can reuse them.
struct DBuf {
  sk_ctx* c = nullptr;
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, c->stream);
    p = nullptr;
  }
  sk_status alloc(sk_ctx* ctx, size_t n) {
    release();
    c = ctx;
    bytes = n ? n : 16;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, ctx->pool, ctx->stream);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return fail(ctx, SK_E_NOMEM, std::string("workspace: ") + cudaGetErrorString(e));
    }
    return SK_OK;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch with programmatic stream serialization (PDL): the kernel may be scheduled while its
// predecessor in the stream drains; it must call dev::griddep_wait() before touching memory.
template <typename... KArgs, typename... Args>
inline sk_status launch_pdl(sk_ctx* c, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&lc, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) return fail(c, SK_E_CUDA, std::string("launch: ") + cudaGetErrorString(e));
  return launched(c);
}

}  // namespace skel

// ---- device helpers ---------------------------------------------------------
namespace skel {
namespace dev {

// Candidate for "argmax |v|, ties to the lowest index", with the runner-up magnitude.
struct Cand {
  double a1;    // best magnitude (or -1 if none)
  double a2;    // second best magnitude (or -1)
  long long i1; // index of the best (LLONG_MAX if none)
};

// PDL: block until the preceding grid in the stream has completed and its memory is visible (a
// no-op when the launch was not programmatic).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// PDL: let the next grid in the stream be scheduled (once every CTA of this grid has called it or exited)
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ Cand cand_none() { return Cand{-1.0, -1.0, 0x7fffffffffffffffLL}; }

__device__ __forceinline__ bool beats(double a, long long ia, double b, long long ib) {
  return a > b || (a == b && ia < ib);
}

__device__ __forceinline__ Cand cand_merge(const Cand& x, const Cand& y) {
  Cand r;
  if (beats(x.a1, x.i1, y.a1, y.i1)) {
    r.a1 = x.a1; r.i1 = x.i1; r.a2 = fmax(x.a2, y.a1);
  } else {
    r.a1 = y.a1; r.i1 = y.i1; r.a2 = fmax(y.a2, x.a1);
  }
  return r;
}

__device__ __forceinline__ Cand cand_shfl_xor(const Cand& c, int o) {
  Cand r;
  r.a1 = __shfl_xor_sync(0xffffffffu, c.a1, o);
  r.a2 = __shfl_xor_sync(0xffffffffu, c.a2, o);
  r.i1 = __shfl_xor_sync(0xffffffffu, c.i1, o);
  return r;
}

__device__ __forceinline__ Cand warp_cand_reduce(Cand c) {
#pragma unroll
  for (int o = 16; o; o >>= 1) c = cand_merge(c, cand_shfl_xor(c, o));
  return c;
}

// Block-wide candidate reduction; every thread gets the result. `sh` >= 32 Cands.
__device__ __forceinline__ Cand block_cand_reduce(Cand c, Cand* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  c = warp_cand_reduce(c);
  if (lane == 0) sh[w] = c;
  __syncthreads();
  if (w == 0) {
    Cand d = lane < nw ? sh[lane] : cand_none();
    d = warp_cand_reduce(d);
    if (lane == 0) sh[32] = d;
  }
  __syncthreads();
  Cand r = sh[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum in a fixed order (deterministic). `sh` >= 33 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (w == 0) {
    double d = lane < nw ? sh[lane] : 0.0;
    d = warp_sum(d);
    if (lane == 0) sh[32] = d;
  }
  __syncthreads();
  double r = sh[32];
  __syncthreads();
  return r;
}

// Nanosecond wall clock (bounded spin waits).
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

}  // namespace dev
}  // namespace skel
