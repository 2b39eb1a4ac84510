// Latency of the one-warp 32 x 32 Cholesky variants of k_potrf_cluster's D phase (dense.cu), and of
// the surrounding global load / store of the block, measured with clock64 in one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chol32_bench chol32_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int CB = 32, LS = CB + 1;
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  // one fourth-order step: e = 1 - d y^2, y' = y (1 + e/2 + 3e^2/8 + 5e^3/16), relative error ~e^4
  const double e = fma(-d * y, y, 1.0);
  const double p = fma(e, fma(0.3125, e, 0.375), 0.5);
  return fma(y * e, p, y);
}

// column T of the register Cholesky (template recursion: every register index is a literal, so the
// row never falls back to local memory)
template <int T>
struct Chol32Col {
  static __device__ __forceinline__ void run(double (&r)[CB], double* colbuf, int lane, int& bad) {
    double d = __shfl_sync(0xffffffffu, r[T], T);    // the pivot A(T, T), held by lane T
    if (!(d > 0.0)) {
      if (!bad) bad = T + 1;
      d = 1.0;
    }
    const double rs = rsqrt_nr(d);
    const double lit = lane == T ? d * rs : (lane > T ? r[T] * rs : 0.0);
    r[T] = lit;
    colbuf[(T & 1) * CB + lane] = lit;                 // column T of L, broadcast through shared memory
    __syncwarp();                                      // (double-buffered: no second barrier per column)
    double cj[CB];
#pragma unroll
    for (int j = T + 1; j < CB; ++j) cj[j] = colbuf[(T & 1) * CB + j];
    // unpredicated: lanes above the diagonal update entries that are never read (lit = 0 for lanes < T)
#pragma unroll
    for (int j = T + 1; j < CB; ++j) r[j] = fma(-lit, cj[j], r[j]);
    Chol32Col<T + 1>::run(r, colbuf, lane, bad);
  }
};
template <>
struct Chol32Col<CB> {
  static __device__ __forceinline__ void run(double (&)[CB], double*, int, int&) {}
};

// one warp: Cholesky of a 32 x 32 block held row-per-lane in registers (r[j] = A(lane, j), j <= lane),
// in place (r = row `lane` of L); colbuf: 64 doubles of shared scratch.  Returns the 1-based failing
// column (a failed pivot continues with 1 so no NaN spreads), 0 if none.
__device__ __forceinline__ int chol32_regs(double (&r)[CB], double* colbuf, int lane) {
  int bad = 0;
  Chol32Col<0>::run(r, colbuf, lane, bad);
  return bad;
}

// the same factorization with the block in shared memory (row `lane` per lane, stride LS): no register
// array, the per-column update predicated over an unrolled column loop.
__device__ __forceinline__ int chol32_smem(double* Ls, int lane) {
  int bad = 0;
#pragma unroll 1
  for (int t = 0; t < CB; ++t) {
    double d = Ls[t * LS + t];
    if (!(d > 0.0)) {
      if (!bad) bad = t + 1;
      d = 1.0;
    }
    const double rs = rsqrt_nr(d);
    const double lit = lane == t ? d * rs : (lane > t ? Ls[lane * LS + t] * rs : 0.0);
    __syncwarp();
    if (lane >= t) Ls[lane * LS + t] = lit;
    __syncwarp();
    // all loads first, then the FMAs, then the stores (loads cannot pass possibly-aliasing stores)
    double colv[CB], rowv[CB];
#pragma unroll
    for (int jj = 1; jj < CB; ++jj) {
      colv[jj] = Ls[jj * LS + t];
      rowv[jj] = Ls[lane * LS + jj];
    }
#pragma unroll
    for (int jj = 1; jj < CB; ++jj)
      if (jj > t && jj <= lane) Ls[lane * LS + jj] = fma(-lit, colv[jj], rowv[jj]);
  }
  __syncwarp();
  return bad;
}

__global__ void kbench(double* G, int64_t ld, int iters, long long* out) {
  __shared__ double Ls[CB * LS], cb[2 * CB];
  const int lane = threadIdx.x;
  long long tl = 0, tr = 0, ts = 0, tst = 0;
  int bad = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    double r[CB];
#pragma unroll
    for (int j = 0; j < CB; ++j) r[j] = j <= lane ? __ldcg(G + lane + (int64_t)j * ld) : 0.0;
    __syncwarp();
    long long t1 = clock64();
    double r2[CB];
#pragma unroll
    for (int j = 0; j < CB; ++j) { r2[j] = r[j]; Ls[lane * LS + j] = r[j]; }
    bad += chol32_regs(r2, cb, lane);
    __syncwarp();
    long long t2 = clock64();
    bad += chol32_smem(Ls, lane);
    long long t3 = clock64();
#pragma unroll
    for (int j = 0; j < CB; ++j) G[lane + (int64_t)j * ld + 64 * ld] = r2[j] + Ls[lane * LS + j];
    __threadfence();
    long long t4 = clock64();
    tl += t1 - t0; tr += t2 - t1; ts += t3 - t2; tst += t4 - t3;
  }
  if (lane == 0) { out[0] = tl / iters; out[1] = tr / iters; out[2] = ts / iters; out[3] = tst / iters; out[4] = bad; }
}

int main() {
  const int n = 128;
  double h[n * n];
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i + j * n] = (i == j ? 64.0 : 0.0) + 1.0 / (1.0 + i + j);
  double* G; long long* o; long long ho[5];
  cudaMalloc(&G, sizeof(h)); cudaMalloc(&o, sizeof(ho));
  cudaMemcpy(G, h, sizeof(h), cudaMemcpyHostToDevice);
  kbench<<<1, 32>>>(G, n, 10, o);
  kbench<<<1, 32>>>(G, n, 100, o);
  cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("one warp, cycles: load 32x32 (L2) %lld | chol32_regs %lld | chol32_smem %lld | store+fence %lld | bad %lld\n",
         ho[0], ho[1], ho[2], ho[3], ho[4]);
  return 0;
}
