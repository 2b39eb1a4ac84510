// Time the 64-wide diagonal Cholesky/inverse kernel alone (k_diag_inv<MODE>), back-to-back launches.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2104_05877_b200/csrc \
//        -o /tmp/diag_inv_bench tools/microbench/diag_inv_bench.cu -L paper_2104_05877_b200 -lskel -lcublas
#include "../../paper_2104_05877_b200/csrc/dense.cu"
#include <vector>

__global__ void k_empty(int* x) { if (threadIdx.x == 1023) x[0] = 1; }
__global__ void k_empty_smem(int* x) {
  extern __shared__ int esm[];
  if (threadIdx.x == 1023) { esm[0] = 1; x[0] = esm[0]; }
}

int main() {
  const int n = 64;
  std::vector<double> h(n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[i + j * n] = (i == j ? n : 0.0) + 1.0 / (1.0 + i + j);   // SPD
  double *G, *G0, *W; int64_t* st;
  cudaMalloc(&G, n * n * 8); cudaMalloc(&G0, n * n * 8); cudaMalloc(&W, n * n * 8); cudaMalloc(&st, 8);
  cudaMemcpy(G0, h.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemset(st, 0, 8);
  cudaFuncSetAttribute(skel::k_diag_inv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)skel::kDiagInvSmem);
  cudaFuncSetAttribute(skel::k_diag_inv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)skel::kDiagInvSmem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      const int N = 200;
      cudaEventRecord(a);
      for (int it = 0; it < N; ++it) {
        cudaMemcpyAsync(G, G0, n * n * 8, cudaMemcpyDeviceToDevice);
        if (mode == 0) skel::k_diag_inv<0><<<1, 256, skel::kDiagInvSmem>>>(G, n, n, W, n, 0, st);
        else skel::k_diag_inv<1><<<1, 256, skel::kDiagInvSmem>>>(G, n, n, W, n, 0, nullptr);
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      cudaEventRecord(a);
      for (int it = 0; it < N; ++it) cudaMemcpyAsync(G, G0, n * n * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms0; cudaEventElapsedTime(&ms0, a, b);
      printf("k_diag_inv<%d>: %.2f us per launch (copy-only loop %.2f us per iteration) err=%s\n", mode,
             1e3 * (ms - ms0) / N, 1e3 * ms0 / N, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // launch overhead: empty 1-CTA and 128-CTA kernels, with and without 72 KB of dynamic smem
  {
    int* d; cudaMalloc(&d, 4);
    cudaFuncSetAttribute(k_empty_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int cfg = 0; cfg < 6; ++cfg) {
      const int grid = cfg % 2 ? 128 : 1;
      const size_t sm = cfg < 2 ? 0 : cfg < 4 ? 72 * 1024 : 200 * 1024;
      const int N = 500;
      cudaEventRecord(a);
      for (int it = 0; it < N; ++it) {
        if (sm) k_empty_smem<<<grid, 256, sm>>>(d); else k_empty<<<grid, 256>>>(d);
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("empty kernel grid=%d smem=%zu KB: %.2f us per launch\n", grid, sm / 1024, 1e3 * ms / N);
    }
  }
  // k_right_tri_mul<true>: X (4096 x 64) <- X W^T in place
  {
    const int rows = 4096;
    double* X; cudaMalloc(&X, (size_t)rows * n * 8); cudaMemset(X, 0, (size_t)rows * n * 8);
    cudaFuncSetAttribute(skel::k_right_tri_mul<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)skel::kRtmSmem);
    for (int rep = 0; rep < 2; ++rep) {
      const int N = 200;
      cudaEventRecord(a);
      for (int it = 0; it < N; ++it)
        skel::k_right_tri_mul<true><<<(rows + 63) / 64, 256, skel::kRtmSmem>>>(X, rows, rows, W, n, n);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("k_right_tri_mul<true> rows=%d jb=64: %.2f us per launch err=%s\n", rows, 1e3 * ms / N,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
