// estimates.cu -- Algorithm 3's sketch-only ID / CUR estimates:
//     C^+ A  ~  X_1^+ X          (X_1 = X(:, J_s), the column pivots of the row sketch)
//     A R^+  ~  Y Y_1^+          (Y_1 = Y(I_s, :), the row pivots of the column sketch)
//     CUR    ~  C S^{-1} R       (S = A(I_s, J_s), C = A(:, J_s), R = A(I_s, :))
// computed without revisiting A beyond the skeletons ("compromise on accuracy and stability",
// P:431-440).  All three are the same operation, D B1 (B1^T B1)^{-1} = D (B1^+)^T:
//     (X_1^+ X)^T = X^T X_1 (X_1^T X_1)^{-1}     B1 = X_1 (lx x k),     D = X^T (n x lx)
//     Y Y_1^+     = Y Y_1^T (Y_1 Y_1^T)^{-1}     B1 = Y_1^T (ly x k),   D = Y (m x ly)
//     C S^{-1}    = C S^T (S S^T)^{-1}           B1 = S^T (k x k),      D = C (m x k)
// evaluated through the row LUPP of B1 (B1 = Lf U, |Lf| <= 1, Lf's pivot block unit lower): the
// Gram matrix that is factored is Lf^T Lf, which is well conditioned even when B1 is not, so
//     D (B1^+)^T = D Lf (Lf^T Lf)^{-1} U^{-T} = ((D Lf) L_G^{-T}) L_G^{-1} U^{-T},  Lf^T Lf = L_G L_G^T
// (three right triangular solves).  This is the same conditioning device as the residual's basis
// (residual.cu); the oracle uses a library least-squares solve.
#include "common.cuh"
#include "internal.h"

namespace skel {

sk_status pinv_apply(sk_ctx* c, const double* B1, int64_t ldb, int64_t p, int64_t k, const double* D, int64_t ldd,
                     int64_t N, double* out, int64_t ldo, int64_t* status_dev) {
  DBuf Bc, Lf, U, Ut, G, piv;
  SK_TRY(Bc.alloc(c, (size_t)p * k * sizeof(double)));
  SK_TRY(Lf.alloc(c, (size_t)p * k * sizeof(double)));
  SK_TRY(U.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Ut.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(piv.alloc(c, (size_t)k * sizeof(int64_t)));
  SK_CUDA(c, cudaMemcpy2DAsync(Bc.p, (size_t)p * sizeof(double), B1, (size_t)ldb * sizeof(double),
                               (size_t)p * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  SK_CUDA(c, cudaMemsetAsync(U.p, 0, (size_t)k * k * sizeof(double), c->stream));
  SK_TRY(lupp(c, Bc.as<double>(), false, p, k, p, piv.as<int64_t>(), Lf.as<double>(), p, U.as<double>(), k, nullptr,
              status_dev));
  SK_TRY(gemm(c, true, false, k, k, p, 1.0, Lf.as<double>(), p, Lf.as<double>(), p, 0.0, G.as<double>(), k));
  SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
  SK_TRY(gemm(c, false, false, N, k, p, 1.0, D, ldd, Lf.as<double>(), p, 0.0, out, ldo));      // D Lf
  SK_TRY(trsm_right_lt(c, out, N, k, ldo, G.as<double>(), k));                                 // . L_G^{-T}
  SK_TRY(trsm_right_l(c, out, N, k, ldo, G.as<double>(), k));                                  // . L_G^{-1}
  SK_TRY(transpose(c, U.as<double>(), k, k, k, Ut.as<double>(), k));                           // U^T: lower
  return trsm_right_l(c, out, N, k, ldo, Ut.as<double>(), k);                                  // . U^{-T}
}

}  // namespace skel

using namespace skel;

namespace {
sk_status finish(sk_ctx* c, const int64_t* st_dev, int64_t* info, const char* what) {
  int64_t st = 0;
  SK_CUDA(c, cudaMemcpyAsync(&st, st_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  if (info) *info = st;
  if (st != 0) return fail(c, SK_E_RANK, std::string(what) + ": rank deficiency at step " + std::to_string(st));
  return SK_OK;
}
}  // namespace

extern "C" {

sk_status sk_sketch_dual(sk_ctx* c, const double* A, int a_on_host, int64_t m, int64_t n, int64_t lda, int64_t lx,
                         int64_t ly, sk_embedding emb, uint64_t seed_x, uint64_t seed_y, double* X, int64_t ldx,
                         double* Y, int64_t ldy) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && X && Y, "sk_sketch_dual: NULL pointer");
  SK_ARG(c, !dist_on(c), "sk_sketch_dual: not available on a distributed context");
  SK_ARG(c, emb == SK_EMB_GAUSSIAN, "sk_sketch_dual: the fused single pass is Gaussian-only");
  SK_ARG(c, m >= 1 && n >= 1 && lda >= m && lx >= 1 && lx <= m && ly >= 1 && ly <= n && ldx >= n && ldy >= m,
         "sk_sketch_dual: need 1 <= lx <= m, 1 <= ly <= n, lda >= m, ldx >= n, ldy >= m");
  SK_CUDA(c, cudaSetDevice(c->device));
  return sketch_dual(c, A, a_on_host != 0, m, n, lda, lx, ly, seed_x, seed_y, X, ldx, Y, ldy);
}

sk_status sk_id_estimate_cols(sk_ctx* c, const double* X, int64_t lx, int64_t n, int64_t ldx, const int64_t* Js,
                              int64_t k, double* Z, int64_t ldz, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, X && Js && Z, "sk_id_estimate_cols: NULL pointer");
  SK_ARG(c, !dist_on(c), "sk_id_estimate_cols: not available on a distributed context");
  SK_ARG(c, k >= 1 && k <= lx && k <= n && ldx >= n && ldz >= k, "sk_id_estimate_cols: need 1 <= k <= min(lx, n)");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf X1, Zt, st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_CUDA(c, cudaMemsetAsync(st.p, 0, sizeof(int64_t), c->stream));
  SK_TRY(X1.alloc(c, (size_t)lx * k * sizeof(double)));
  SK_TRY(Zt.alloc(c, (size_t)n * k * sizeof(double)));
  // X row-major lx x n (ldx) == X^T column-major n x lx; X_1 = X(:, Js) = (X^T(Js, :))^T
  SK_TRY(gather_rows_t(c, X, n, lx, ldx, Js, k, X1.as<double>(), lx));
  SK_TRY(pinv_apply(c, X1.as<double>(), lx, lx, k, X, ldx, n, Zt.as<double>(), n, st.as<int64_t>()));
  SK_TRY(transpose(c, Zt.as<double>(), n, k, n, Z, ldz));
  return finish(c, st.as<int64_t>(), info, "sk_id_estimate_cols");
}

sk_status sk_id_estimate_rows(sk_ctx* c, const double* Y, int64_t m, int64_t ly, int64_t ldy, const int64_t* Is,
                              int64_t k, double* W, int64_t ldw, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, Y && Is && W, "sk_id_estimate_rows: NULL pointer");
  SK_ARG(c, !dist_on(c), "sk_id_estimate_rows: not available on a distributed context");
  SK_ARG(c, k >= 1 && k <= ly && k <= m && ldy >= m && ldw >= m, "sk_id_estimate_rows: need 1 <= k <= min(ly, m)");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf Y1t, st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_CUDA(c, cudaMemsetAsync(st.p, 0, sizeof(int64_t), c->stream));
  SK_TRY(Y1t.alloc(c, (size_t)ly * k * sizeof(double)));
  SK_TRY(gather_rows_t(c, Y, m, ly, ldy, Is, k, Y1t.as<double>(), ly));                       // Y_1^T (ly x k)
  SK_TRY(pinv_apply(c, Y1t.as<double>(), ly, ly, k, Y, ldy, m, W, ldw, st.as<int64_t>()));
  return finish(c, st.as<int64_t>(), info, "sk_id_estimate_rows");
}

}  // extern "C"
