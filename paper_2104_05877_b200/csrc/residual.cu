// residual.cu -- S6: Frobenius residual of the column ID, row ID, stable CUR and C*Z.
//
// Paper: CC^+A (eq:def_column_id), AR^+R (eq:def_row_id), stable CUR
// Q_C (Q_C^T A Q_R) Q_R^T (Remark 2.3, eq:cur_stable; protocol P:554) and
// A ~ C Z (eq:colID).  Frobenius norm (R12).
//
// ortho(C): shifted CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020;
// cond(C) = 1.6e11 at C2 k=512, R20): Gram + shift, then Cholesky
// passes on the single-launch pair of dense.cu, the last pass a Newton-Schulz step when the one
// before leaves Q nearly orthonormal.  If a pass breaks down (C numerically rank deficient), the
// LUPP basis: the row LUPP of C (the S4 kernel) gives C = Lf_C U, range(C) = range(Lf_C), Lf_C
// well conditioned by construction (|entries| <= 1, unit lower pivot block), then CholeskyQR2
// (DESIGN.md section 7.6).  The residual A - Q (Q^T A) is never materialised: the last GEMM squares
// and sums its tiles in the epilogue.
#include "common.cuh"
#include "internal.h"

namespace skel {

// G <- G + s I with s = 11 (rows k + k (k + 1)) u trace(G)  (the shift of shifted CholeskyQR3,
// Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020: makes the first Cholesky succeed for
// cond(C) up to ~u^-1, after which CholeskyQR2 restores orthogonality).
__global__ void k_add_shift(double* G, int64_t k, int64_t ld, int64_t rows) {
  __shared__ double red[34];
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) t += G[i + i * ld];
  t = dev::block_sum(t, red);
  const double s = 11.0 * ((double)rows * (double)k + (double)k * (double)(k + 1)) * 1.1102230246251565e-16 * t;
  for (int64_t i = threadIdx.x; i < k; i += blockDim.x) G[i + i * ld] += s;
}

sk_status add_shift(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t rows) {
  k_add_shift<<<1, 1024, 0, c->stream>>>(G, k, ld, rows);
  return launched(c);
}

// Shifted CholeskyQR3: Q = C, G = Q^T Q + s I, Q <- Q L^{-T}, then CholeskyQR2 (whose second pass
// is a Newton-Schulz step when the first leaves |Q^T Q - I| <= 1e-10).
static sk_status basis_shifted_cholqr3(sk_ctx* c, const double* C, int64_t rows, int64_t k, double* Q,
                                       int64_t* status_dev) {
  SK_CUDA(c, cudaMemcpyAsync(Q, C, (size_t)rows * k * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if (k <= 1024) return cholqr_adaptive(c, Q, rows, k, rows, status_dev);   // the shift only where needed
  DBuf G;
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(gram_lower(c, Q, rows, k, rows, G.as<double>(), k));
  k_add_shift<<<1, 1024, 0, c->stream>>>(G.as<double>(), k, k, rows);
  SK_TRY(launched(c));
  SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
  SK_TRY(trsm_right_lt(c, Q, rows, k, rows, G.as<double>(), k));
  return cholqr2(c, Q, rows, k, rows, status_dev);
}

// sums[0] = ||A - L W||_F^2, sums[1] = ||A||_F^2 for L (m x k, ldl) and W given either as a k x n
// column-major matrix (Wc, ldw) or by its transpose (Wt, n x k column-major, ldwt): on the TMA + DMMA
// pipeline with the residual epilogue when the layouts allow it (W column-major with an even ld),
// else on the cp.async DMMA GEMM's sum-of-squares epilogue.
sk_status lowrank_sumsq(sk_ctx* c, const double* L, int64_t ldl, const double* Wc, int64_t ldw, const double* Wt,
                               int64_t ldwt, const double* A, int64_t lda, int64_t m, int64_t n, int64_t k, double* sums) {
  // the TMA pipeline amortises its per-tile ring fill over K = k: measured ahead at k = 1000 (C5
  // residual 1211 -> 1171 ms), even at k = 512 (C2), behind at k = 200 (C4 row ID 7.8 -> 8.3 ms)
  const bool tma = (reinterpret_cast<uintptr_t>(A) & 7) == 0 && m < (1LL << 31) && k >= 512;
  if (tma && Wc && ldw % 2 == 0 && (reinterpret_cast<uintptr_t>(Wc) & 15) == 0)
    return residual_sumsq_tma(c, L, ldl, Wc, ldw, A, lda, m, n, k, sums);
  if (tma) {
    DBuf W;
    const int64_t ld = k + (k & 1);
    SK_TRY(W.alloc(c, (size_t)ld * n * sizeof(double)));
    if (Wt) SK_TRY(transpose(c, Wt, n, k, ldwt, W.as<double>(), ld));
    else SK_CUDA(c, cudaMemcpy2DAsync(W.p, (size_t)ld * sizeof(double), Wc, (size_t)ldw * sizeof(double),
                                      (size_t)k * sizeof(double), (size_t)n, cudaMemcpyDeviceToDevice, c->stream));
    return residual_sumsq_tma(c, L, ldl, W.as<double>(), ld, A, lda, m, n, k, sums);
  }
  if (Wc) return gemm_sumsq(c, false, false, m, n, k, -1.0, L, ldl, Wc, ldw, 1.0, A, lda, sums);
  return gemm_sumsq(c, false, true, m, n, k, -1.0, L, ldl, Wt, ldwt, 1.0, A, lda, sums);
}

// sum of squares of a rows x cols block (ld) into part[2 * blockIdx.x + slot] (the other slot 0):
// column-strided over a fixed grid, so the reduction order is fixed
__global__ void k_sumsq_block(const double* __restrict__ X, int64_t rows, int64_t cols, int64_t ld, double* part,
                              int slot) {
  __shared__ double red[34];
  double s = 0.0;
  for (int64_t j = blockIdx.x; j < cols; j += gridDim.x)
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
      const double v = __ldcs(X + i + j * ld);
      s = fma(v, v, s);
    }
  s = dev::block_sum(s, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x + slot] = s;
    part[2 * blockIdx.x + 1 - slot] = 0.0;
  }
}

// When the projected part does not nearly exhaust A, the projection residual needs no second GEMM:
// for an orthogonal projection P (P A = Q W with W = Q^T A, or A P = W Q^T, or P_C A P_R with
// ||P_C A P_R|| = ||Q_C^T A Q_R||), ||A - P(A)||^2 = ||A||^2 - ||W||^2 exactly.  In floating point the
// difference loses log10(||A||^2 / r^2) digits; ||W||^2 carries ~(u ||Q^T Q - I|| + u sqrt(m)) relative
// error, so with r^2 >= 1e-3 ||A||^2 the result is good to ~1e-10 relative (the parity tolerance is
// 1e-9 r).  Returns true (sums written) when that holds, false when the explicit A - QW GEMM is needed.
static sk_status projection_residual(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* W,
                                     int64_t wr, int64_t wc, int64_t ldw, double* sums, bool* done) {
  *done = false;
  const int ga = (int)std::min<int64_t>(n, 4LL * c->num_sms), gw = (int)std::min<int64_t>(wc, 2LL * c->num_sms);
  DBuf part, out;
  SK_TRY(part.alloc(c, (size_t)2 * (ga + gw) * sizeof(double)));
  SK_TRY(out.alloc(c, 2 * sizeof(double)));
  k_sumsq_block<<<ga, 256, 0, c->stream>>>(A, m, n, lda, part.as<double>(), 0);
  SK_TRY(launched(c));
  k_sumsq_block<<<gw, 256, 0, c->stream>>>(W, wr, wc, ldw, part.as<double>() + 2 * ga, 1);
  SK_TRY(launched(c));
  SK_TRY(reduce_pairs(c, part.as<double>(), ga + gw, out.as<double>()));
  double h[2];
  SK_CUDA(c, cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  const double a2 = h[0], w2 = h[1], r2 = a2 - w2;
  if (!(a2 > 0.0) || !(r2 >= 1e-3 * a2)) return SK_OK;
  const double hs[2] = {r2, a2};
  SK_CUDA(c, cudaMemcpyAsync(sums, hs, sizeof(hs), cudaMemcpyHostToDevice, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  *done = true;
  return SK_OK;
}

sk_status col_id_sumsq(sk_ctx* c, const double* Q, const double* A, int64_t m, int64_t n, int64_t lda, int64_t k,
                       double* sums, bool try_projection) {
  // W = Q^T A by the sketch's TMA + DMMA GEMM (Omega := Q^T; written as W^T, n x k column-major),
  // turned column-major k x n (ld even, the tensor-map rule), then ||A - Q W||^2 and ||A||^2 on the
  // same pipeline with the residual epilogue (Q packed as the row operand, A read once in the epilogue)
  DBuf Wt, W;
  SK_TRY(Wt.alloc(c, (size_t)k * n * sizeof(double)));
  SK_TRY(gemm_qta(c, Q, m, A, m, n, lda, k, Wt.as<double>(), n));
  if (try_projection) {
    bool done = false;
    SK_TRY(projection_residual(c, A, m, n, lda, Wt.as<double>(), n, k, n, sums, &done));
    if (done) return SK_OK;
  }
  const int64_t ldw = k + (k & 1);
  if ((reinterpret_cast<uintptr_t>(A) & 7) == 0 && m < (1LL << 31) && k >= 512) {
    SK_TRY(W.alloc(c, (size_t)ldw * n * sizeof(double)));
    SK_TRY(transpose(c, Wt.as<double>(), n, k, n, W.as<double>(), ldw));
    Wt.release();
    return residual_sumsq_tma(c, Q, m, W.as<double>(), ldw, A, lda, m, n, k, sums);
  }
  return gemm_sumsq(c, false, true, m, n, k, -1.0, Q, m, Wt.as<double>(), n, 1.0, A, lda, sums);
}

sk_status orthonormal_basis(sk_ctx* c, const double* C, int64_t rows, int64_t k, double* Q, int64_t* status_dev) {
  // shifted CholeskyQR3 (all GEMMs + two single-launch Cholesky passes, the third pass a Newton-Schulz
  // step when the second leaves |Q^T Q - I| <= 1e-10; Fukaya et al. 2020, R20 for its
  // stability condition and the measured range).  When a pass breaks down (C numerically rank
  // deficient), the LUPP basis: range(C) = range(Lf_C), Lf_C well conditioned by construction, then
  // CholeskyQR2.
  SK_TRY(basis_shifted_cholqr3(c, C, rows, k, Q, status_dev));
  if (rows > lupp_max_rows(c)) return SK_OK;
  int64_t st = 0;
  SK_CUDA(c, cudaMemcpyAsync(&st, status_dev, sizeof(st), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  if (st == 0) return SK_OK;
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  DBuf piv;
  SK_TRY(piv.alloc(c, (size_t)k * sizeof(int64_t)));
  SK_TRY(lupp(c, C, false, rows, k, rows, piv.as<int64_t>(), Q, rows, nullptr, 0, nullptr, status_dev));
  return cholqr2(c, Q, rows, k, rows, status_dev);
}

sk_status residual(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* Js,
                   const int64_t* Is, int64_t k, int kind, const double* Z, int64_t ldz, double* sums,
                   int64_t* status_dev) {
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  if (kind == SK_RES_ID_COEFFS) {
    DBuf C;
    SK_TRY(C.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(gather_cols(c, A, m, lda, Js, k, C.as<double>(), m));
    return lowrank_sumsq(c, C.as<double>(), m, Z, ldz, nullptr, 0, A, lda, m, n, k, sums);
  }
  if (kind == SK_RES_ROW_COEFFS || kind == SK_RES_CUR_CSS) {
    // ||A - W R||, R = A(I_s, :): W given (the row-ID estimate Y Y_1^+) or W = C S^{-1}
    // (the CUR estimate C S^{-1} R) through the row LUPP of S^T (estimates.cu)
    DBuf Rt, V, Cb, St;
    SK_TRY(Rt.alloc(c, (size_t)n * k * sizeof(double)));
    SK_TRY(gather_rows_t(c, A, m, n, lda, Is, k, Rt.as<double>(), n));
    const double* Wp = Z;
    int64_t ldw = ldz;
    if (kind == SK_RES_CUR_CSS) {
      SK_TRY(Cb.alloc(c, (size_t)m * k * sizeof(double)));
      SK_TRY(St.alloc(c, (size_t)k * k * sizeof(double)));
      SK_TRY(V.alloc(c, (size_t)m * k * sizeof(double)));
      SK_TRY(gather_cols(c, A, m, lda, Js, k, Cb.as<double>(), m));
      SK_TRY(gather_rows_t(c, Cb.as<double>(), m, k, m, Is, k, St.as<double>(), k));          // S^T = C(I_s, :)^T
      SK_TRY(pinv_apply(c, St.as<double>(), k, k, k, Cb.as<double>(), m, m, V.as<double>(), m, status_dev));
      Wp = V.as<double>();
      ldw = m;
    }
    return lowrank_sumsq(c, Wp, ldw, nullptr, 0, Rt.as<double>(), n, A, lda, m, n, k, sums);
  }
  DBuf Qc, Qr, Cb, Rt, W;
  if (kind == SK_RES_COL_ID || kind == SK_RES_CUR) {
    SK_TRY(Cb.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(Qc.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(gather_cols(c, A, m, lda, Js, k, Cb.as<double>(), m));
    SK_TRY(orthonormal_basis(c, Cb.as<double>(), m, k, Qc.as<double>(), status_dev));
    Cb.release();
  }
  if (kind == SK_RES_ROW_ID || kind == SK_RES_CUR) {
    SK_TRY(Rt.alloc(c, (size_t)n * k * sizeof(double)));
    SK_TRY(Qr.alloc(c, (size_t)n * k * sizeof(double)));
    SK_TRY(gather_rows_t(c, A, m, n, lda, Is, k, Rt.as<double>(), n));
    SK_TRY(orthonormal_basis(c, Rt.as<double>(), n, k, Qr.as<double>(), status_dev));
    Rt.release();
  }
  if (kind == SK_RES_COL_ID) return col_id_sumsq(c, Qc.as<double>(), A, m, n, lda, k, sums, true);
  if (kind == SK_RES_ROW_ID) {
    SK_TRY(W.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(gemm(c, false, false, m, k, n, 1.0, A, lda, Qr.as<double>(), n, 0.0, W.as<double>(), m));
    bool done = false;
    SK_TRY(projection_residual(c, A, m, n, lda, W.as<double>(), m, k, m, sums, &done));
    if (done) return SK_OK;
    return lowrank_sumsq(c, W.as<double>(), m, nullptr, 0, Qr.as<double>(), n, A, lda, m, n, k, sums);
  }
  // CUR: W = Qc^T A (k x n), Mid = W Qr (k x k), B = Qc Mid (m x k), residual A - B Qr^T
  DBuf Mid, B;
  SK_TRY(W.alloc(c, (size_t)k * n * sizeof(double)));
  SK_TRY(Mid.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(B.alloc(c, (size_t)m * k * sizeof(double)));
  SK_TRY(gemm_qta(c, Qc.as<double>(), m, A, m, n, lda, k, W.as<double>(), n));            // W^T, n x k
  SK_TRY(gemm(c, true, false, k, k, n, 1.0, W.as<double>(), n, Qr.as<double>(), n, 0.0, Mid.as<double>(), k));
  bool done = false;
  SK_TRY(projection_residual(c, A, m, n, lda, Mid.as<double>(), k, k, k, sums, &done));
  if (done) return SK_OK;
  SK_TRY(gemm(c, false, false, m, k, k, 1.0, Qc.as<double>(), m, Mid.as<double>(), k, 0.0, B.as<double>(), m));
  return lowrank_sumsq(c, B.as<double>(), m, nullptr, 0, Qr.as<double>(), n, A, lda, m, n, k, sums);
}

sk_status residual_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* C, int64_t k,
                        int64_t ldc, double* sums, int64_t* status_dev) {
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  DBuf Cc, Qc, W;
  SK_TRY(Cc.alloc(c, (size_t)m * k * sizeof(double)));
  SK_TRY(Qc.alloc(c, (size_t)m * k * sizeof(double)));
  SK_CUDA(c, cudaMemcpy2DAsync(Cc.p, (size_t)m * sizeof(double), C, (size_t)ldc * sizeof(double), (size_t)m * sizeof(double),
                               (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  SK_TRY(orthonormal_basis(c, Cc.as<double>(), m, k, Qc.as<double>(), status_dev));
  Cc.release();
  return col_id_sumsq(c, Qc.as<double>(), A, m, n, lda, k, sums, true);
}

}  // namespace skel
