// deim.cu -- RSVD-DEIM column skeletons (the paper's pivoting comparator,
// Sec. 5 item 3; eq:rsvd_procedures P:237-243):
//     Q_X = ortho(X^T)                    (n x l, X = Gamma A the row sketch)
//     [U, S, V~] = svd(A Q_X, 'econ'),   V^ = Q_X V~               (eq:rsvd_procedures)
//     J_s = DEIM on V^(:, 0:k) = column-wise LUPP of V^(:, 0:k)^T  (Sorensen-Embree)
// The n x l and m x l products are this library's DMMA GEMMs, ortho(X^T) its LUPP-basis
// CholeskyQR2 (or shifted CholeskyQR3 for very tall panels), and the pivoting its cluster LUPP.
// The small SVD is cuSOLVER's: the l x l triangular factor R of A Q_X (geqrf) is decomposed
// with gesvd -- V~ of R equals V~ of A Q_X, and working on R avoids squaring the condition
// number (a Gram/eigh route would lose the trailing singular vectors at C2's 1e10 range).
// This is the comparison arm, not the method's hot path: a library SVD is a plain step here.
#include <cusolverDn.h>

#include "common.cuh"
#include "internal.h"

namespace skel {

namespace {
cusolverDnHandle_t solver(sk_ctx* c) {
  static cusolverDnHandle_t hs[kMaxDevices] = {};          // one handle per device (created on it)
  cusolverDnHandle_t& h = hs[c->device % kMaxDevices];
  if (!h) cusolverDnCreate(&h);
  cusolverDnSetStream(h, c->stream);
  return h;
}
}  // namespace

sk_status select_cols_deim(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* X, int64_t l,
                           int64_t ldx, int64_t k, int64_t* Js, int64_t* status_dev) {
  cusolverDnHandle_t h = solver(c);
  if (!h) return fail(c, SK_E_CUDA, "sk_select_cols_deim: cusolverDnCreate failed");
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  // Q_X = ortho(X^T): X row-major l x n (ldx) == X^T column-major n x l (ld ldx)
  DBuf Xt, Q, B, tau, S, VT, work, info, Vk;
  SK_TRY(Xt.alloc(c, (size_t)n * l * sizeof(double)));
  SK_TRY(Q.alloc(c, (size_t)n * l * sizeof(double)));
  SK_CUDA(c, cudaMemcpy2DAsync(Xt.p, n * sizeof(double), X, ldx * sizeof(double), n * sizeof(double), l,
                               cudaMemcpyDeviceToDevice, c->stream));
  SK_TRY(orthonormal_basis(c, Xt.as<double>(), n, l, Q.as<double>(), status_dev));
  Xt.release();
  // B = A Q_X (m x l), then B = Q_B R (geqrf), svd(R) -> V~^T (l x l)
  SK_TRY(B.alloc(c, (size_t)m * l * sizeof(double)));
  SK_TRY(gemm(c, false, false, m, l, n, 1.0, A, lda, Q.as<double>(), n, 0.0, B.as<double>(), m));
  SK_TRY(tau.alloc(c, (size_t)l * sizeof(double)));
  SK_TRY(info.alloc(c, sizeof(int)));
  int lw1 = 0, lw2 = 0;
  if (cusolverDnDgeqrf_bufferSize(h, (int)m, (int)l, B.as<double>(), (int)m, &lw1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDgesvd_bufferSize(h, (int)l, (int)l, &lw2) != CUSOLVER_STATUS_SUCCESS)
    return fail(c, SK_E_CUDA, "sk_select_cols_deim: cuSOLVER workspace query failed");
  SK_TRY(work.alloc(c, (size_t)std::max(lw1, lw2) * sizeof(double)));
  if (cusolverDnDgeqrf(h, (int)m, (int)l, B.as<double>(), (int)m, tau.as<double>(), work.as<double>(), lw1,
                       info.as<int>()) != CUSOLVER_STATUS_SUCCESS)
    return fail(c, SK_E_CUDA, "sk_select_cols_deim: geqrf failed");
  {
    int qinfo = 0;
    SK_CUDA(c, cudaMemcpyAsync(&qinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    if (qinfo != 0) return fail(c, SK_E_CUDA, "sk_select_cols_deim: cuSOLVER geqrf info = " + std::to_string(qinfo));
  }
  DBuf R;
  SK_TRY(R.alloc(c, (size_t)l * l * sizeof(double)));
  SK_TRY(upper_triangle(c, B.as<double>(), m, l, R.as<double>(), l));           // R (l x l), zeros below
  B.release();
  SK_TRY(S.alloc(c, (size_t)l * sizeof(double)));
  SK_TRY(VT.alloc(c, (size_t)l * l * sizeof(double)));
  DBuf rwork;
  SK_TRY(rwork.alloc(c, (size_t)l * sizeof(double)));
  if (cusolverDnDgesvd(h, 'N', 'A', (int)l, (int)l, R.as<double>(), (int)l, S.as<double>(), nullptr, (int)l,
                       VT.as<double>(), (int)l, work.as<double>(), std::max(lw1, lw2), rwork.as<double>(),
                       info.as<int>()) != CUSOLVER_STATUS_SUCCESS)
    return fail(c, SK_E_CUDA, "sk_select_cols_deim: gesvd failed");
  // cuSOLVER reports a failed factorisation only through the device info of each call: geqrf's
  // (illegal argument, < 0) was overwritten by gesvd's, so both are checked -- gesvd's info > 0 is
  // the number of superdiagonals of the bidiagonal form that did not converge
  int hinfo = 0;
  SK_CUDA(c, cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  if (hinfo != 0)
    return fail(c, SK_E_CUDA, "sk_select_cols_deim: cuSOLVER gesvd info = " + std::to_string(hinfo));
  // V^_k = Q_X V~(:, 0:k) = Q_X (V~^T(0:k, :))^T  (n x k, column-major)
  SK_TRY(Vk.alloc(c, (size_t)n * k * sizeof(double)));
  SK_TRY(gemm(c, false, true, n, k, l, 1.0, Q.as<double>(), n, VT.as<double>(), l, 0.0, Vk.as<double>(), n));
  // DEIM = LUPP on V^_k^T: pivot over the rows of the n x k panel V^_k, column t at step t
  return lupp(c, Vk.as<double>(), false, n, k, n, Js, nullptr, 0, nullptr, 0, nullptr, status_dev);
}

}  // namespace skel
