// internal.h -- host-side drivers shared by the translation units of libskel.so.
#pragma once
#include <functional>

#include "common.cuh"

namespace skel {

// ---------------------------------------------------------------- GEMM (gemm.cu)
// C (M x N, col-major, ldc) = alpha * op(A) op(B) + beta * C, all FP64 column-major.
// op(A) is M x K (A stored M x K if !ta, K x M if ta); op(B) is K x N.
sk_status gemm(sk_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
               const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
               int64_t ldc);
// G = Q^T Q (k x k, ldg): only the 64 x 64 tiles on or below the diagonal are written
sk_status gram_lower(sk_ctx* c, const double* Q, int64_t m, int64_t k, int64_t ldq, double* G, int64_t ldg);
// sums[0] += ||beta*C + alpha*op(A)op(B)||_F^2 and sums[1] += ||C||_F^2, C read only
// (the fused residual reduction).  sums: device double[2], overwritten.
sk_status gemm_sumsq(sk_ctx* c, bool ta, bool tb, int64_t M, int64_t N, int64_t K, double alpha,
                     const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                     const double* C, int64_t ldc, double* sums);

// ---------------------------------------------------------------- sketch (sketch.cu)
sk_status sketch_dense(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                       uint64_t seed, double* X, int64_t ldx);
sk_status sketch_sparse(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                        int zeta, uint64_t seed, double* X, int64_t ldx);

// X = Gamma A with the SRTT embedding (srtt.cu); m a power of two <= 16384.
sk_status sketch_srtt(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, uint64_t seed,
                      double* X, int64_t ldx);
// X (l x n row-major, ldx >= n; == X^T column-major) = Q^T A for a given Q (m x l column-major, ldq):
// the sketch's TMA + DMMA GEMM with Omega = Q^T packed into its image (falls back to gemm()).
sk_status gemm_qta(sk_ctx* c, const double* Q, int64_t ldq, const double* A, int64_t m, int64_t n, int64_t lda,
                   int64_t l, double* X, int64_t ldx);
// Algorithm 3's dual sketch in one pass over A: X = Gamma A (lx x n row-major), Y = A Omega^T (m x ly
// col-major), both Gaussian (Gamma over A's rows from seed_x, Omega over A's columns from seed_y).
sk_status sketch_dual(sk_ctx* c, const double* A, bool a_on_host, int64_t m, int64_t n, int64_t lda, int64_t lx,
                      int64_t ly, uint64_t seed_x, uint64_t seed_y, double* X, int64_t ldx, double* Y, int64_t ldy);
// sums[0] = ||A - Q W||_F^2, sums[1] = ||A||_F^2 (Q m x k col-major, W k x n col-major with an even
// ldw, A m x n col-major) on the TMA + DMMA sketch pipeline with the residual epilogue (S6).
sk_status residual_sumsq_tma(sk_ctx* c, const double* Q, int64_t ldq, const double* W, int64_t ldw, const double* A,
                             int64_t lda, int64_t m, int64_t n, int64_t k, double* sums);
// Y = A Omega^T (m x l col-major, ldy >= m), Omega l x n (Alg. 3 column sketch).
sk_status sketch_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                      int zeta, uint64_t seed, double* Y, int64_t ldy);
// X = Omega (A^T A)^q (eq:def_power_iter), Omega l x n drawn like the sketch's Gamma
// over the n index; q >= 1.  X l x n row-major (ldx >= n).
sk_status sketch_power(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                       int zeta, uint64_t seed, int q, double* X, int64_t ldx);
// eq:ortho_power_iter: X = ortho(Y_q)^T A with Y_1 = A Omega^T, Y_i = ortho(A ortho(A^T Y_{i-1}));
// status_dev = 0 or the rank failure of an orthogonalisation.
sk_status sketch_power_ortho(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l, int emb,
                             int zeta, uint64_t seed, int q, double* X, int64_t ldx, int64_t* status_dev);

// ---------------------------------------------------------------- LUPP (lupp.cu)
// k-step swap-free LUPP on the rows of an n x k panel.  The panel is given either
// as rows 0..k-1 of a row-major X (row_major = true, ld = ldx) or as a column-major
// n x k matrix (row_major = false, ld = ldc).  Outputs device Js[k]; Lf (n x k, ldlf)
// is required (workspace-backed if the caller passed NULL); U/gaps optional.
// status_dev: device int64 written with 0 or the failing 1-based step.
sk_status lupp(sk_ctx* c, const double* P, bool row_major, int64_t n, int64_t k, int64_t ld,
               int64_t* Js, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* gaps,
               int64_t* status_dev);

// Q (rows x k, ld rows) = an orthonormal basis of range(C) (C rows x k, ld rows): LUPP basis +
// CholeskyQR2, or shifted CholeskyQR3 for panels taller than one cluster's LUPP (residual.cu).
sk_status orthonormal_basis(sk_ctx* c, const double* C, int64_t rows, int64_t k, double* Q, int64_t* status_dev);
// sums[0] = ||A - L W||_F^2, sums[1] = ||A||_F^2, L m x k (ldl), W k x n given column-major (Wc, ldw)
// or as its transpose (Wt n x k column-major, ldwt; pass the other nullptr) (residual.cu).
sk_status lowrank_sumsq(sk_ctx* c, const double* L, int64_t ldl, const double* Wc, int64_t ldw, const double* Wt,
                        int64_t ldwt, const double* A, int64_t lda, int64_t m, int64_t n, int64_t k, double* sums);
// sums[0] = ||A - Q Q^T A||_F^2, sums[1] = ||A||_F^2 for an orthonormal Q (m x k, ld m) (residual.cu).
sk_status col_id_sumsq(sk_ctx* c, const double* Q, const double* A, int64_t m, int64_t n, int64_t lda, int64_t k,
                       double* sums,
                       bool try_projection = false);
// R (n x n, ldr) = upper triangle of B (first n columns, ldb), zeros below (dense.cu).
sk_status upper_triangle(sk_ctx* c, const double* B, int64_t ldb, int64_t n, double* R, int64_t ldr);
// RSVD-DEIM column skeletons from A and its row sketch X (deim.cu).
sk_status select_cols_deim(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* X, int64_t l,
                           int64_t ldx, int64_t k, int64_t* Js, int64_t* status_dev);
// The context's lowest-priority helper stream and its two events, created on first use.
sk_status ensure_aux(sk_ctx* c);
// Tallest panel the cluster LUPP handles (rows).
int64_t lupp_max_rows(sk_ctx* c);

// ---------------------------------------------------------------- distributed LUPP (lupp_dist.cu)
// Per-step-exchange column LUPP on a column-sharded panel; see include/skel.h.
size_t lupp_dist_state_bytes(int64_t nloc, int64_t k);
size_t lupp_dist_mailbox_bytes(int64_t k, int world);
// peers == nullptr: the caller all-gathers `cand` into `gathered` between steps; else P2P mailboxes
sk_status lupp_dist_begin(sk_ctx* c, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0, void* state,
                          double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand, double* const* peers = nullptr,
                          int rank = 0, int world = 1, double* own_mailbox = nullptr);
sk_status lupp_dist_step(sk_ctx* c, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                         const double* gathered, int world, int64_t* Js, double* Lf, int64_t ldlf, double* U,
                         int64_t ldu, double* cand, double* const* peers = nullptr, int rank = 0);
sk_status lupp_dist_status(sk_ctx* c, const void* state, int64_t* status_dev_out);

// ---------------------------------------------------------------- CPQR (cpqr.cu)
sk_status cpqr(sk_ctx* c, const double* X, int64_t l, int64_t n, int64_t ldx, int64_t k,
               int64_t* Js, double* R, int64_t ldr, int64_t* status_dev);

// ---------------------------------------------------------------- small dense kernels (dense.cu)
sk_status gather_cols(sk_ctx* c, const double* A, int64_t m, int64_t lda, const int64_t* J,
                      int64_t k, double* C, int64_t ldc);
// Out (cols x rows, ldout) = In^T, In rows x cols (ldin), column-major.
sk_status transpose(sk_ctx* c, const double* In, int64_t rows, int64_t cols, int64_t ldin, double* Out,
                    int64_t ldout);
// Shard-aware gather: C(:, t) = A(:, J[t] - col0) if the column is in [col0, col0 + ncols), else 0.
sk_status gather_cols_shard(sk_ctx* c, const double* A, int64_t m, int64_t lda, int64_t col0, int64_t ncols,
                            const int64_t* J, int64_t k, double* C, int64_t ldc);
// R^T (n x k, col-major ld n) = A(I, :)^T, A m x n; indices outside [0, m) give zero columns
sk_status gather_rows_t(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I,
                        int64_t k, double* Rt, int64_t ldrt);
// In-place blocked Cholesky of the SPD k x k matrix G (lower, col-major ld); status_dev = 0 or
// 1-based failing column.
sk_status potrf_lower(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t* status_dev);
// X (rows x k, ldx) <- X * L^{-T} with L lower k x k non-unit (Cholesky factor).
sk_status trsm_right_lt(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L,
                        int64_t ldl);
// X (rows x k, ldx) <- X * L^{-1} with L unit lower k x k.
sk_status trsm_right_l_unit(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx,
                            const double* L, int64_t ldl);
// X (rows x k, ldx) <- X * L^{-1} with L non-unit lower k x k.
sk_status trsm_right_l(sk_ctx* c, double* X, int64_t rows, int64_t k, int64_t ldx, const double* L, int64_t ldl);
// out (N x k, ldo) = D B1 (B1^T B1)^{-1} = D (B1^+)^T for B1 p x k (col-major, ld ldb, p >= k, full
// column rank) and D N x p (ldd): through B1 = Lf U (row LUPP, |Lf| <= 1) so only the well-conditioned
// Gram Lf^T Lf is factored: out = D Lf (Lf^T Lf)^{-1} U^{-T} (estimates.cu).
sk_status pinv_apply(sk_ctx* c, const double* B1, int64_t ldb, int64_t p, int64_t k, const double* D, int64_t ldd,
                     int64_t N, double* out, int64_t ldo, int64_t* status_dev);
// Q (m x k, ldq) := orthonormal basis of range(Q) by two Cholesky-QR passes.
sk_status cholqr2(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev);
// the CholeskyQR tail (Gram, then Newton-Schulz when |Q^T Q - I| <= 1e-10, else a Cholesky pass), and the
// basis's first pass with the shift only where needed (both for k <= 1024; dense.cu)
sk_status cholqr_tail(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev);
sk_status cholqr_adaptive(sk_ctx* c, double* Q, int64_t m, int64_t k, int64_t ldq, int64_t* status_dev);
// out[0] = sum of in[0..n) pairs etc: finishes per-CTA partial sums deterministically.
sk_status reduce_pairs(sk_ctx* c, const double* partial, int64_t count, double* out);
// largest eigenvalue of the SPD k x k matrix G by power iteration (device result).
sk_status lambda_max(sk_ctx* c, const double* G, int64_t k, int64_t ld, double* out_dev);

// ---------------------------------------------------------------- ID coefficients (idcoef.cu)
sk_status id_coeffs(sk_ctx* c, const double* Lf, int64_t n, int64_t k, int64_t ldlf,
                    const int64_t* Js, double* Z, int64_t ldz, double* eta_dev);

// ---------------------------------------------------------------- residual (residual.cu)
sk_status residual(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda,
                   const int64_t* Js, const int64_t* Is, int64_t k, int kind, const double* Z,
                   int64_t ldz, double* sums_dev, int64_t* status_dev);

// sums[0] = ||A - Q Q^T A||_F^2, sums[1] = ||A||_F^2 with Q = ortho(C) (C m x k given explicitly;
// the distributed column-ID residual, where C is assembled across ranks).
sk_status residual_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* C, int64_t k,
                        int64_t ldc, double* sums_dev, int64_t* status_dev);

// Stream a HOST column-major m x n A through a 3-slot device ring in column blocks (capi.cu):
// fn(block, j0, jw) runs on the context stream for each block (device copy, ld m) in order.
sk_status for_host_blocks(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda,
                          const std::function<sk_status(const double*, int64_t, int64_t)>& fn);

// ---------------------------------------------------------------- column-sharded context (dist.cu)
// A context made by sk_create_dist owns an NCCL communicator and this rank's column block
// [col0, col0 + ncols) of an m x n_global A (partition of every rank known to all).
struct DistView {
  int rank = 0, world = 1;
  int64_t n_global = 0, col0 = 0, ncols = 0;
  int exchange = 0;   // 0 gather-then-replicate, 1 per-step all-gather (CUDA graph)
};
bool dist_on(const sk_ctx* c);
DistView dist_view(const sk_ctx* c);
void dist_destroy(sk_ctx* c);
// in-place sum over ranks (count doubles) / all-gather of count doubles per rank, on the ctx stream
sk_status dist_allreduce_sum(sk_ctx* c, double* buf, int64_t count);
sk_status dist_allgather(sk_ctx* c, const double* send, double* recv, int64_t count);
// S2 on this rank's sketch block X (l x ncols): Js replicated, Lf this rank's rows, U/gaps replicated
sk_status dist_select_cols(sk_ctx* c, const double* X, int64_t ncols, int64_t ldx, int64_t k, int64_t* Js, double* Lf,
                           int64_t ldlf, double* U, int64_t ldu, double* gaps, int64_t* status_dev);
// S3: C = A_global(:, Js) replicated on every rank (synchronises: reads Js on the host).  A is this
// rank's block (device, or host when a_on_host).
sk_status dist_gather_cols(sk_ctx* c, const double* A, bool a_on_host, int64_t m, int64_t lda, const int64_t* Js,
                           int64_t k, double* C, int64_t ldc);
// S5 on this rank's rows of Lf: Z (k x ncols) for this rank's columns; eta over all ranks
sk_status dist_id_coeffs(sk_ctx* c, const double* Lf, int64_t k, int64_t ldlf, const int64_t* Js, double* Z,
                         int64_t ldz, double* eta_dev);
// S6: squared sums over all ranks of the residual of `kind` and of A (sums_dev[2])
sk_status dist_residual(sk_ctx* c, const double* A, int64_t m, int64_t lda, const int64_t* Js, const int64_t* Is,
                        int64_t k, int kind, const double* Z, int64_t ldz, double* sums_dev, int64_t* status_dev);
// G <- G + s I, the shift of shifted CholeskyQR3 for a basis of `rows` rows (residual.cu)
sk_status add_shift(sk_ctx* c, double* G, int64_t k, int64_t ld, int64_t rows);
// ID-coefficient pieces shared with the distributed path (idcoef.cu): L1 = Lf(Js - off, :) with rows
// outside [0, nrows) zero; Z = Y^T with Z(:, Js - off) = I and those rows of Y zeroed; eta from Y^T Y
sk_status id_l1(sk_ctx* c, const double* Lf, int64_t nrows, int64_t ldlf, const int64_t* Js, int64_t k, int64_t off,
                double* L1);
sk_status id_finish(sk_ctx* c, double* Y, int64_t nrows, int64_t k, const int64_t* Js, int64_t off, double* Z,
                    int64_t ldz);

}  // namespace skel
