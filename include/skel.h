/*
 * skel.h -- C ABI of libskel.so: the B200 (sm_100a) hot path of randomized
 * LUPP skeleton selection (Dong & Martinsson, "Simpler is better: a
 * comparative study of randomized pivoting algorithms for CUR and
 * interpolative decompositions", arXiv 2104.05877).
 *
 * Citations: P:<n> = line n of the paper text (PAPER.md, the LaTeX source);
 * readings R<n> = DESIGN.md section 3, where every place the paper is silent
 * or ambiguous is resolved.
 *
 * Conventions (all entry points)
 *   - Matrices are IEEE FP64.  Indices are int64, 0-based (the paper is
 *     1-based MATLAB).
 *   - A is COLUMN-major m x n with leading dimension lda >= m.
 *   - The sketch X is ROW-major l x n with row stride ldx >= n (== X^T
 *     column-major n x l, the panel the LUPP works on).
 *   - C (m x k), Lf (n x k), Z (k x n), R^T panels are column-major.
 *   - Pointers are CUDA device pointers on the context's device unless the
 *     argument is documented "host".  The caller owns every buffer; a context
 *     owns only its workspace (grown on demand, reused, freed by sk_destroy).
 *   - Every call is enqueued on the context's stream and returns without
 *     synchronising, EXCEPT calls that write a host scalar (info, eta,
 *     res_fro, ...), which synchronise that stream before returning.
 *   - Errors: the return value.  SK_E_ARG for a bad size, leading dimension,
 *     NULL required pointer or parameter out of range (checked before any
 *     work is enqueued, nothing is written); SK_E_RANK when a pivot of
 *     magnitude <= 1e-14 * max|panel| is met (R7), with *info = the 1-based
 *     failing step (LAPACK style); SK_E_CUDA for a CUDA runtime error;
 *     SK_E_NOMEM when the workspace cannot grow.  sk_last_error() returns a
 *     human-readable message for the last non-OK status of the context.
 *   - Thread safety: one context per (thread, stream).  Contexts are
 *     independent; different contexts may run concurrently.
 *   - There is no CPU fallback: every step runs in this library's kernels.
 */
#ifndef SKEL_H_
#define SKEL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sk_ctx sk_ctx;

typedef enum {
  SK_OK = 0,
  SK_E_ARG = 1,
  SK_E_RANK = 2,
  SK_E_CUDA = 3,
  SK_E_NCCL = 4,
  SK_E_NOMEM = 5,
  SK_E_STATE = 6
} sk_status;

/* Oblivious l2 embeddings Gamma.  Gaussian: i.i.d. N(0, 1/l)
 * (R3).  Sparse sign: zeta nonzeros +-1/sqrt(zeta) per column at
 * uniformly random distinct rows (R4); zeta = min(l, 8) in practice
 * (P:185).  Both are regenerated on the fly from (seed, row, column) with
 * Philox4x32-10 (R1, R2) and never stored whole: the dense sketch regenerates
 * Gaussian Gamma one K-chunk at a time into a reused, L2-sized image slot (at
 * most 80 MB; its stores are evict_last, so the slot stays in L2), the sparse
 * sketch keeps only the nonzero structure (4 bytes per nonzero) and
 * regenerates nothing else.  SRTT:
 * sqrt(m/l) Pi_{m->l} T Phi Pi_{m->m} with T the unitary discrete Hartley transform, the random
 * permutation / selection as keyed Feistel bijections and the signs from Philox (R18); applied by
 * a per-column radix-2 FFT in shared memory: m a power of two <= 16384 in one CTA per column, and
 * 32768 <= m <= 131072 (with l <= 5800) in a cluster of m/16384 CTAs per column whose partial
 * transforms are combined over distributed shared memory (R19); SK_E_ARG otherwise. */
typedef enum { SK_EMB_GAUSSIAN = 0, SK_EMB_SPARSE_SIGN = 1, SK_EMB_SRTT = 2 } sk_embedding;

/* Which approximation sk_residual measures (Frobenius norm, R12).
 *   COL_ID    ||A - C C^+ A||              eq:def_column_id
 *   ROW_ID    ||A - A R^+ R||              eq:def_row_id,
 *   CUR       ||A - Q_C (Q_C^T A Q_R) Q_R^T||   stable CUR, Remark 2.3
 *   ID_COEFFS ||A - C Z||                  eq:colID, with Z from sk_id_coeffs (or the
 *                                          column-ID estimate X_1^+ X of sk_id_estimate_cols)
 *   ROW_COEFFS ||A - W R||                 R = A(I_s, :), W (m x k) given -- e.g. the row-ID estimate
 *                                          Y Y_1^+ of sk_id_estimate_rows
 *   CUR_CSS   ||A - C S^{-1} R||           S = A(I_s, J_s): the sketch-free CUR estimate */
typedef enum {
  SK_RES_COL_ID = 0,
  SK_RES_ROW_ID = 1,
  SK_RES_CUR = 2,
  SK_RES_ID_COEFFS = 3,
  SK_RES_ROW_COEFFS = 4,
  SK_RES_CUR_CSS = 5
} sk_residual_kind;

/* ---- context ----------------------------------------------------------- */

/* Create a context on CUDA device `device`, enqueueing on `stream`
 * (a cudaStream_t; NULL = the legacy default stream).  *ctx is set on success. */
sk_status sk_create(sk_ctx** ctx, int device, void* stream);
/* Re-target the context to another stream of the same device. */
sk_status sk_set_stream(sk_ctx* ctx, void* stream);
/* ---- column-sharded (multi-GPU) context -------------------------------
 * One process per GPU; A (m x n_global) is split into contiguous column blocks in rank order, this
 * rank holding columns [col0, col0 + ncols) (ncols may be 0).  The context owns an NCCL
 * communicator over the `world` ranks (NCCL resolved at run time from libnccl.so.2) and issues
 * every exchange of the path itself, on the context's stream:
 *   sk_sketch       unchanged: this rank's block, no communication (Gamma depends on the row index
 *                   of A only, R1, so every rank regenerates the same Gamma).
 *   sk_select_cols  X = this rank's l x ncols sketch block (n = ncols); Js, U, gaps replicated
 *                   (GLOBAL column indices), Lf = this rank's ncols x k rows.  Exchange
 *                   (sk_set_dist_exchange): 0 (default) one all-gather of the k LUPP-visible sketch
 *                   rows then the single-GPU LUPP on identical bytes; 1 one all-gather of the
 *                   ranks' candidate records per pivot step (the begin + k steps captured once in a
 *                   CUDA graph owned by the context; gaps != NULL falls back to 0).  Both equal
 *                   sk_select_cols on the unsharded sketch (ties to the lowest GLOBAL index, R6).
 *   sk_gather_cols  A = this rank's block (n = ncols), Js global; C (m x k) = A_global(:, Js) on
 *                   every rank (one all-gather of the owners' columns).  Synchronises.
 *   sk_id_coeffs    Lf = this rank's rows (n = ncols); Z (k x ncols) = this rank's columns of Z;
 *                   eta over all ranks.
 *   sk_residual     A = this rank's block; res_fro / normA_fro over the whole A (all kinds): Q_C by
 *                   Cholesky QR distributed over row blocks (one k x k all-reduce per pass), Q_R
 *                   kept sharded with A's columns, one all-reduce of the squared sums.
 *   sk_rand_lupp    A = this rank's block (device or host); Js / Is global, on every rank.
 * Every rank must make the same sequence of calls (collectives).  Errors: SK_E_NCCL when NCCL
 * cannot be loaded or a collective fails; SK_E_ARG when the ranks' blocks are not contiguous in
 * rank order or do not cover [0, n_global). */
#define SK_NCCL_UNIQUE_ID_BYTES 128
/* Write a fresh NCCL unique id (SK_NCCL_UNIQUE_ID_BYTES bytes, host) -- on one rank, then share it. */
sk_status sk_nccl_unique_id(void* out);
/* Collective over the `world` ranks: create a column-sharded context on `device` / `stream`. */
sk_status sk_create_dist(sk_ctx** ctx, int device, void* stream, const void* nccl_uid, int rank, int world,
                         int64_t n_global, int64_t col0, int64_t ncols);
/* Select the column-LUPP exchange of a distributed context: 0 gather-then-replicate, 1 per step. */
sk_status sk_set_dist_exchange(sk_ctx* ctx, int32_t exchange);
/* This context's place in the partition (world = 1, n_global = 0 for a single-GPU context). */
sk_status sk_dist_info(const sk_ctx* ctx, int32_t* rank, int32_t* world, int64_t* n_global, int64_t* col0,
                       int64_t* ncols);
/* Release the workspace and the context (synchronises its stream). NULL is a no-op. */
void sk_destroy(sk_ctx* ctx);
/* Message of the last non-OK status returned through ctx ("" if none). Never NULL. */
const char* sk_last_error(const sk_ctx* ctx);
/* Library version string, e.g. "skel 0.1 sm_100a". */
const char* sk_version(void);
/* Bytes of device workspace currently held by ctx. */
int64_t sk_workspace_bytes(const sk_ctx* ctx);
/* Number of kernels this context has launched so far (for the bench's gpu_launches count). */
int64_t sk_launch_count(const sk_ctx* ctx);

/* ---- S0 + S1: sketch  (Algorithm 2 lines 1-2) ---------------- */

/* X = Gamma A.  Gamma (l x m) is drawn from (emb, zeta, seed) on every call (Philox4x32-10,
 * R1-R4) and never held in HBM as a whole: the Gaussian one is generated one K-chunk of A's rows
 * at a time into an L2-sized workspace slot (<= ~80 MB) that the FP64 tensor-core GEMM reads
 * before the next chunk overwrites it; the sparse-sign structure goes into a per-call CSR
 * (4 bytes per nonzero, values never stored), SRTT's permutations and signs are drawn per CTA.
 *   A   m x n column-major (lda >= m), read only.
 *   X   l x n row-major (ldx >= n), written.
 *   Requires 1 <= l <= m, n >= 0; for SK_EMB_SPARSE_SIGN 2 <= zeta <= min(l, 64)
 *   (zeta is ignored for SK_EMB_GAUSSIAN).  X must not alias A. */
sk_status sk_sketch(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                    int64_t l, sk_embedding emb, int32_t zeta, uint64_t seed,
                    double* X, int64_t ldx);

/* Tuning of the dense (Gaussian) sketch for this context; 0 everywhere = automatic (the default).
 *   path        0 automatic (TMA + DMMA over K-chunks), 1 the fallback kernel that generates each
 *               Gamma tile in shared memory (used automatically when A's layout rules out TMA),
 *               2 / 3 the TMA path with K-splits summed through HBM partials / through the
 *               distributed shared memory of a cluster of the splits
 *   bm          CTA row-tile height: 0 or one of 32, 40, 48, 56, 64, 80
 *   warps       consumer warps per CTA: 7 (224 columns) or 8 (256) of BM x 32 each; 4 (bm = 80) or
 *               2 (bm = 40): the 112-column tiles of 40 x 56 warps; 0 = planner.  The (bm, warps)
 *               pairs that exist: (32|40|48|56|64, 8), (40|48, 7), (80, 4), (40, 2)
 *   splits      K-splits per chunk (0 = planner, 1..64)
 *   chunk_rows  rows of A per K-chunk, rounded up to 16 (0 = the largest whose Gamma slot fits ~80 MB)
 * Results are identical up to summation order (parity tests use it to reach every plan). */
sk_status sk_set_sketch_tuning(sk_ctx* ctx, int32_t path, int32_t bm, int32_t warps, int32_t splits,
                               int64_t chunk_rows);

/* ---- column sketch for streaming two-sided selection (Algorithm 3) ----
 * Y = A Omega^T with Omega an l x n embedding drawn like sk_sketch's Gamma over the column index
 * of A (an independent draw from X = Gamma A when the seed differs, Alg. 3 line 1).  Row-wise
 * LUPP on Y (sk_select_rows) gives I_s without forming C (Alg. 3 line 4).  A m x n column-major;
 * Y m x l column-major (ldy >= m).  Requires 1 <= l <= n.  Gaussian: one pass over A, Omega generated
 * one block of A's columns at a time (L2-sized slot) and accumulated by the DMMA GEMM; sparse sign
 * and SRTT: the row sketch of a transposed copy of A. */
sk_status sk_sketch_cols(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                         sk_embedding emb, int32_t zeta, uint64_t seed, double* Y, int64_t ldy);

/* ---- Algorithm 3's dual sketch in ONE pass over A ----
 * X = Gamma A (lx x n row-major, ldx >= n; Gamma over A's rows from seed_x, exactly sk_sketch's) and
 * Y = A Omega^T (m x ly column-major, ldy >= m; Omega over A's columns from seed_y, exactly
 * sk_sketch_cols') -- independent embeddings (Alg. 3 line 1).  a_on_host = 1: A is a HOST pointer
 * (the streaming setting of Alg. 3) and crosses PCIe exactly once, in column blocks
 * through a 3-slot device ring, each block feeding both products (X's block of columns and Y's
 * term A_block Omega_block^T, accumulated in block order).  a_on_host = 0: A in device memory, the
 * two products as two full-efficiency passes.  Gaussian only (SK_E_ARG otherwise).  Requires
 * 1 <= lx <= m, 1 <= ly <= n. */
sk_status sk_sketch_dual(sk_ctx* ctx, const double* A, int a_on_host, int64_t m, int64_t n, int64_t lda, int64_t lx,
                         int64_t ly, sk_embedding emb, uint64_t seed_x, uint64_t seed_y, double* X, int64_t ldx,
                         double* Y, int64_t ldy);

/* ---- sketch-only ID estimates without revisiting A ----
 * sk_id_estimate_cols: Z = X_1^+ X (k x n column-major, ldz >= k), X_1 = X(:, Js) the lx x k column
 *   pivots of the row sketch (C^+ A ~ X_1^+ X; Z(:, Js) = I up to rounding).
 * sk_id_estimate_rows: W = Y Y_1^+ (m x k column-major, ldw >= m), Y_1 = Y(Is, :) the k x ly row
 *   pivots of the column sketch (A R^+ ~ Y Y_1^+).
 * Both through the row LUPP of the pivot block (B1 = Lf U, |Lf| <= 1) and the Cholesky factor of
 * Lf^T Lf, i.e. without forming the normal equations of B1.  Require 1 <= k <= min(l, n or m).
 * info as for sk_select_cols (SK_E_RANK if the pivot block is numerically rank deficient).
 * The residuals ||A - C Z|| / ||A - W R|| / ||A - C S^{-1} R|| are sk_residual kinds ID_COEFFS /
 * ROW_COEFFS / CUR_CSS. */
sk_status sk_id_estimate_cols(sk_ctx* ctx, const double* X, int64_t lx, int64_t n, int64_t ldx, const int64_t* Js,
                              int64_t k, double* Z, int64_t ldz, int64_t* info);
sk_status sk_id_estimate_rows(sk_ctx* ctx, const double* Y, int64_t m, int64_t ly, int64_t ldy, const int64_t* Is,
                              int64_t k, double* W, int64_t ldw, int64_t* info);

/* ---- S1 with power iterations (Rand-LUPP-1piter) ----
 * X = Omega (A^T A)^q, the plain power-iteration row-space approximator of eq:def_power_iter
 * with Omega an l x n embedding drawn exactly like sk_sketch's Gamma but over the
 * column index of A (R1: Omega(r, j) from (seed, r, j)).  q = 0 is sk_sketch (X = Gamma A,
 * Gamma l x m).  Computed as T^T = A Omega^T, then X = T A, q - 1 times T^T = A X^T, X = T A
 * (2q passes over A, no transpose of A for the Gaussian Omega).  A m x n column-major; X l x n row-major (ldx >= n).  Requires 1 <= l <= n
 * for q >= 1, 0 <= q <= 64.  Not orthogonalised: the paper notes the plain form is unstable for
 * ill-conditioned A and q > 1. */
sk_status sk_sketch_power(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                          sk_embedding emb, int32_t zeta, uint64_t seed, int32_t q, double* X, int64_t ldx);

/* ---- the same with orthogonalisation at every iteration (eq:ortho_power_iter) ----
 *   Y_1 = A Omega^T;  Y_i = ortho(A ortho(A^T Y_{i-1})), i = 2..q;  X = ortho(Y_q)^T A
 * with Omega as for sk_sketch_power and ortho = an orthonormal basis of the range (this library's
 * LUPP basis + Cholesky QR; unique up to the signs of its columns, so X is
 * unique up to the signs of its rows, which no LUPP pivot depends on).  Stable for ill-conditioned
 * A where the plain form is not; X spans the same row space as sk_sketch_power's.
 * 2q passes over A; the Gaussian column sketch A Omega^T generates Omega per block of columns and
 * never transposes A.  Requires 1 <= q <= 64, 1 <= l <= min(m, n).  info as for sk_select_cols
 * (a rank failure of an orthogonalisation: SK_E_RANK). */
sk_status sk_sketch_power_ortho(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                                sk_embedding emb, int32_t zeta, uint64_t seed, int32_t q, double* X, int64_t ldx,
                                int64_t* info);

/* ---- S2: column skeletons by LUPP on the sketch  (eq:def_LUPP; Alg. 2 line 3) ----
 * k-step LU with partial pivoting on the n x k panel X^T(:, 0:k) = rows 0..k-1
 * of X (R5: only those rows can influence the first k pivots).  Step t picks
 * the active row j of the panel maximising |M(j, t)|, ties to the
 * lowest original index (R6), then applies the Schur-complement update.
 *   X     l x n row-major (ldx >= n); read only.  Requires 1 <= k <= l, k <= n.
 *   Js    device int64[k]: the pivots in pivot order (J_s of eq:Js).
 *   Lf    NULL or n x k column-major (ldlf >= n): Lf(i,t) = multiplier of row i
 *         at step t (|Lf| <= 1), Lf(Js[t],t) = 1, Lf(Js[t],t') = 0 for t' > t.
 *         X^T(:,0:k) = Lf U in exact arithmetic.
 *   U     NULL or k x k column-major upper triangular (ldu >= k): row t = pivot row.
 *   gaps  NULL or device double[k]: (a1 - a2)/a1 for the two largest candidate
 *         magnitudes at step t (near-tie diagnostics).
 *   info  NULL or host int64: 0, or the 1-based step of a rank failure (R7).
 *         Non-NULL info synchronises the stream and makes a rank failure
 *         return SK_E_RANK; with NULL the call is asynchronous and a rank
 *         failure leaves Js[t..k-1] = -1.
 * Panel height: up to 16384 rows run in one 16-CTA cluster; taller panels run in several
 * co-resident clusters exchanging each step's winner through global memory (on a B200 up to
 * 32 clusters of 4 CTAs, i.e. 131072 rows at 4 rows per thread; beyond that the one-cluster
 * shared-memory kernel, up to 65536 rows, else SK_E_ARG).  The bounded cross-cluster wait
 * reports SK_E_STATE (info = -step) instead of hanging if the clusters are not co-resident. */
sk_status sk_select_cols(sk_ctx* ctx, const double* X, int64_t l, int64_t n, int64_t ldx,
                         int64_t k, int64_t* Js, double* Lf, int64_t ldlf, double* U,
                         int64_t ldu, double* gaps, int64_t* info);

/* ---- S2 on a column-sharded sketch, one exchange per pivot step ----
 * The same k-step LUPP as sk_select_cols (eq:def_LUPP; R5-R7), with the n x k panel
 * M = X(0:k, :)^T split by rows over P ranks: rank r owns global rows col0 .. col0 + nloc - 1
 * (the sketch columns of its block of A).  Per step every rank proposes its best active row as a
 * RECORD of SK_LUPP_DIST_REC(k) doubles; the caller all-gathers the P records (any order) into
 * `gathered` (P x REC, contiguous) and calls sk_lupp_dist_step, which applies the merged decision
 * (max |value|, ties to the lowest GLOBAL index; rank failure below 1e-14 max|panel| over all
 * ranks) to this rank's rows and writes the next proposal.  Pivots, Lf and U equal
 * sk_select_cols on the unsharded panel.  No call synchronises or allocates, so the k-step
 * sequence (steps interleaved with the collective) can be captured in a CUDA graph.
 *   state   device buffer of sk_lupp_dist_state_bytes(nloc, k) bytes, caller-owned, holds the
 *           local panel copy; one per concurrent selection.
 *   X       rows 0..k-1 of this rank's l x nloc row-major sketch block (ldx >= nloc); read by
 *           sk_lupp_dist_begin only.  nloc may be 0 (a rank with no columns).
 *   cand    device double[REC]: this rank's proposal, written by begin (step 0) and by
 *           sk_lupp_dist_step(t) for t < k.
 *   Js      device int64[k] (replicated on every rank), written at t = 1..k; -1 from the failing
 *           step on after a rank failure.
 *   Lf      NULL or nloc x k column-major (ldlf >= nloc): this rank's rows of sk_select_cols' Lf.
 *   U       NULL or k x k column-major (ldu >= k), replicated.
 * Call begin, then for t = 1..k: all-gather(cand -> gathered), sk_lupp_dist_step(t) (world <= 64).  Then
 * sk_lupp_dist_info (synchronises) returns SK_E_RANK with *info = the failing 1-based step. */
#define SK_LUPP_DIST_REC(k) ((k) + 4)
size_t sk_lupp_dist_state_bytes(int64_t nloc, int64_t k);
sk_status sk_lupp_dist_begin(sk_ctx* ctx, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0,
                             void* state, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand);
sk_status sk_lupp_dist_step(sk_ctx* ctx, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                            const double* gathered, int32_t world, int64_t* Js, double* Lf, int64_t ldlf,
                            double* U, int64_t ldu, double* cand);
sk_status sk_lupp_dist_info(sk_ctx* ctx, const void* state, int64_t* info);

/* ---- the same LUPP with the exchange fused into the step kernel (P2P mailboxes) ----
 * Instead of an all-gather between steps, every rank owns a MAILBOX of
 * sk_lupp_dist_mailbox_bytes(k, world) bytes = [2][world][REC] doubles (records by step parity)
 * + [world] uint64 flags + 1 uint64 selection epoch, zero-initialised, mapped into every rank
 * (NVLink peer memory via sk_ipc_export / sk_ipc_import, or plain device memory when all ranks
 * share a GPU).  `peers` is a DEVICE array of world pointers, peers[q] = rank q's mailbox as seen
 * from this rank; own_mailbox = peers[rank] (host copy of the address).  begin advances the
 * mailbox's device-side epoch by k + 2 (so flags of earlier selections never satisfy a wait and a
 * captured graph of the whole selection can be replayed).  The kernel of step t waits until every
 * flag of its own mailbox reaches epoch + t, reads the records of step t-1 there, eliminates,
 * and publishes its step-t record by storing it into slot [(epoch + t) & 1][rank] of every mailbox followed
 * by a system-scope fence and flag release (epoch + t + 1).  Every rank must run the same sequence
 * of selections on its mailbox.  Same results as sk_lupp_dist_begin/step; no host call or
 * collective between steps.  The wait is bounded: if a peer's flag does not arrive within
 * SKEL_PEER_TIMEOUT_MS (environment, read once; default 30000) the kernel latches -t and the
 * remaining steps do nothing; sk_lupp_dist_info then returns SK_E_STATE with *info = -t. */
size_t sk_lupp_dist_mailbox_bytes(int64_t k, int32_t world);
sk_status sk_lupp_dist_begin_p2p(sk_ctx* ctx, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0,
                                 void* state, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand,
                                 double* const* peers, double* own_mailbox, int32_t rank, int32_t world);
sk_status sk_lupp_dist_step_p2p(sk_ctx* ctx, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                                double* const* peers, int32_t rank, int32_t world, int64_t* Js, double* Lf,
                                int64_t ldlf, double* U, int64_t ldu, double* cand);
/* Device memory shareable with other processes (cudaMalloc + zero fill, CUDA IPC): export writes a
 * 64-byte handle to host memory, import maps a peer's handle into this process (close unmaps). */
sk_status sk_ipc_alloc(sk_ctx* ctx, size_t bytes, void** ptr);
sk_status sk_ipc_free(sk_ctx* ctx, void* ptr);
sk_status sk_ipc_export(sk_ctx* ctx, void* ptr, void* handle);
sk_status sk_ipc_import(sk_ctx* ctx, const void* handle, void** ptr);
sk_status sk_ipc_close(sk_ctx* ctx, void* ptr);

/* ---- S2': column skeletons by CPQR on the sketch (eq:def_QRCP; Sec. 5 "Rand-CPQR") ----
 * k steps of Householder QR with column pivoting on all l rows of X; the pivot
 * is the active column of largest remaining norm, norms recomputed
 * exactly each step (R9), ties to the lowest index (R6).
 *   Js  device int64[k] pivots;  R  NULL or k x n column-major (ldr >= k):
 *   R(t, j) = row t of the triangular factor for ORIGINAL column j.
 *   Requires 1 <= k <= min(l, n).  info as for sk_select_cols. */
sk_status sk_select_cols_cpqr(sk_ctx* ctx, const double* X, int64_t l, int64_t n, int64_t ldx,
                              int64_t k, int64_t* Js, double* R, int64_t ldr, int64_t* info);

/* ---- RSVD-DEIM column skeletons (comparator of Sec. 5) ----
 * Q_X = ortho(X^T) (n x l), [U, S, V~] = svd(A Q_X, 'econ'), V^ = Q_X V~ (eq:rsvd_procedures,
 * P:237-243), then DEIM = column-wise LUPP on V^(:, 0:k)^T.  A m x n column-major,
 * X = Gamma A the l x n row-major sketch (ldx >= n).  Js device int64[k] in pivot order.
 * Requires 1 <= k <= l <= min(m, n).  Every step runs in this library's kernels: the l x l triangular
 * factor of A Q_X from its row LUPP and Cholesky QR (no Householder QR), its right singular vectors by
 * one-sided Jacobi in one cooperative launch.  info as sk_select_cols. */
sk_status sk_select_cols_deim(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, const double* X,
                              int64_t l, int64_t ldx, int64_t k, int64_t* Js, int64_t* info);

/* ---- S3: gather C = A(:, Js)  (eq:Js; columns in pivot order, R8) ----
 * A m x n column-major (lda >= m); Js device int64[k]; C m x k column-major (ldc >= m).
 * Js lives on the device and is not read on the host: an index outside [0, n) yields a zero
 * column of C (no out-of-bounds read).  Asynchronous on the context stream. */
sk_status sk_gather_cols(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                         const int64_t* Js, int64_t k, double* C, int64_t ldc);

/* ---- S3 on a column-sharded A ----
 * A is this rank's column block (m x ncols, columns col0 .. col0+ncols-1 of the global A).
 * C(:, t) = A(:, Js[t] - col0) for the skeletons this rank owns and 0 for the others, so a
 * sum-all-reduce over ranks assembles C = A_global(:, Js) exactly (x + 0 = x). */
sk_status sk_gather_cols_shard(sk_ctx* ctx, const double* A, int64_t m, int64_t ncols, int64_t lda, int64_t col0,
                               const int64_t* Js, int64_t k, double* C, int64_t ldc);

/* ---- S4: row skeletons by row-wise LUPP on C  (Alg. 2 line 4) ----
 * Step t scans column t of C (m x k column-major, ldc >= m); outputs as for
 * sk_select_cols with n -> m (Is = I_s of eq:Is).  Requires 1 <= k <= m. */
sk_status sk_select_rows(sk_ctx* ctx, const double* C, int64_t m, int64_t k, int64_t ldc,
                         int64_t* Is, double* Lf, int64_t ldlf, double* U, int64_t ldu,
                         double* gaps, int64_t* info);

/* ---- S5: ID coefficients  (eq:colID P:645-652; [I_k, R11^-1 R12] P:599; Thm 4.1) ----
 * Z (k x n column-major, ldz >= k): Z(:, Js) = I_k exactly; the other columns
 * T = X1^{-1} X2 = L1^{-T} L2^T with L1 = Lf(Js, :), L2 = Lf(rest, :) (R10).
 *   Lf, Js  as produced by sk_select_cols (Lf non-NULL there).
 *   eta     NULL or host double: sqrt(1 + ||T||_2^2) (Theorem 4.1 certificate);
 *           non-NULL synchronises. */
sk_status sk_id_coeffs(sk_ctx* ctx, const double* Lf, int64_t n, int64_t k, int64_t ldlf,
                       const int64_t* Js, double* Z, int64_t ldz, double* eta);

/* ---- S6: residual  (Remark 2.3 P:133-137; protocol P:554) ----
 * res_fro (host) = ||A - approx||_F for `kind`, normA_fro (host, NULL-able) = ||A||_F.
 * The m x n residual is never materialised.  Js (device int64[k]) is required
 * for COL_ID, CUR, ID_COEFFS; Is (device int64[k]) for ROW_ID and CUR; Z
 * (k x n, ldz >= k) for ID_COEFFS only.  Orthonormal bases are computed from
 * the LUPP factor of the skeleton (range(C) = range(Lf_C))
 * by two rounds of Cholesky QR.  Synchronises the stream. */
sk_status sk_residual(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda,
                      const int64_t* Js, const int64_t* Is, int64_t k, sk_residual_kind kind,
                      const double* Z, int64_t ldz, double* res_fro, double* normA_fro);

/* ---- S6 for a given skeleton matrix (column-sharded residual) ----
 * sums (host double[2]): sums[0] = ||A - Q Q^T A||_F^2, sums[1] = ||A||_F^2 with Q = ortho(C)
 * (eq:def_column_id, Frobenius R12), for A m x n column-major and C m x k column-major
 * (ldc >= m) supplied by the caller (e.g. assembled across ranks).  Squared sums, so the column
 * blocks of a sharded A add up: ||A - CC^+A||_F^2 = sum over ranks.  Synchronises.  SK_E_RANK if
 * C is numerically rank deficient. */
sk_status sk_residual_cols(sk_ctx* ctx, const double* A, int64_t m, int64_t n, int64_t lda, const double* C,
                           int64_t k, int64_t ldc, double* sums);

/* ---- Algorithm 2 end to end ---------------------------------
 * Sketch (S0+S1) + column LUPP (S2) and, if Is != NULL, gather + row LUPP
 * (S3+S4).  A may be a HOST pointer (a_on_host = 1): it is then copied to the
 * context's workspace inside the call (pinned host memory gives full PCIe
 * bandwidth) in up to 8 column blocks on the context's helper stream, each block
 * sketched as soon as it lands (X = Gamma A is column-separable), so the copy
 * overlaps the sketch.  Js / Is are HOST int64[k] outputs (Is NULL-able).  Synchronises.
 * l, emb, zeta, seed as for sk_sketch; k as for sk_select_cols. */
sk_status sk_rand_lupp(sk_ctx* ctx, const double* A, int a_on_host, int64_t m, int64_t n,
                       int64_t lda, int64_t l, sk_embedding emb, int32_t zeta, uint64_t seed,
                       int64_t k, int64_t* Js, int64_t* Is, int64_t* info);

#ifdef __cplusplus
}
#endif

#endif /* SKEL_H_ */
