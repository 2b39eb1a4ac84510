// dist.cu -- the column-sharded context (SURVEY 8(b) sk_nccl_unique_id / sk_create_dist, 8(e)).
//
// One process per GPU.  A (m x n_global) is split into contiguous column blocks; rank r holds
// columns [col0_r, col0_r + ncols_r).  The library owns the NCCL communicator (NCCL is resolved
// at run time from the process -- torch's libnccl.so.2 when torch is loaded) and every exchange
// of the path is issued here, on the context's stream:
//   sketch      X_r = Gamma A_r, no communication (Gamma(r, i) depends on the row index of A,
//               which is not sharded, so every rank regenerates the same Gamma; R1)
//   select_cols exchange 0 (default): one all-gather of the k LUPP-visible sketch rows (R5),
//               then the single-GPU cluster LUPP on identical bytes on every rank;
//               exchange 1: the panel stays sharded and every pivot step is one all-gather of
//               the ranks' candidate records (lupp_dist.cu), the begin + k (all-gather, step)
//               sequence captured once in a CUDA graph owned by the context and replayed.
//               Both equal sk_select_cols on the unsharded panel (ties to the lowest GLOBAL index).
//   gather C    each rank packs the skeleton columns it owns; one all-gather (blocks padded to the
//               largest owner count) and a gather into pivot order give C = A(:, J_s) on every rank.
//   residual    Q_C = ortho(C) by Cholesky QR distributed over row blocks of the basis (local
//               Gram, one k x k sum all-reduce per pass, replicated Cholesky, local triangular
//               solve, one all-gather of the row blocks at the end); then the local residual
//               blocks A_r - Q_C (Q_C^T A_r) and one all-reduce of (sum r^2, sum A^2).  Row ID / CUR
//               use R^T = A(I_s, :)^T, which is row-sharded exactly like A's columns, so Q_R stays
//               distributed and only k x k or m x k products are reduced.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace skel {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = nullptr;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
    return api;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.AllReduce &&
           api.GetErrorString;
  if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  return api;
}

#define SK_NCCL(ctx, expr)                                                                       \
  do {                                                                                          \
    ncclResult_t r__ = (expr);                                                                  \
    if (r__ != ncclSuccess)                                                                     \
      return ::skel::fail((ctx), SK_E_NCCL, std::string(#expr " -> ") + nccl().GetErrorString(r__)); \
  } while (0)

// The per-step exchange, captured once (begin + k x (all-gather, step)) and replayed while the
// arguments stay the same.
struct StepGraph {
  const void* key[10] = {};
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

struct DistState {
  ncclComm_t comm = nullptr;
  DistView v;
  std::vector<int64_t> col0s, ncolss;   // every rank's block
  int64_t nmax = 0;                     // the largest block
  // persistent buffers of the per-step exchange (cudaMalloc: they outlive calls and graphs)
  void* step_state = nullptr;
  size_t step_state_bytes = 0;
  double* cand = nullptr;
  double* gathered = nullptr;
  size_t cand_doubles = 0;
  StepGraph graph;
  cudaStream_t cap = nullptr;           // private stream the per-step graph is captured on (the
                                        // caller's may be the legacy default stream, not capturable)
};

bool dist_on(const sk_ctx* c) { return c && c->dist; }
DistView dist_view(const sk_ctx* c) { return c && c->dist ? c->dist->v : DistView{}; }

void dist_destroy(sk_ctx* c) {
  if (!c || !c->dist) return;
  DistState* d = c->dist;
  if (d->graph.exec) cudaGraphExecDestroy(d->graph.exec);
  if (d->step_state) cudaFree(d->step_state);
  if (d->cand) cudaFree(d->cand);
  if (d->gathered) cudaFree(d->gathered);
  if (d->cap) cudaStreamDestroy(d->cap);
  if (d->comm && nccl().ok) nccl().CommDestroy(d->comm);
  delete d;
  c->dist = nullptr;
}

sk_status dist_allreduce_sum(sk_ctx* c, double* buf, int64_t count) {
  if (count <= 0) return SK_OK;
  SK_NCCL(c, nccl().AllReduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, c->dist->comm, c->stream));
  return SK_OK;
}

sk_status dist_allgather(sk_ctx* c, const double* send, double* recv, int64_t count) {
  SK_NCCL(c, nccl().AllGather(send, recv, (size_t)count, ncclFloat64, c->dist->comm, c->stream));
  return SK_OK;
}

// ------------------------------------------------------------------------------------ S2
static sk_status select_cols_replicate(sk_ctx* c, const double* X, int64_t ldx, int64_t k, int64_t* Js, double* Lf,
                                       int64_t ldlf, double* U, int64_t ldu, double* gaps, int64_t* status_dev) {
  DistState* d = c->dist;
  const int64_t n = d->v.n_global, P = d->v.world, nm = std::max<int64_t>(d->nmax, 1);
  DBuf snd, rcv, panel, Lfull;
  SK_TRY(snd.alloc(c, (size_t)k * nm * sizeof(double)));
  SK_TRY(rcv.alloc(c, (size_t)P * k * nm * sizeof(double)));
  SK_TRY(panel.alloc(c, (size_t)k * n * sizeof(double)));
  if (d->v.ncols > 0)
    SK_CUDA(c, cudaMemcpy2DAsync(snd.p, (size_t)nm * sizeof(double), X, (size_t)ldx * sizeof(double),
                                 (size_t)d->v.ncols * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  SK_TRY(dist_allgather(c, snd.as<double>(), rcv.as<double>(), k * nm));
  for (int64_t r = 0; r < P; ++r)       // rank blocks -> the k x n_global row-major panel
    if (d->ncolss[r] > 0)
      SK_CUDA(c, cudaMemcpy2DAsync(panel.as<double>() + d->col0s[r], (size_t)n * sizeof(double),
                                   rcv.as<double>() + r * k * nm, (size_t)nm * sizeof(double),
                                   (size_t)d->ncolss[r] * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  rcv.release();
  snd.release();
  SK_TRY(Lfull.alloc(c, (size_t)n * k * sizeof(double)));
  SK_TRY(lupp(c, panel.as<double>(), true, n, k, n, Js, Lfull.as<double>(), n, U, ldu, gaps, status_dev));
  if (Lf && d->v.ncols > 0)             // this rank's rows of the replicated factor
    SK_CUDA(c, cudaMemcpy2DAsync(Lf, (size_t)ldlf * sizeof(double), Lfull.as<double>() + d->v.col0, (size_t)n * sizeof(double),
                                 (size_t)d->v.ncols * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  return SK_OK;
}

static sk_status select_cols_step(sk_ctx* c, const double* X, int64_t ldx, int64_t k, int64_t* Js, double* Lf,
                                  int64_t ldlf, double* U, int64_t ldu, int64_t* status_dev) {
  DistState* d = c->dist;
  const int64_t nloc = d->v.ncols, REC = k + 4;
  const size_t sb = lupp_dist_state_bytes(nloc, k);
  if (sb > d->step_state_bytes || (size_t)(d->v.world * REC) > d->cand_doubles) {
    if (d->graph.exec) { cudaGraphExecDestroy(d->graph.exec); d->graph.exec = nullptr; }
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    if (d->step_state) cudaFree(d->step_state);
    if (d->cand) cudaFree(d->cand);
    if (d->gathered) cudaFree(d->gathered);
    d->step_state = nullptr; d->cand = d->gathered = nullptr;
    SK_CUDA(c, cudaMalloc(&d->step_state, sb));
    SK_CUDA(c, cudaMalloc(&d->cand, (size_t)d->v.world * REC * sizeof(double)));
    SK_CUDA(c, cudaMalloc(&d->gathered, (size_t)d->v.world * REC * sizeof(double)));
    d->step_state_bytes = sb;
    d->cand_doubles = (size_t)d->v.world * REC;
  }
  const void* key[10] = {X, (const void*)ldx, (const void*)k, Js, Lf, (const void*)ldlf, U, (const void*)ldu,
                         c->stream, d->step_state};
  if (!d->graph.exec || std::memcmp(key, d->graph.key, sizeof(key)) != 0) {
    if (d->graph.exec) { cudaGraphExecDestroy(d->graph.exec); d->graph.exec = nullptr; }
    const int64_t l0 = c->launches;
    if (!d->cap) SK_CUDA(c, cudaStreamCreateWithFlags(&d->cap, cudaStreamNonBlocking));
    cudaStream_t user = c->stream;
    c->stream = d->cap;                 // every launch below records into the graph
    sk_status st = SK_OK;
    if (cudaStreamBeginCapture(d->cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      c->stream = user;
      return fail(c, SK_E_CUDA, "capture of the per-step LUPP: cudaStreamBeginCapture failed");
    }
    st = lupp_dist_begin(c, X, nloc, ldx, k, d->v.col0, d->step_state, Lf, ldlf, U, ldu, d->cand);
    for (int64_t t = 1; t <= k && st == SK_OK; ++t) {
      const ncclResult_t r = nccl().AllGather(d->cand, d->gathered, (size_t)REC, ncclFloat64, d->comm, c->stream);
      if (r != ncclSuccess) { st = fail(c, SK_E_NCCL, std::string("ncclAllGather: ") + nccl().GetErrorString(r)); break; }
      st = lupp_dist_step(c, d->step_state, nloc, k, d->v.col0, t, d->gathered, d->v.world, Js, Lf, ldlf, U, ldu, d->cand);
    }
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(d->cap, &g);
    c->stream = user;
    if (st != SK_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (ce != cudaSuccess) return fail(c, SK_E_CUDA, std::string("capture of the per-step LUPP: ") + cudaGetErrorString(ce));
    const cudaError_t ie = cudaGraphInstantiate(&d->graph.exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(c, SK_E_CUDA, std::string("instantiate: ") + cudaGetErrorString(ie));
    std::memcpy(d->graph.key, key, sizeof(key));
    d->graph.kernels = c->launches - l0;
    c->launches = l0;
  }
  SK_CUDA(c, cudaGraphLaunch(d->graph.exec, c->stream));
  c->launches += d->graph.kernels;
  return lupp_dist_status(c, d->step_state, status_dev);
}

sk_status dist_select_cols(sk_ctx* c, const double* X, int64_t ncols, int64_t ldx, int64_t k, int64_t* Js, double* Lf,
                           int64_t ldlf, double* U, int64_t ldu, double* gaps, int64_t* status_dev) {
  (void)ncols;
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  if (c->dist->v.exchange == 1 && !gaps)
    return select_cols_step(c, X, ldx, k, Js, Lf, ldlf, U, ldu, status_dev);
  return select_cols_replicate(c, X, ldx, k, Js, Lf, ldlf, U, ldu, gaps, status_dev);
}

// ------------------------------------------------------------------------------------ S3
sk_status dist_gather_cols(sk_ctx* c, const double* A, bool a_on_host, int64_t m, int64_t lda, const int64_t* Js,
                           int64_t k, double* C, int64_t ldc) {
  DistState* d = c->dist;
  const int P = d->v.world;
  std::vector<int64_t> J(k);
  SK_CUDA(c, cudaMemcpyAsync(J.data(), Js, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  std::vector<int64_t> cnt(P, 0), own, perm(k);
  std::vector<int> owner(k, -1);
  for (int64_t t = 0; t < k; ++t)
    for (int r = 0; r < P; ++r)
      if (J[t] >= d->col0s[r] && J[t] < d->col0s[r] + d->ncolss[r]) { owner[t] = r; break; }
  int64_t cmax = 1;
  for (int64_t t = 0; t < k; ++t)
    if (owner[t] >= 0) cmax = std::max(cmax, ++cnt[owner[t]]);
  std::fill(cnt.begin(), cnt.end(), 0);
  for (int64_t t = 0; t < k; ++t) {
    const int r = owner[t];
    if (r < 0) { perm[t] = -1; continue; }             // invalid index (rank failure): zero column
    perm[t] = r * cmax + cnt[r]++;
    if (r == d->v.rank) own.push_back(J[t] - d->v.col0);
  }
  DBuf snd, rcv, idx;
  SK_TRY(snd.alloc(c, (size_t)m * cmax * sizeof(double)));
  SK_TRY(rcv.alloc(c, (size_t)P * m * cmax * sizeof(double)));
  SK_TRY(idx.alloc(c, (size_t)(k + own.size() + 1) * sizeof(int64_t)));
  if (!own.empty()) {
    if (a_on_host) {
      for (size_t i = 0; i < own.size(); ++i)
        SK_CUDA(c, cudaMemcpyAsync(snd.as<double>() + i * m, A + own[i] * lda, (size_t)m * sizeof(double),
                                   cudaMemcpyHostToDevice, c->stream));
    } else {
      SK_CUDA(c, cudaMemcpyAsync(idx.as<int64_t>() + k, own.data(), own.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                                 c->stream));
      SK_TRY(gather_cols_shard(c, A, m, lda, 0, d->v.ncols, idx.as<int64_t>() + k, (int64_t)own.size(), snd.as<double>(), m));
    }
  }
  SK_CUDA(c, cudaMemcpyAsync(idx.p, perm.data(), (size_t)k * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  SK_TRY(dist_allgather(c, snd.as<double>(), rcv.as<double>(), m * cmax));
  SK_TRY(gather_cols_shard(c, rcv.as<double>(), m, m, 0, (int64_t)P * cmax, idx.as<int64_t>(), k, C, ldc));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));        // the host index vectors go out of scope
  return SK_OK;
}

// ------------------------------------------------------------------------------------ S6
// Cholesky QR of the replicated basis B (m x k) distributed over row blocks: rank r owns rows
// [r mb, (r+1) mb) (mb = ceil(m / P)); per pass a local Gram matrix, one k x k sum all-reduce, the
// (replicated, identical) Cholesky factor and the local right triangular solve; the first pass
// shifted for a basis that is not well conditioned (shifted CholeskyQR3).  Q (m x k, ld m) is
// replicated at the end by one all-gather of the row blocks.
static sk_status dist_cholqr(sk_ctx* c, const double* B, int64_t m, int64_t k, int passes, bool shift, double* Q,
                             int64_t* status_dev) {
  const int P = c->dist->v.world, me = c->dist->v.rank;
  const int64_t mb = cdiv(m, P);
  const int64_t r0 = std::min<int64_t>(m, me * mb), rows = std::min<int64_t>(mb, m - r0);
  DBuf Bl, G, rcv;
  SK_TRY(Bl.alloc(c, (size_t)mb * k * sizeof(double)));
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  SK_CUDA(c, cudaMemsetAsync(Bl.p, 0, (size_t)mb * k * sizeof(double), c->stream));   // padded rows stay 0
  if (rows > 0)
    SK_CUDA(c, cudaMemcpy2DAsync(Bl.p, (size_t)mb * sizeof(double), B + r0, (size_t)m * sizeof(double),
                                 (size_t)rows * sizeof(double), (size_t)k, cudaMemcpyDeviceToDevice, c->stream));
  for (int pass = 0; pass < passes; ++pass) {
    SK_TRY(gemm(c, true, false, k, k, mb, 1.0, Bl.as<double>(), mb, Bl.as<double>(), mb, 0.0, G.as<double>(), k));
    SK_TRY(dist_allreduce_sum(c, G.as<double>(), k * k));
    if (shift && pass == 0) SK_TRY(add_shift(c, G.as<double>(), k, k, m));
    SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
    SK_TRY(trsm_right_lt(c, Bl.as<double>(), mb, k, mb, G.as<double>(), k));
  }
  SK_TRY(rcv.alloc(c, (size_t)P * mb * k * sizeof(double)));
  SK_TRY(dist_allgather(c, Bl.as<double>(), rcv.as<double>(), mb * k));
  for (int r = 0; r < P; ++r) {
    const int64_t q0 = std::min<int64_t>(m, r * mb), qr = std::min<int64_t>(mb, m - q0);
    if (qr > 0)
      SK_CUDA(c, cudaMemcpy2DAsync(Q + q0, (size_t)m * sizeof(double), rcv.as<double>() + r * mb * k,
                                   (size_t)mb * sizeof(double), (size_t)qr * sizeof(double), (size_t)k,
                                   cudaMemcpyDeviceToDevice, c->stream));
  }
  return SK_OK;
}

// Cholesky QR of a basis whose rows are ALREADY sharded (R^T: row j = column j of A, owned by the
// rank owning that column): in place on the local rows, nothing gathered (shifted CholeskyQR3).
static sk_status dist_cholqr_local(sk_ctx* c, double* Bl, int64_t rows, int64_t rows_total, int64_t k,
                                   int64_t* status_dev) {
  DBuf G;
  SK_TRY(G.alloc(c, (size_t)k * k * sizeof(double)));
  for (int pass = 0; pass < 3; ++pass) {
    if (rows > 0) SK_TRY(gemm(c, true, false, k, k, rows, 1.0, Bl, rows, Bl, rows, 0.0, G.as<double>(), k));
    else SK_CUDA(c, cudaMemsetAsync(G.p, 0, (size_t)k * k * sizeof(double), c->stream));
    SK_TRY(dist_allreduce_sum(c, G.as<double>(), k * k));
    if (pass == 0) SK_TRY(add_shift(c, G.as<double>(), k, k, rows_total));
    SK_TRY(potrf_lower(c, G.as<double>(), k, k, status_dev));
    if (rows > 0) SK_TRY(trsm_right_lt(c, Bl, rows, k, rows, G.as<double>(), k));
  }
  return SK_OK;
}

// Q_C = ortho(C) for the replicated C: the LUPP basis (range(C) = range(Lf_C), |Lf_C| <= 1, as on one
// GPU) + distributed CholeskyQR2 when C's row LUPP fits the cluster kernel, else distributed
// shifted CholeskyQR3 on C itself (R20).
static sk_status dist_basis_c(sk_ctx* c, const double* C, int64_t m, int64_t k, double* Q, int64_t* status_dev) {
  if (m <= 65536) {
    DBuf Lb, piv;
    SK_TRY(Lb.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(piv.alloc(c, (size_t)k * sizeof(int64_t)));
    SK_TRY(lupp(c, C, false, m, k, m, piv.as<int64_t>(), Lb.as<double>(), m, nullptr, 0, nullptr, status_dev));
    return dist_cholqr(c, Lb.as<double>(), m, k, 2, false, Q, status_dev);
  }
  return dist_cholqr(c, C, m, k, 3, true, Q, status_dev);
}

sk_status dist_residual(sk_ctx* c, const double* A, int64_t m, int64_t lda, const int64_t* Js, const int64_t* Is,
                        int64_t k, int kind, const double* Z, int64_t ldz, double* sums, int64_t* status_dev) {
  const DistView v = c->dist->v;
  const int64_t n = v.ncols;
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  SK_CUDA(c, cudaMemsetAsync(sums, 0, 2 * sizeof(double), c->stream));
  DBuf C, Qc, Qr, W, Mid, Bm;
  if (kind != SK_RES_ROW_ID) {
    SK_TRY(C.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(dist_gather_cols(c, A, false, m, lda, Js, k, C.as<double>(), m));
  }
  if (kind == SK_RES_ID_COEFFS) {
    if (n > 0) SK_TRY(lowrank_sumsq(c, C.as<double>(), m, Z, ldz, nullptr, 0, A, lda, m, n, k, sums));
    return dist_allreduce_sum(c, sums, 2);
  }
  if (kind == SK_RES_COL_ID || kind == SK_RES_CUR) {
    SK_TRY(Qc.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(dist_basis_c(c, C.as<double>(), m, k, Qc.as<double>(), status_dev));
    C.release();
  }
  if (kind == SK_RES_ROW_ID || kind == SK_RES_CUR) {   // Q_R: rows of R^T live with this rank's columns
    SK_TRY(Qr.alloc(c, (size_t)std::max<int64_t>(n, 1) * k * sizeof(double)));
    if (n > 0) SK_TRY(gather_rows_t(c, A, m, n, lda, Is, k, Qr.as<double>(), n));
    SK_TRY(dist_cholqr_local(c, Qr.as<double>(), n, v.n_global, k, status_dev));
  }
  if (kind == SK_RES_COL_ID) {
    if (n > 0) SK_TRY(col_id_sumsq(c, Qc.as<double>(), A, m, n, lda, k, sums));
    return dist_allreduce_sum(c, sums, 2);
  }
  if (kind == SK_RES_ROW_ID) {   // A Q_R = sum_r A_r Q_R,r (m x k, one all-reduce), then local blocks
    SK_TRY(W.alloc(c, (size_t)m * k * sizeof(double)));
    if (n > 0) SK_TRY(gemm(c, false, false, m, k, n, 1.0, A, lda, Qr.as<double>(), n, 0.0, W.as<double>(), m));
    else SK_CUDA(c, cudaMemsetAsync(W.p, 0, (size_t)m * k * sizeof(double), c->stream));
    SK_TRY(dist_allreduce_sum(c, W.as<double>(), m * k));
    if (n > 0) SK_TRY(lowrank_sumsq(c, W.as<double>(), m, nullptr, 0, Qr.as<double>(), n, A, lda, m, n, k, sums));
    return dist_allreduce_sum(c, sums, 2);
  }
  // CUR: Mid = Q_C^T A Q_R = sum_r (Q_C^T A_r) Q_R,r (k x k, one all-reduce); residual A_r - (Q_C Mid) Q_R,r^T
  SK_TRY(Mid.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(Bm.alloc(c, (size_t)m * k * sizeof(double)));
  if (n > 0) {
    SK_TRY(W.alloc(c, (size_t)k * n * sizeof(double)));
    SK_TRY(gemm_qta(c, Qc.as<double>(), m, A, m, n, lda, k, W.as<double>(), n));                 // W^T, n x k
    SK_TRY(gemm(c, true, false, k, k, n, 1.0, W.as<double>(), n, Qr.as<double>(), n, 0.0, Mid.as<double>(), k));
  } else {
    SK_CUDA(c, cudaMemsetAsync(Mid.p, 0, (size_t)k * k * sizeof(double), c->stream));
  }
  SK_TRY(dist_allreduce_sum(c, Mid.as<double>(), k * k));
  SK_TRY(gemm(c, false, false, m, k, k, 1.0, Qc.as<double>(), m, Mid.as<double>(), k, 0.0, Bm.as<double>(), m));
  if (n > 0) SK_TRY(lowrank_sumsq(c, Bm.as<double>(), m, nullptr, 0, Qr.as<double>(), n, A, lda, m, n, k, sums));
  return dist_allreduce_sum(c, sums, 2);
}

}  // namespace skel

using namespace skel;

extern "C" {

sk_status sk_nccl_unique_id(void* out) {
  if (!out) return SK_E_ARG;
  if (!nccl().ok) return SK_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return SK_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return SK_OK;
}

sk_status sk_create_dist(sk_ctx** out, int device, void* stream, const void* uid, int rank, int world, int64_t n_global,
                         int64_t col0, int64_t ncols) {
  if (!out || !uid || world < 1 || rank < 0 || rank >= world || n_global < 1 || col0 < 0 || ncols < 0 ||
      col0 + ncols > n_global)
    return SK_E_ARG;
  *out = nullptr;
  if (!nccl().ok) return SK_E_NCCL;
  sk_ctx* c = nullptr;
  sk_status st = sk_create(&c, device, stream);
  if (st != SK_OK) return st;
  DistState* d = new DistState();
  d->v.rank = rank; d->v.world = world; d->v.n_global = n_global; d->v.col0 = col0; d->v.ncols = ncols;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  if (nccl().CommInitRank(&d->comm, world, id, rank) != ncclSuccess) {
    delete d;
    sk_destroy(c);
    return SK_E_NCCL;
  }
  c->dist = d;
  // every rank's block: one all-gather of (col0, ncols)
  int64_t* buf = nullptr;
  st = SK_OK;
  if (cudaMalloc(&buf, (size_t)(2 + 2 * world) * sizeof(int64_t)) != cudaSuccess) st = SK_E_NOMEM;
  std::vector<int64_t> h(2 * world);
  const int64_t mine[2] = {col0, ncols};
  if (st == SK_OK && cudaMemcpyAsync(buf, mine, sizeof(mine), cudaMemcpyHostToDevice, c->stream) != cudaSuccess) st = SK_E_CUDA;
  if (st == SK_OK && nccl().AllGather(buf, buf + 2, 2, ncclInt64, d->comm, c->stream) != ncclSuccess) st = SK_E_NCCL;
  if (st == SK_OK && cudaMemcpyAsync(h.data(), buf + 2, h.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess)
    st = SK_E_CUDA;
  if (st == SK_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) st = SK_E_CUDA;
  if (buf) cudaFree(buf);
  if (st == SK_OK) {
    int64_t next = 0;
    for (int r = 0; r < world; ++r) {
      d->col0s.push_back(h[2 * r]);
      d->ncolss.push_back(h[2 * r + 1]);
      d->nmax = std::max(d->nmax, h[2 * r + 1]);
      if (h[2 * r] != next) st = SK_E_ARG;                // blocks must be contiguous, in rank order
      next = h[2 * r] + h[2 * r + 1];
    }
    if (next != n_global) st = SK_E_ARG;
  }
  if (st != SK_OK) {
    sk_destroy(c);
    return st;
  }
  *out = c;
  return SK_OK;
}

sk_status sk_set_dist_exchange(sk_ctx* c, int32_t exchange) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, c->dist, "sk_set_dist_exchange: not a distributed context (sk_create_dist)");
  SK_ARG(c, exchange == 0 || exchange == 1, "sk_set_dist_exchange: exchange must be 0 (replicate) or 1 (per step)");
  c->dist->v.exchange = exchange;
  return SK_OK;
}

sk_status sk_dist_info(const sk_ctx* c, int32_t* rank, int32_t* world, int64_t* n_global, int64_t* col0, int64_t* ncols) {
  if (!c) return SK_E_ARG;
  const DistView v = dist_view(c);
  if (rank) *rank = v.rank;
  if (world) *world = c->dist ? v.world : 1;
  if (n_global) *n_global = v.n_global;
  if (col0) *col0 = v.col0;
  if (ncols) *ncols = v.ncols;
  return SK_OK;
}

}  // extern "C"
