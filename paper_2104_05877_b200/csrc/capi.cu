// capi.cu -- the extern "C" entry points of libskel.so (include/skel.h).
// Argument validation happens here, before anything is enqueued; the work is done by
// the kernels in sketch.cu, lupp.cu, cpqr.cu, dense.cu, idcoef.cu, residual.cu.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>

#include "common.cuh"
#include "internal.h"

using namespace skel;

namespace {

// Copy n device int64/double values to host (pinned scratch) and synchronise.
sk_status to_host(sk_ctx* c, void* dst, const void* src_dev, size_t bytes) {
  if (bytes > 4096) {
    SK_CUDA(c, cudaMemcpyAsync(dst, src_dev, bytes, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(c, cudaStreamSynchronize(c->stream));
    return SK_OK;
  }
  SK_CUDA(c, cudaMemcpyAsync(c->host_scratch, src_dev, bytes, cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(c, cudaStreamSynchronize(c->stream));
  std::memcpy(dst, c->host_scratch, bytes);
  return SK_OK;
}

sk_status finish_info(sk_ctx* c, const int64_t* status_dev, int64_t* info, const char* what) {
  if (!info) return SK_OK;
  int64_t st = 0;
  SK_TRY(to_host(c, &st, status_dev, sizeof(int64_t)));
  *info = st;
  if (st < 0)   // a bounded device-side wait gave up (multi-cluster LUPP exchange): a launch problem, not data
    return fail(c, SK_E_STATE, std::string(what) + ": cross-cluster exchange timed out at step " + std::to_string(-st));
  if (st != 0)
    return fail(c, SK_E_RANK, std::string(what) + ": rank deficiency at step " + std::to_string(st));
  return SK_OK;
}

}  // namespace

namespace skel {

sk_status for_host_blocks(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda,
                          const std::function<sk_status(const double*, int64_t, int64_t)>& fn) {
  // A ring of NR device slots of W columns (<= 2 GB each), not the whole of A: the host->device copy
  // of block b (helper stream) overlaps the work on block b - 1 (context stream); a slot is refilled
  // only after the work that read it is done.
  constexpr int NR = 3;
  const int64_t wmax = std::max<int64_t>(128, ((int64_t)(2.0 * (1 << 30) / (8.0 * (double)m)) / 128) * 128);
  const int64_t W = std::min(wmax, std::max<int64_t>(128, cdiv(cdiv(n, 8), 128) * 128));
  const int64_t nb = cdiv(n, W);
  const int nr = (int)std::min<int64_t>(NR, nb);
  if (nb == 0) return SK_OK;
  DBuf slot[NR];
  for (int r = 0; r < nr; ++r) SK_TRY(slot[r].alloc(c, (size_t)m * W * sizeof(double)));
  SK_TRY(ensure_aux(c));
  cudaEvent_t ev[2 * NR + 1] = {};
  sk_status rs = SK_OK;
  for (int e = 0; e < 2 * nr + 1 && rs == SK_OK; ++e)
    if (cudaEventCreateWithFlags(&ev[e], cudaEventDisableTiming) != cudaSuccess) rs = fail(c, SK_E_CUDA, "host stream: event");
  cudaEvent_t* copied = ev;            // [nr]: block in slot r has landed
  cudaEvent_t* consumed = ev + nr;     // [nr]: the work on the block in slot r is done
  if (rs == SK_OK && (cudaEventRecord(ev[2 * nr], c->stream) != cudaSuccess ||      // slots allocated (stream order)
                      cudaStreamWaitEvent(c->aux, ev[2 * nr], 0) != cudaSuccess))
    rs = fail(c, SK_E_CUDA, "host stream: event");
  for (int64_t b = 0; b < nb && rs == SK_OK; ++b) {
    const int r = (int)(b % nr);
    const int64_t j0 = b * W, jw = std::min(W, n - j0);
    double* dst = slot[r].as<double>();
    if (b >= nr && cudaStreamWaitEvent(c->aux, consumed[r], 0) != cudaSuccess) { rs = fail(c, SK_E_CUDA, "host stream: event"); break; }
    if (cudaMemcpy2DAsync(dst, (size_t)m * sizeof(double), A + j0 * lda, (size_t)lda * sizeof(double),
                          (size_t)m * sizeof(double), (size_t)jw, cudaMemcpyHostToDevice, c->aux) != cudaSuccess ||
        cudaEventRecord(copied[r], c->aux) != cudaSuccess || cudaStreamWaitEvent(c->stream, copied[r], 0) != cudaSuccess) {
      rs = fail(c, SK_E_CUDA, "host stream: host-to-device copy");
      break;
    }
    rs = fn(dst, j0, jw);
    if (rs == SK_OK && cudaEventRecord(consumed[r], c->stream) != cudaSuccess) rs = fail(c, SK_E_CUDA, "host stream: event");
  }
  // (every copy was waited for by the context stream, so the slots are freed after their last use)
  for (int e = 0; e < 2 * nr + 1; ++e)
    if (ev[e]) cudaEventDestroy(ev[e]);
  return rs;
}

}  // namespace skel

extern "C" {

sk_status sk_create(sk_ctx** out, int device, void* stream) {
  if (!out) return SK_E_ARG;
  *out = nullptr;
  sk_ctx* c = new (std::nothrow) sk_ctx();
  if (!c) return SK_E_NOMEM;
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&c->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e == cudaSuccess) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    if (major != 10 || minor != 0) {
      c->err = "libskel.so is built for sm_100a (B200) only";
      delete c;
      return SK_E_CUDA;
    }
  }
  if (e == cudaSuccess) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    e = cudaMemPoolCreate(&c->pool, &props);
    if (e == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      e = cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  if (e == cudaSuccess) e = cudaMallocHost(&c->host_scratch, 4096);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (c->pool) cudaMemPoolDestroy(c->pool);
    delete c;
    return SK_E_CUDA;
  }
  *out = c;
  return SK_OK;
}

sk_status sk_set_sketch_tuning(sk_ctx* c, int32_t path, int32_t bm, int32_t warps, int32_t splits, int64_t chunk_rows) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, path >= 0 && path <= 3, "sk_set_sketch_tuning: path must be 0..3");
  SK_ARG(c, bm == 0 || bm == 32 || bm == 40 || bm == 48 || bm == 56 || bm == 64 || bm == 80 || bm == 96,
         "sk_set_sketch_tuning: bm must be 0, 32, 40, 48, 56, 64, 80 or 96");
  SK_ARG(c, warps == 0 || warps == 2 || warps == 4 || warps == 7 || warps == 8 || warps == 12,
         "sk_set_sketch_tuning: warps must be 0, 2, 4, 7, 8 or 12");
  SK_ARG(c, splits >= 0 && splits <= 64 && chunk_rows >= 0, "sk_set_sketch_tuning: bad splits / chunk_rows");
  c->tune_sketch_path = path;
  c->tune_sketch_bm = bm;
  c->tune_sketch_nw = warps;
  c->tune_sketch_splits = splits;
  c->tune_sketch_chunk = chunk_rows;
  return SK_OK;
}

sk_status sk_set_stream(sk_ctx* c, void* stream) {
  if (!c) return SK_E_ARG;
  c->stream = static_cast<cudaStream_t>(stream);
  return SK_OK;
}

void sk_destroy(sk_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->stream);
  dist_destroy(c);
  if (c->aux) { cudaStreamSynchronize(c->aux); cudaStreamDestroy(c->aux); }
  if (c->img) { cudaStreamSynchronize(c->img); cudaStreamDestroy(c->img); }
  if (c->ev_a) cudaEventDestroy(c->ev_a);
  if (c->ev_b) cudaEventDestroy(c->ev_b);
  if (c->pool) cudaMemPoolDestroy(c->pool);
  if (c->host_scratch) cudaFreeHost(c->host_scratch);
  delete c;
}

const char* sk_last_error(const sk_ctx* c) { return c ? c->err.c_str() : "null context"; }

const char* sk_version(void) { return "skel 0.1 sm_100a"; }

int64_t sk_workspace_bytes(const sk_ctx* c) {
  if (!c || !c->pool) return 0;
  uint64_t v = 0;
  cudaMemPoolGetAttribute(c->pool, cudaMemPoolAttrReservedMemCurrent, &v);
  return (int64_t)v;
}

int64_t sk_launch_count(const sk_ctx* c) { return c ? c->launches : 0; }

sk_status sk_sketch(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                    sk_embedding emb, int32_t zeta, uint64_t seed, double* X, int64_t ldx) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, n == 0 || (A && X), "sk_sketch: NULL A or X");
  SK_ARG(c, m >= 1 && n >= 0 && l >= 1 && l <= m, "sk_sketch: need 1 <= l <= m, n >= 0");
  SK_ARG(c, lda >= m && ldx >= n, "sk_sketch: lda >= m and ldx >= n required");
  SK_ARG(c, m < (1LL << 40) && l <= (1 << 20), "sk_sketch: size out of range");
  SK_CUDA(c, cudaSetDevice(c->device));
  if (emb == SK_EMB_GAUSSIAN) return sketch_dense(c, A, m, n, lda, l, seed, X, ldx);
  if (emb == SK_EMB_SPARSE_SIGN) {
    SK_ARG(c, zeta >= 2 && zeta <= l && zeta <= 64, "sk_sketch: sparse sign needs 2 <= zeta <= min(l, 64)");
    return sketch_sparse(c, A, m, n, lda, l, zeta, seed, X, ldx);
  }
  if (emb == SK_EMB_SRTT) return sketch_srtt(c, A, m, n, lda, l, seed, X, ldx);
  return fail(c, SK_E_ARG, "sk_sketch: unknown embedding");
}

sk_status sk_sketch_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                         sk_embedding emb, int32_t zeta, uint64_t seed, double* Y, int64_t ldy) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && Y, "sk_sketch_cols: NULL A or Y");
  SK_ARG(c, m >= 1 && n >= 1 && l >= 1 && l <= n, "sk_sketch_cols: need 1 <= l <= n, m >= 1");
  SK_ARG(c, lda >= m && ldy >= m, "sk_sketch_cols: lda >= m and ldy >= m required");
  SK_ARG(c, emb >= SK_EMB_GAUSSIAN && emb <= SK_EMB_SRTT, "sk_sketch_cols: unknown embedding");
  SK_ARG(c, emb != SK_EMB_SPARSE_SIGN || (zeta >= 2 && zeta <= l && zeta <= 64), "sk_sketch_cols: bad zeta");
  SK_CUDA(c, cudaSetDevice(c->device));
  return sketch_cols(c, A, m, n, lda, l, (int)emb, zeta, seed, Y, ldy);
}

sk_status sk_sketch_power(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                          sk_embedding emb, int32_t zeta, uint64_t seed, int32_t q, double* X, int64_t ldx) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && X, "sk_sketch_power: NULL A or X");
  SK_ARG(c, q >= 0 && q <= 64, "sk_sketch_power: 0 <= q <= 64");
  if (q == 0) return sk_sketch(c, A, m, n, lda, l, emb, zeta, seed, X, ldx);
  SK_ARG(c, m >= 1 && n >= 1 && l >= 1 && l <= n, "sk_sketch_power: need 1 <= l <= n, m >= 1");
  SK_ARG(c, lda >= m && ldx >= n, "sk_sketch_power: lda >= m and ldx >= n required");
  SK_ARG(c, emb >= SK_EMB_GAUSSIAN && emb <= SK_EMB_SRTT, "sk_sketch_power: unknown embedding");
  SK_ARG(c, emb != SK_EMB_SPARSE_SIGN || (zeta >= 2 && zeta <= l && zeta <= 64), "sk_sketch_power: bad zeta");
  SK_CUDA(c, cudaSetDevice(c->device));
  return sketch_power(c, A, m, n, lda, l, (int)emb, zeta, seed, q, X, ldx);
}

sk_status sk_sketch_power_ortho(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, int64_t l,
                                sk_embedding emb, int32_t zeta, uint64_t seed, int32_t q, double* X, int64_t ldx,
                                int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && X, "sk_sketch_power_ortho: NULL A or X");
  SK_ARG(c, q >= 1 && q <= 64, "sk_sketch_power_ortho: 1 <= q <= 64");
  SK_ARG(c, m >= 1 && n >= 1 && l >= 1 && l <= n && l <= m, "sk_sketch_power_ortho: need 1 <= l <= min(m, n)");
  SK_ARG(c, lda >= m && ldx >= n, "sk_sketch_power_ortho: lda >= m and ldx >= n required");
  SK_ARG(c, emb >= SK_EMB_GAUSSIAN && emb <= SK_EMB_SRTT, "sk_sketch_power_ortho: unknown embedding");
  SK_ARG(c, emb != SK_EMB_SPARSE_SIGN || (zeta >= 2 && zeta <= l && zeta <= 64), "sk_sketch_power_ortho: bad zeta");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(sketch_power_ortho(c, A, m, n, lda, l, (int)emb, zeta, seed, q, X, ldx, st.as<int64_t>()));
  return finish_info(c, st.as<int64_t>(), info, "sk_sketch_power_ortho (orthogonalisation)");
}

sk_status sk_select_cols(sk_ctx* c, const double* X, int64_t l, int64_t n, int64_t ldx, int64_t k,
                         int64_t* Js, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* gaps,
                         int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, X && Js, "sk_select_cols: NULL X or Js");
  SK_ARG(c, !Lf || ldlf >= n, "sk_select_cols: ldlf >= n required");
  SK_ARG(c, !U || ldu >= k, "sk_select_cols: ldu >= k required");
  if (dist_on(c)) {   // X is this rank's l x ncols block; Js / U / gaps replicated, Lf this rank's rows
    const DistView v = dist_view(c);
    SK_ARG(c, n == v.ncols && ldx >= std::max<int64_t>(n, 1) && k >= 1 && k <= l && k <= v.n_global,
           "sk_select_cols (distributed): n must be this rank's ncols, 1 <= k <= min(l, n_global)");
    SK_CUDA(c, cudaSetDevice(c->device));
    DBuf st;
    SK_TRY(st.alloc(c, sizeof(int64_t)));
    SK_TRY(dist_select_cols(c, X, n, ldx, k, Js, Lf, ldlf, U, ldu, gaps, st.as<int64_t>()));
    return finish_info(c, st.as<int64_t>(), info, "sk_select_cols (distributed)");
  }
  SK_ARG(c, k >= 1 && k <= l && k <= n && ldx >= n, "sk_select_cols: need 1 <= k <= min(l, n), ldx >= n");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(lupp(c, X, true, n, k, ldx, Js, Lf, ldlf, U, ldu, gaps, st.as<int64_t>()));
  return finish_info(c, st.as<int64_t>(), info, "sk_select_cols");
}

sk_status sk_select_cols_cpqr(sk_ctx* c, const double* X, int64_t l, int64_t n, int64_t ldx, int64_t k,
                              int64_t* Js, double* R, int64_t ldr, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, X && Js, "sk_select_cols_cpqr: NULL X or Js");
  SK_ARG(c, k >= 1 && k <= l && k <= n && ldx >= n, "sk_select_cols_cpqr: need 1 <= k <= min(l, n)");
  SK_ARG(c, !R || ldr >= k, "sk_select_cols_cpqr: ldr >= k required");
  SK_ARG(c, l <= 8192, "sk_select_cols_cpqr: l <= 8192");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(cpqr(c, X, l, n, ldx, k, Js, R, ldr, st.as<int64_t>()));
  return finish_info(c, st.as<int64_t>(), info, "sk_select_cols_cpqr");
}

sk_status sk_select_cols_deim(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* X,
                              int64_t l, int64_t ldx, int64_t k, int64_t* Js, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && X && Js, "sk_select_cols_deim: NULL pointer");
  SK_ARG(c, k >= 1 && k <= l && l <= m && l <= n && lda >= m && ldx >= n,
         "sk_select_cols_deim: need 1 <= k <= l <= min(m, n), lda >= m, ldx >= n");
  SK_ARG(c, m < (1LL << 31) && n < (1LL << 31), "sk_select_cols_deim: size out of range");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(select_cols_deim(c, A, m, n, lda, X, l, ldx, k, Js, st.as<int64_t>()));
  return finish_info(c, st.as<int64_t>(), info, "sk_select_cols_deim");
}

sk_status sk_gather_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* Js,
                         int64_t k, double* C, int64_t ldc) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, (A || (dist_on(c) && n == 0)) && Js && C, "sk_gather_cols: NULL pointer");
  SK_ARG(c, m >= 0 && n >= 0 && k >= 0 && lda >= m && ldc >= m, "sk_gather_cols: bad sizes");
  SK_CUDA(c, cudaSetDevice(c->device));
  if (dist_on(c)) {   // A is this rank's block, Js global; C replicated (synchronises)
    SK_ARG(c, n == dist_view(c).ncols, "sk_gather_cols (distributed): n must be this rank's ncols");
    return dist_gather_cols(c, A, false, m, lda, Js, k, C, ldc);
  }
  return gather_cols_shard(c, A, m, lda, 0, n, Js, k, C, ldc);   // Js outside [0, n): zero column
}

sk_status sk_gather_cols_shard(sk_ctx* c, const double* A, int64_t m, int64_t ncols, int64_t lda, int64_t col0,
                               const int64_t* Js, int64_t k, double* C, int64_t ldc) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, Js && C && (A || ncols == 0), "sk_gather_cols_shard: NULL pointer");
  SK_ARG(c, m >= 0 && ncols >= 0 && k >= 0 && col0 >= 0 && lda >= m && ldc >= m, "sk_gather_cols_shard: bad sizes");
  SK_CUDA(c, cudaSetDevice(c->device));
  return gather_cols_shard(c, A, m, lda, col0, ncols, Js, k, C, ldc);
}

size_t sk_lupp_dist_state_bytes(int64_t nloc, int64_t k) {
  if (nloc < 0 || k < 1) return 0;
  return lupp_dist_state_bytes(nloc, k);
}

sk_status sk_lupp_dist_begin(sk_ctx* c, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0,
                             void* state, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, state && cand && (X || nloc == 0), "sk_lupp_dist_begin: NULL pointer");
  SK_ARG(c, nloc >= 0 && k >= 1 && col0 >= 0 && ldx >= nloc, "sk_lupp_dist_begin: bad sizes");
  SK_ARG(c, !Lf || ldlf >= nloc, "sk_lupp_dist_begin: ldlf >= nloc required");
  SK_ARG(c, !U || ldu >= k, "sk_lupp_dist_begin: ldu >= k required");
  SK_CUDA(c, cudaSetDevice(c->device));
  return lupp_dist_begin(c, X, nloc, ldx, k, col0, state, Lf, ldlf, U, ldu, cand);
}

sk_status sk_lupp_dist_step(sk_ctx* c, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                            const double* gathered, int32_t world, int64_t* Js, double* Lf, int64_t ldlf, double* U,
                            int64_t ldu, double* cand) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, state && gathered && Js && cand, "sk_lupp_dist_step: NULL pointer");
  SK_ARG(c, nloc >= 0 && k >= 1 && t >= 1 && t <= k && world >= 1 && world <= 64 && col0 >= 0, "sk_lupp_dist_step: bad sizes (world <= 64)");
  SK_ARG(c, !Lf || ldlf >= nloc, "sk_lupp_dist_step: ldlf >= nloc required");
  SK_ARG(c, !U || ldu >= k, "sk_lupp_dist_step: ldu >= k required");
  SK_CUDA(c, cudaSetDevice(c->device));
  return lupp_dist_step(c, state, nloc, k, col0, t, gathered, world, Js, Lf, ldlf, U, ldu, cand);
}

size_t sk_lupp_dist_mailbox_bytes(int64_t k, int32_t world) {
  if (k < 1 || world < 1 || world > 64) return 0;
  return lupp_dist_mailbox_bytes(k, world);
}

sk_status sk_lupp_dist_begin_p2p(sk_ctx* c, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0,
                                 void* state, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand,
                                 double* const* peers, double* own_mailbox, int32_t rank, int32_t world) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, state && cand && peers && own_mailbox && (X || nloc == 0), "sk_lupp_dist_begin_p2p: NULL pointer");
  SK_ARG(c, nloc >= 0 && k >= 1 && col0 >= 0 && ldx >= nloc, "sk_lupp_dist_begin_p2p: bad sizes");
  SK_ARG(c, world >= 1 && world <= 64 && rank >= 0 && rank < world, "sk_lupp_dist_begin_p2p: bad rank/world");
  SK_ARG(c, !Lf || ldlf >= nloc, "sk_lupp_dist_begin_p2p: ldlf >= nloc required");
  SK_ARG(c, !U || ldu >= k, "sk_lupp_dist_begin_p2p: ldu >= k required");
  SK_CUDA(c, cudaSetDevice(c->device));
  return lupp_dist_begin(c, X, nloc, ldx, k, col0, state, Lf, ldlf, U, ldu, cand, peers, rank, world, own_mailbox);
}

sk_status sk_lupp_dist_step_p2p(sk_ctx* c, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                                double* const* peers, int32_t rank, int32_t world, int64_t* Js,
                                double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, state && peers && Js && cand, "sk_lupp_dist_step_p2p: NULL pointer");
  SK_ARG(c, nloc >= 0 && k >= 1 && t >= 1 && t <= k && col0 >= 0, "sk_lupp_dist_step_p2p: bad sizes");
  SK_ARG(c, world >= 1 && world <= 64 && rank >= 0 && rank < world, "sk_lupp_dist_step_p2p: bad rank/world");
  SK_ARG(c, !Lf || ldlf >= nloc, "sk_lupp_dist_step_p2p: ldlf >= nloc required");
  SK_ARG(c, !U || ldu >= k, "sk_lupp_dist_step_p2p: ldu >= k required");
  SK_CUDA(c, cudaSetDevice(c->device));
  return lupp_dist_step(c, state, nloc, k, col0, t, nullptr, world, Js, Lf, ldlf, U, ldu, cand, peers, rank);
}

sk_status sk_ipc_alloc(sk_ctx* c, size_t bytes, void** ptr) {
  if (!c || !ptr) return SK_E_ARG;
  c->err.clear();
  SK_CUDA(c, cudaSetDevice(c->device));
  SK_CUDA(c, cudaMalloc(ptr, bytes ? bytes : 16));
  SK_CUDA(c, cudaMemset(*ptr, 0, bytes ? bytes : 16));
  return SK_OK;
}

sk_status sk_ipc_free(sk_ctx* c, void* ptr) {
  if (!c) return SK_E_ARG;
  SK_CUDA(c, cudaSetDevice(c->device));
  SK_CUDA(c, cudaFree(ptr));
  return SK_OK;
}

sk_status sk_ipc_export(sk_ctx* c, void* ptr, void* handle) {
  if (!c || !ptr || !handle) return SK_E_ARG;
  c->err.clear();
  cudaIpcMemHandle_t h;
  SK_CUDA(c, cudaIpcGetMemHandle(&h, ptr));
  std::memcpy(handle, &h, sizeof(h));
  return SK_OK;
}

sk_status sk_ipc_import(sk_ctx* c, const void* handle, void** ptr) {
  if (!c || !handle || !ptr) return SK_E_ARG;
  c->err.clear();
  SK_CUDA(c, cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  SK_CUDA(c, cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SK_OK;
}

sk_status sk_ipc_close(sk_ctx* c, void* ptr) {
  if (!c) return SK_E_ARG;
  SK_CUDA(c, cudaSetDevice(c->device));
  SK_CUDA(c, cudaIpcCloseMemHandle(ptr));
  return SK_OK;
}

sk_status sk_lupp_dist_info(sk_ctx* c, const void* state, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, state && info, "sk_lupp_dist_info: NULL pointer");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(lupp_dist_status(c, state, st.as<int64_t>()));
  int64_t v = 0;
  SK_TRY(to_host(c, &v, st.p, sizeof(int64_t)));
  *info = v;
  if (v < 0)
    return fail(c, SK_E_STATE, "sk_lupp_dist: no record from a peer within the timeout (SKEL_PEER_TIMEOUT_MS, default 30 s) at step " + std::to_string(-v));
  if (v > 0) return fail(c, SK_E_RANK, "sk_lupp_dist: rank deficiency at step " + std::to_string(v));
  return SK_OK;
}

sk_status sk_residual_cols(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const double* C, int64_t k,
                           int64_t ldc, double* sums) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && C && sums, "sk_residual_cols: NULL pointer");
  SK_ARG(c, m >= 1 && n >= 1 && k >= 1 && k <= m && lda >= m && ldc >= m, "sk_residual_cols: bad sizes");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf d, st;
  SK_TRY(d.alloc(c, 2 * sizeof(double)));
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(residual_cols(c, A, m, n, lda, C, k, ldc, d.as<double>(), st.as<int64_t>()));
  int64_t info = 0;
  SK_TRY(finish_info(c, st.as<int64_t>(), &info, "sk_residual_cols (basis of C)"));
  return to_host(c, sums, d.p, 2 * sizeof(double));
}

sk_status sk_select_rows(sk_ctx* c, const double* C, int64_t m, int64_t k, int64_t ldc, int64_t* Is,
                         double* Lf, int64_t ldlf, double* U, int64_t ldu, double* gaps, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, C && Is, "sk_select_rows: NULL C or Is");
  SK_ARG(c, k >= 1 && k <= m && ldc >= m, "sk_select_rows: need 1 <= k <= m, ldc >= m");
  SK_ARG(c, !Lf || ldlf >= m, "sk_select_rows: ldlf >= m required");
  SK_ARG(c, !U || ldu >= k, "sk_select_rows: ldu >= k required");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf st;
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  SK_TRY(lupp(c, C, false, m, k, ldc, Is, Lf, ldlf, U, ldu, gaps, st.as<int64_t>()));
  return finish_info(c, st.as<int64_t>(), info, "sk_select_rows");
}

sk_status sk_id_coeffs(sk_ctx* c, const double* Lf, int64_t n, int64_t k, int64_t ldlf, const int64_t* Js,
                       double* Z, int64_t ldz, double* eta) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, (Lf || (dist_on(c) && n == 0)) && Js && Z, "sk_id_coeffs: NULL pointer");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf e;
  if (eta) SK_TRY(e.alloc(c, sizeof(double)));
  if (dist_on(c)) {   // Lf: this rank's rows (n = ncols), Z: this rank's columns; eta over all ranks
    const DistView v = dist_view(c);
    SK_ARG(c, n == v.ncols && k >= 1 && k <= v.n_global && ldlf >= std::max<int64_t>(n, 1) && ldz >= k,
           "sk_id_coeffs (distributed): bad sizes");
    SK_TRY(dist_id_coeffs(c, Lf, k, ldlf, Js, Z, ldz, eta ? e.as<double>() : nullptr));
  } else {
    SK_ARG(c, k >= 1 && k <= n && ldlf >= n && ldz >= k, "sk_id_coeffs: bad sizes");
    SK_TRY(id_coeffs(c, Lf, n, k, ldlf, Js, Z, ldz, eta ? e.as<double>() : nullptr));
  }
  if (eta) SK_TRY(to_host(c, eta, e.p, sizeof(double)));
  return SK_OK;
}

sk_status sk_residual(sk_ctx* c, const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* Js,
                      const int64_t* Is, int64_t k, sk_residual_kind kind, const double* Z, int64_t ldz,
                      double* res_fro, double* normA_fro) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, (A || (dist_on(c) && n == 0)) && res_fro, "sk_residual: NULL A or res_fro");
  if (dist_on(c)) {
    const DistView v = dist_view(c);
    SK_ARG(c, n == v.ncols && m >= 1 && lda >= m && k >= 1 && k <= m && k <= v.n_global,
           "sk_residual (distributed): n must be this rank's ncols, 1 <= k <= min(m, n_global)");
  } else {
    SK_ARG(c, m >= 1 && n >= 1 && lda >= m && k >= 1 && k <= m && k <= n, "sk_residual: bad sizes");
  }
  SK_ARG(c, kind >= SK_RES_COL_ID && kind <= SK_RES_CUR_CSS, "sk_residual: unknown kind");
  const bool need_js = kind != SK_RES_ROW_ID && kind != SK_RES_ROW_COEFFS;
  const bool need_is = kind == SK_RES_ROW_ID || kind == SK_RES_CUR || kind == SK_RES_ROW_COEFFS || kind == SK_RES_CUR_CSS;
  SK_ARG(c, !need_js || Js, "sk_residual: Js required");
  SK_ARG(c, !need_is || Is, "sk_residual: Is required");
  SK_ARG(c, kind != SK_RES_ID_COEFFS || (Z && ldz >= k), "sk_residual: Z (ldz >= k) required");
  SK_ARG(c, kind != SK_RES_ROW_COEFFS || (Z && ldz >= m), "sk_residual: W (passed as Z, ldz >= m) required");
  SK_ARG(c, !dist_on(c) || kind <= SK_RES_ID_COEFFS, "sk_residual: the estimate kinds are single-GPU only");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf sums, st;
  SK_TRY(sums.alloc(c, 2 * sizeof(double)));
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  if (dist_on(c)) SK_TRY(dist_residual(c, A, m, lda, Js, Is, k, (int)kind, Z, ldz, sums.as<double>(), st.as<int64_t>()));
  else SK_TRY(residual(c, A, m, n, lda, Js, Is, k, (int)kind, Z, ldz, sums.as<double>(), st.as<int64_t>()));
  int64_t info = 0;
  SK_TRY(finish_info(c, st.as<int64_t>(), &info, "sk_residual (basis of the skeleton)"));
  double h[2];
  SK_TRY(to_host(c, h, sums.p, sizeof(h)));
  *res_fro = std::sqrt(h[0]);
  if (normA_fro) *normA_fro = std::sqrt(h[1]);
  return SK_OK;
}

sk_status sk_rand_lupp(sk_ctx* c, const double* A, int a_on_host, int64_t m, int64_t n, int64_t lda,
                       int64_t l, sk_embedding emb, int32_t zeta, uint64_t seed, int64_t k, int64_t* Js,
                       int64_t* Is, int64_t* info) {
  if (!c) return SK_E_ARG;
  c->err.clear();
  SK_ARG(c, A && Js, "sk_rand_lupp: NULL A or Js");
  const bool dist = dist_on(c);
  SK_ARG(c, m >= 1 && (n >= 1 || dist) && lda >= m && l >= 1 && l <= m && k >= 1 && k <= l &&
                k <= (dist ? dist_view(c).n_global : n) && (!dist || n == dist_view(c).ncols),
         "sk_rand_lupp: need 1 <= k <= l <= m, k <= n (distributed: n = this rank's ncols, k <= n_global)");
  SK_CUDA(c, cudaSetDevice(c->device));
  DBuf Xd, Jd, Cd, Id, st;
  SK_TRY(Xd.alloc(c, (size_t)l * n * sizeof(double)));
  SK_TRY(Jd.alloc(c, (size_t)k * sizeof(int64_t)));
  SK_TRY(st.alloc(c, sizeof(int64_t)));
  if (a_on_host) {
    // A stays in host memory: X = Gamma A is column-separable, so A's column blocks stream through
    // the device ring of for_host_blocks (copy of block b overlapping the sketch of block b - 1)
    SK_TRY(for_host_blocks(c, A, m, n, lda, [&](const double* blk, int64_t j0, int64_t jw) {
      return sk_sketch(c, blk, m, jw, m, l, emb, zeta, seed, Xd.as<double>() + j0, n);
    }));
  } else {
    SK_TRY(sk_sketch(c, A, m, n, lda, l, emb, zeta, seed, Xd.as<double>(), n));
  }
  if (dist) SK_TRY(dist_select_cols(c, Xd.as<double>(), n, std::max<int64_t>(n, 1), k, Jd.as<int64_t>(), nullptr, 0,
                                    nullptr, 0, nullptr, st.as<int64_t>()));
  else SK_TRY(lupp(c, Xd.as<double>(), true, n, k, n, Jd.as<int64_t>(), nullptr, 0, nullptr, 0, nullptr,
                   st.as<int64_t>()));
  int64_t inf = 0;
  sk_status rc = finish_info(c, st.as<int64_t>(), &inf, "sk_rand_lupp (columns)");
  if (info) *info = inf;                                   // set on SK_E_RANK too (the failing step)
  SK_TRY(rc);
  SK_TRY(to_host(c, Js, Jd.p, (size_t)k * sizeof(int64_t)));
  if (Is) {
    SK_ARG(c, k <= m, "sk_rand_lupp: k <= m required for row skeletons");
    SK_TRY(Cd.alloc(c, (size_t)m * k * sizeof(double)));
    SK_TRY(Id.alloc(c, (size_t)k * sizeof(int64_t)));
    if (dist) {          // C = A_global(:, J_s) assembled across ranks
      SK_TRY(dist_gather_cols(c, A, a_on_host != 0, m, lda, Jd.as<int64_t>(), k, Cd.as<double>(), m));
    } else if (a_on_host) {     // C = A(:, J_s) straight from the host columns (pivot order, R8)
      for (int64_t t = 0; t < k; ++t)
        SK_CUDA(c, cudaMemcpyAsync(Cd.as<double>() + t * m, A + Js[t] * lda, (size_t)m * sizeof(double),
                                   cudaMemcpyHostToDevice, c->stream));
    } else {
      SK_TRY(gather_cols(c, A, m, lda, Jd.as<int64_t>(), k, Cd.as<double>(), m));
    }
    SK_TRY(lupp(c, Cd.as<double>(), false, m, k, m, Id.as<int64_t>(), nullptr, 0, nullptr, 0, nullptr,
                st.as<int64_t>()));
    rc = finish_info(c, st.as<int64_t>(), &inf, "sk_rand_lupp (rows)");
    if (info) *info = inf;
    SK_TRY(rc);
    SK_TRY(to_host(c, Is, Id.p, (size_t)k * sizeof(int64_t)));
  }
  return SK_OK;
}

}  // extern "C"
