// lupp_dist.cu -- column LUPP on a column-sharded sketch with ONE exchange per pivot step
// (the per-step AllGather design; eq:def_LUPP and the pivot rule).
//
// Rank r owns the rows col0 .. col0 + nloc - 1 of the n x k panel M = X(0:k, :)^T (R5), i.e.
// the sketch columns of its own block of A.  Step t of the swap-free LUPP becomes
//   propose   every rank: its best active row (|M(i, t)|, lowest local index on ties) and that
//             row's current entries M(i, 0:k)  -> one record of k + 4 doubles (``cand``);
//   exchange  an all-gather of the records (the caller's collective, NCCL on the product path);
//   decide    every rank, on identical bytes: max |value|, ties to the lowest GLOBAL index (R6),
//             rank failure if the winner is <= 1e-14 max|panel| over all ranks (R7);
//   update    every rank eliminates its own active rows with the winner's row:
//             L(i, t) = M(i, t) / u_t,  M(i, c) -= L(i, t) u_c  (c > t).
// One kernel (k_dist_step) fuses "decide + update" of step t - 1 with "propose" of step t, so a
// step is one launch plus one collective; the launch sequence has no host synchronisation and is
// captured in a CUDA graph by the caller (paper_2104_05877_b200.dist).  The update rounds exactly
// like the oracle's (separate multiply and subtract, no FMA contraction), so pivots, L and U are
// bit-identical to oracle.lupp.select_cols on the unsharded panel.
//
// Record layout (double[k + 4]): [0] |value| or -1 if the rank has no active row, [1] global row
// index or -1, [2] the rank's max |panel| (for R7), [3] reserved (0), [4 + c] M(i, c), c < k.
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace skel {
namespace {

constexpr int DT = 256;   // panel rows per CTA (one row per thread)
constexpr int DCW = 32;   // panel columns per CTA

struct DistHdr {
  long long status;            // 0, the 1-based failing step (latched), or -t: peer timeout at step t
  unsigned ctr;                // last-CTA ticket counter (reset by the last CTA)
  unsigned pad;
  unsigned long long lmax;     // bits of max |M| over this rank's panel (non-negative doubles order as u64)
};

struct DistLayout {
  DistHdr* hdr;
  double* part_a;
  long long* part_i;
  int* flags;    // -1 active, else the step that pivoted the row
  double* M;     // nloc x k column-major (ld nloc)
};

__host__ __device__ inline size_t al256(size_t b) { return (b + 255) & ~size_t(255); }

// mailbox of `world` ranks: [2][world][REC] records, [world] flags, [1] selection epoch (local)
__device__ __forceinline__ unsigned long long* mb_flags(double* mb, int world, int64_t REC) {
  return reinterpret_cast<unsigned long long*>(mb + 2 * (int64_t)world * REC);
}
__host__ __device__ inline int64_t dist_rb(int64_t nloc) { return nloc > 0 ? (nloc + DT - 1) / DT : 1; }

__host__ __device__ inline DistLayout dist_layout(void* state, int64_t nloc) {
  unsigned char* p = reinterpret_cast<unsigned char*>(state);
  const int64_t rb = dist_rb(nloc);
  DistLayout L;
  L.hdr = reinterpret_cast<DistHdr*>(p);
  p += 256;
  L.part_a = reinterpret_cast<double*>(p);
  p += al256(8 * rb);
  L.part_i = reinterpret_cast<long long*>(p);
  p += al256(8 * rb);
  L.flags = reinterpret_cast<int*>(p);
  p += al256(4 * (nloc > 0 ? nloc : 1));
  L.M = reinterpret_cast<double*>(p);
  return L;
}

size_t dist_state_bytes(int64_t nloc, int64_t k) {
  const int64_t rb = dist_rb(nloc);
  return 256 + 2 * al256(8 * rb) + al256(4 * (nloc > 0 ? nloc : 1)) + (size_t)8 * (nloc > 0 ? nloc : 0) * k + 256;
}

// M(i, c) = X(c, i) (X row-major, rows 0..k-1 of the local sketch block), flags = -1, lmax.
__global__ void k_dist_begin_epoch(double* mb, int world, int64_t k) {
  unsigned long long* e = mb_flags(mb, world, k + 4) + world;
  *e = *e + (unsigned long long)(k + 2);            // above every flag of earlier selections
}

__global__ void k_dist_begin(const double* __restrict__ X, int64_t ldx, int64_t nloc, int64_t k, DistLayout L) {
  double mx = 0.0;
  const int64_t total = nloc * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % nloc, c = e / nloc;
    const double v = X[c * ldx + i];
    L.M[e] = v;
    mx = fmax(mx, fabs(v));
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x)
    L.flags[i] = -1;
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx > 0.0)
    atomicMax(&L.hdr->lmax, (unsigned long long)__double_as_longlong(mx));
}

struct StepArgs {
  DistLayout L;
  int64_t nloc, k, col0, t;
  const double* gathered; int world;
  int64_t* Js; double* Lf; int64_t ldlf; double* U; int64_t ldu;
  double* cand;
  // P2P mode (peers != nullptr): every rank's mailbox = [2][world][REC] doubles (records by step
  // parity) + [world] u64 flags; peers[q] is rank q's mailbox mapped into this process (NVLink peer
  // memory / CUDA IPC), peers[rank] the local one.  The step kernel waits for the flags, reads the
  // records from its own mailbox, and publishes its next record by storing it into every peer's
  // mailbox and releasing the flags -- the exchange is part of the kernel, no collective call.
  double* const* peers; int rank;
  unsigned long long timeout_ns;   // bound on the wait for a peer's record (P2P mode)
};



__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* f) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* f, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}

__global__ void __launch_bounds__(DT) k_dist_step(StepArgs a) {
  __shared__ double su[DCW];
  __shared__ int s_bw;
  __shared__ long long s_g;
  __shared__ dev::Cand sred[33];
  __shared__ int s_last;
  const DistLayout& L = a.L;
  const int64_t k = a.k, nloc = a.nloc, t = a.t;
  const int tid = threadIdx.x;
  const int64_t REC = k + 4;
  if (*(volatile long long*)&L.hdr->status != 0) return;           // failure latched in an earlier step
  const bool corner = blockIdx.x == 0 && blockIdx.y == 0;
  if (a.world > 64) return;                                          // checked on the host
  const double* gathered = a.gathered;
  unsigned long long epoch = 0;
  if (a.peers != nullptr) {
    // the selection's epoch: a device-side counter advanced by k_dist_begin, so captured graphs replay
    double* mb = a.peers[a.rank];
    unsigned long long* flags = mb_flags(mb, a.world, REC);
    epoch = *(volatile unsigned long long*)(flags + a.world);
    if (t > 0) {
      // records of step t-1 sit in buffer (t-1) & 1 of the local mailbox once every flag >= epoch + t
      // bounded wait: a peer that never publishes (crashed rank) latches status -t after
      // a.timeout_ns (30 s; SKEL_PEER_TIMEOUT_MS) instead of hanging the GPU; sk_lupp_dist_info
      // reports it as SK_E_STATE
      __shared__ int s_late;
      if (tid == 0) s_late = 0;
      __syncthreads();
      if (tid < a.world) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(flags + tid) < epoch + (unsigned long long)t) {
          if (globaltimer_ns() - t0 > a.timeout_ns) { s_late = 1; break; }
        }
      }
      __syncthreads();
      if (s_late) {
        if (tid == 0) atomicCAS(reinterpret_cast<unsigned long long*>(&L.hdr->status), 0ull,
                                (unsigned long long)(-(long long)t));
        return;
      }
      // buffer parity (epoch + t - 1) & 1, not (t - 1) & 1: epochs advance by k + 2 per selection, so
      // step 0 of the NEXT selection (buffer (epoch + k + 2) & 1 = (epoch + k) & 1) never overwrites
      // the buffer the last step of this one reads ((epoch + k - 1) & 1), even for odd k
      gathered = mb + (int64_t)((epoch + (unsigned long long)t - 1ull) & 1ull) * a.world * REC;
    }
  }

  const int64_t c0 = t + (int64_t)blockIdx.y * DCW;                  // this CTA's first updated column
  const int64_t i = (int64_t)blockIdx.x * DT + tid;
  const bool in = i < nloc;
  // prefetch this thread's row data (independent of the decision, overlaps its latency)
  double mv[DCW];
  double mprev = 0.0;
  int fl = 0;
  if (in) {
    fl = L.flags[i];
    if (t > 0) {
      mprev = L.M[i + (t - 1) * nloc];
#pragma unroll
      for (int j = 0; j < DCW; ++j) mv[j] = c0 + j < k ? L.M[i + (c0 + j) * nloc] : 0.0;
    } else {
      mv[0] = L.M[i];
    }
  }

  // ---- decide step t - 1 from the gathered records (identical on every rank): warp 0 reads the
  //      records in parallel (lane w <- record w) and reduces max |value|, ties -> lowest index
  long long pl = -1;               // local index of the pivot row if this rank owns it
  const double* rec = nullptr;
  if (t > 0) {
    if (tid < 32) {
      double gmax = 0.0;
      dev::Cand cd = dev::cand_none();
      for (int w = tid; w < a.world; w += 32) {
        const double* r = gathered + (int64_t)w * REC;
        gmax = fmax(gmax, __ldcg(r + 2));
        const long long idx = (long long)__ldcg(r + 1);
        if (idx >= 0) {
          dev::Cand x = dev::cand_none();
          x.a1 = __ldcg(r);
          x.i1 = idx * 64 + w;                      // rank index rides in the low bits (world <= 64)
          cd = dev::cand_merge(cd, x);
        }
      }
      cd = dev::warp_cand_reduce(cd);
#pragma unroll
      for (int o = 16; o; o >>= 1) gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
      if (tid == 0) {
        const bool ok = cd.i1 != LLONG_MAX && cd.a1 > 1e-14 * gmax;
        s_bw = ok ? (int)(cd.i1 & 63) : -1;
        s_g = ok ? cd.i1 >> 6 : -1;
      }
    }
    __syncthreads();
    if (s_bw < 0) {                                                   // R7: rank failure at step t
      if (corner) {
        if (tid == 0) L.hdr->status = t;
        for (int64_t s = t - 1 + tid; s < k; s += DT) a.Js[s] = -1;
      }
      return;
    }
    rec = gathered + (int64_t)s_bw * REC;
    const long long g = s_g;
    if (g >= a.col0 && g < a.col0 + nloc) pl = g - a.col0;
    if (corner) {
      if (tid == 0) a.Js[t - 1] = g;
      if (a.U)
        for (int64_t c = t - 1 + tid; c < k; c += DT) a.U[(t - 1) + c * a.ldu] = __ldcg(rec + 4 + c);
    }
    if (tid < DCW) su[tid] = c0 + tid < k ? __ldcg(rec + 4 + c0 + tid) : 0.0;
    __syncthreads();
  }
  bool act = in && fl < 0 && i != pl;
  double mt = 0.0;                                                    // M(i, t) after the update
  if (t > 0) {
    const double piv = __ldcg(rec + 4 + t - 1);
    const double li = act ? __ddiv_rn(mprev, piv) : 0.0;
    if (blockIdx.y == 0 && in) {
      if (act) {
        if (a.Lf) a.Lf[i + (t - 1) * a.ldlf] = li;
      } else if (i == pl) {
        if (a.Lf) a.Lf[i + (t - 1) * a.ldlf] = 1.0;
        L.flags[i] = (int)(t - 1);
      }
    }
    if (act) {
      double* Mi = L.M + i;
#pragma unroll
      for (int j = 0; j < DCW; ++j) {
        const int64_t c = c0 + j;
        if (c < k) {
          const double v = __dsub_rn(mv[j], __dmul_rn(li, su[j]));
          Mi[c * nloc] = v;
          if (j == 0) mt = v;
        }
      }
    }
  } else if (act) {
    mt = mv[0];
  }
  if (t >= k) return;                                                  // last step: decision only

  // ---- propose step t: argmax |M(i, t)| over active rows (column t lives in the blockIdx.y == 0 CTAs)
  if (blockIdx.y == 0) {
    dev::Cand cd = dev::cand_none();
    if (act) { cd.a1 = fabs(mt); cd.i1 = i; }
    cd = dev::block_cand_reduce(cd, sred);
    if (tid == 0) {
      L.part_a[blockIdx.x] = cd.a1;
      L.part_i[blockIdx.x] = cd.i1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y;
    s_last = atomicAdd(&L.hdr->ctr, 1u) == total - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  dev::Cand cd = dev::cand_none();
  for (int64_t b = tid; b < gridDim.x; b += DT) {
    const long long bi = __ldcg(L.part_i + b);
    if (bi != LLONG_MAX) {
      dev::Cand x = dev::cand_none();
      x.a1 = __ldcg(L.part_a + b);
      x.i1 = bi;
      cd = dev::cand_merge(cd, x);
    }
  }
  cd = dev::block_cand_reduce(cd, sred);
  const bool has = cd.i1 != LLONG_MAX;
  if (tid == 0) {
    a.cand[0] = has ? cd.a1 : -1.0;
    a.cand[1] = has ? (double)(a.col0 + cd.i1) : -1.0;
    a.cand[2] = __longlong_as_double((long long)*(volatile unsigned long long*)&L.hdr->lmax);
    a.cand[3] = 0.0;
    L.hdr->ctr = 0u;
  }
  for (int64_t c = tid; c < k; c += DT) a.cand[4 + c] = has ? __ldcg(L.M + cd.i1 + c * nloc) : 0.0;
  if (a.peers != nullptr) {
    // publish the record of step t into slot [(epoch + t) & 1][rank] of every mailbox, then the flags
    __syncthreads();
    const double hdr[4] = {a.cand[0], a.cand[1], a.cand[2], 0.0};
    const int64_t off = (int64_t)((epoch + (unsigned long long)t) & 1ull) * a.world * REC + (int64_t)a.rank * REC;
    for (int q = 0; q < a.world; ++q) {
      double* dst = a.peers[q] + off;
      for (int64_t c = tid; c < REC; c += DT) dst[c] = c < 4 ? hdr[c] : a.cand[c];
    }
    __threadfence_system();
    __syncthreads();
    if (tid < a.world) st_release_sys(mb_flags(a.peers[tid], a.world, REC) + a.rank, epoch + (unsigned long long)t + 1ull);
  }
}

}  // namespace

size_t lupp_dist_state_bytes(int64_t nloc, int64_t k) { return dist_state_bytes(nloc, k); }
size_t lupp_dist_mailbox_bytes(int64_t k, int world) {
  return (size_t)8 * (2 * (size_t)world * (size_t)(k + 4) + (size_t)world + 1);
}

sk_status lupp_dist_begin(sk_ctx* c, const double* X, int64_t nloc, int64_t ldx, int64_t k, int64_t col0, void* state,
                          double* Lf, int64_t ldlf, double* U, int64_t ldu, double* cand, double* const* peers,
                          int rank, int world, double* own_mailbox) {
  DistLayout L = dist_layout(state, nloc);
  SK_CUDA(c, cudaMemsetAsync(state, 0, 256, c->stream));
  if (Lf && nloc > 0) SK_CUDA(c, cudaMemset2DAsync(Lf, ldlf * sizeof(double), 0, nloc * sizeof(double), k, c->stream));
  if (U) SK_CUDA(c, cudaMemset2DAsync(U, ldu * sizeof(double), 0, k * sizeof(double), k, c->stream));
  if (nloc > 0) {
    const int64_t total = nloc * k;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), 8 * (int64_t)c->num_sms);
    k_dist_begin<<<grid, 256, 0, c->stream>>>(X, ldx, nloc, k, L);
    SK_TRY(launched(c));
  }
  if (peers) {
    k_dist_begin_epoch<<<1, 1, 0, c->stream>>>(own_mailbox, world, k);
    SK_TRY(launched(c));
  }
  return lupp_dist_step(c, state, nloc, k, col0, 0, nullptr, world, nullptr, Lf, ldlf, U, ldu, cand, peers, rank);
}

sk_status lupp_dist_step(sk_ctx* c, void* state, int64_t nloc, int64_t k, int64_t col0, int64_t t,
                         const double* gathered, int world, int64_t* Js, double* Lf, int64_t ldlf, double* U,
                         int64_t ldu, double* cand, double* const* peers, int rank) {
  StepArgs a{};
  a.L = dist_layout(state, nloc);
  a.nloc = nloc; a.k = k; a.col0 = col0; a.t = t;
  a.gathered = gathered; a.world = world;
  a.Js = Js; a.Lf = Lf; a.ldlf = ldlf; a.U = U; a.ldu = ldu; a.cand = cand;
  a.peers = peers; a.rank = rank;
  static const unsigned long long timeout_ns = [] {
    const char* v = std::getenv("SKEL_PEER_TIMEOUT_MS");
    const long long ms = v ? std::atoll(v) : 30000;
    return (unsigned long long)(ms > 0 ? ms : 30000) * 1000000ull;
  }();
  a.timeout_ns = timeout_ns;
  const int64_t cols = t == 0 ? 1 : std::max<int64_t>(1, cdiv(k - t, DCW));
  dim3 grid((unsigned)dist_rb(nloc), (unsigned)cols);
  k_dist_step<<<grid, DT, 0, c->stream>>>(a);
  return launched(c);
}

sk_status lupp_dist_status(sk_ctx* c, const void* state, int64_t* status_dev_out) {
  SK_CUDA(c, cudaMemcpyAsync(status_dev_out, state, sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
  return SK_OK;
}

}  // namespace skel
