// lupp.cu -- S2 / S4: k-step LU with partial pivoting on a tall n x k panel.
//
// Paper: eq:def_LUPP and the pivot rule: step t scans ONE line of the
// active submatrix, picks j_t = argmax |X^{(t)}(t, j)| and applies the Schur-complement
// update.  Column LUPP on the sketch X gives J_s (Alg. 2 line 3); row LUPP
// on C = A(:, J_s) gives I_s (line 4).  Both are the same computation on an n x k
// panel M whose ROWS are pivoted (M = X(0:k, :)^T, resp. M = C).  Readings: R5 (only
// rows 0..k-1 of X enter), R6 (ties -> lowest original index, no physical swaps),
// R7 (rank failure when |pivot| <= 1e-14 max|M|).
//
// B200 design.  The k-long chain of global argmaxes is the
// critical path.  The pivot search therefore runs inside ONE thread-block cluster
// (16 CTAs on 16 SMs, distributed shared memory): an exchange costs one cluster
// barrier instead of a grid-wide flag barrier (3.7 us measured, tools/microbench).
// The panel is factored in column blocks of width bp held in the cluster's shared
// memory (one thread per row), so a step is
//     warp argmax -> CTA argmax -> DSMEM publish -> cluster barrier -> remote fetch of
//     the winning row (<= bp doubles) -> update pass (which also yields the next argmax),
// two CTA barriers and one cluster barrier per pivot.  Between column blocks:
//     k_lupp_u12 (grid) : U(c0:c1, c1:k) = L11^{-1} M(piv, c1:k)   (forward substitution)
//     gemm       (grid) : M(:, c1:k) -= Lf(:, c0:c1) U(c0:c1, c1:k) (DMMA)
// Blocked and unblocked elimination are the same algorithm; only rounding differs.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdlib>

#include "common.cuh"
#include "dmma.cuh"
#include "internal.h"

namespace cg = cooperative_groups;

namespace skel {
namespace {

constexpr int PNT = 256;            // threads per panel CTA
constexpr int PNW = PNT / 32;       // warps
constexpr int MAXCS = 16;           // max cluster size
constexpr int U12_BP = 64;          // max block width when there is a trailing update
constexpr int kMaxG = 32;           // max clusters of one multi-cluster LUPP panel (one warp reduces them)

struct Slot {            // a warp's pivot candidate, published to every CTA of the cluster
  unsigned long long key;  // bits(|v|) + 1 (0 = none): orders like |v|
  long long idx;           // global row
  unsigned long long sec;  // runner-up key (for the gap diagnostic)
  double lp;               // the candidate row's multiplier of the previous step
};

struct PanelParams {
  double* W;  int64_t n;  int k;        // working panel, n x k col-major (ld n), trailing-updated
  int c0, bp;                            // this column block
  int R;                                 // rows per CTA
  int* rowstate;                         // global: -1 active, else step at which picked
  int64_t* Js; double* Lf; int64_t ldlf; double* Uw;   // Uw: k x k col-major (ld k)
  double* gaps;
  const unsigned long long* maxbits;     // max |M| (bit pattern)
  int64_t* status;                       // 0 or 1-based failing step
  // several clusters (v2 kernel, G > 1, tall panels): the cluster winners of every step meet in
  // global memory -- gbox [2][G][4 + NB] messages by step parity, gflag [G] = last published step + 1
  int G;
  double* gbox;
  unsigned long long* gflag;
  unsigned long long timeout_ns;
};

// W (n x k col-major) = the panel, rowstate = -1, maxbits = max |panel|.  Grid (n / 1024, k): no
// 64-bit divisions, and each thread issues its 4 loads before its stores.
__global__ void k_lupp_init(const double* P, bool row_major, int64_t n, int k, int64_t ld, double* W,
                            int* rowstate, unsigned long long* maxbits) {
  const int64_t t = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  double v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + 256 * u;
    v[u] = i < n ? (row_major ? P[t * ld + i] : P[i + t * ld]) : 0.0;
  }
  double mx = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + 256 * u;
    if (i < n) {
      W[i + t * n] = v[u];
      if (t == 0) rowstate[i] = -1;
    }
    mx = fmax(mx, fabs(v[u]));
  }
  __shared__ double wmx[8];
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) wmx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {                                  // one atomic per CTA, not per warp
    double b = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) b = fmax(b, wmx[q]);
    if (b > 0.0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(b));
  }
}

// Shared-memory layout of the panel kernel (bytes), shared by host and device.
struct PanelSmem {
  size_t P, urow, wrow, slots, ub, js, gp, state, mbar, total;
  int stride, rs;
  __host__ __device__ PanelSmem(int R, int bp) {
    stride = ((bp + 1) | 3) - 1;            // = 2 mod 4 doubles: 16-byte row-per-lane access is conflict-free
    if (stride < bp) stride += 4;
    rs = (bp + 3) & ~1;                     // row buffers (even: 16-byte aligned)
    P = 0;
    size_t o = (size_t)R * stride * sizeof(double);
    urow = o;  o += (size_t)2 * rs * sizeof(double);                // pivot rows U(s,:), U(s-1,:) (CTA)
    wrow = o;  o += (size_t)2 * PNW * rs * sizeof(double);          // published candidate rows per warp
    o = (o + 15) & ~(size_t)15;
    slots = o; o += (size_t)2 * MAXCS * PNW * sizeof(Slot);
    ub = o;    o += (size_t)bp * bp * sizeof(double);                  // U block (CTA 0)
    js = o;    o += (size_t)bp * sizeof(long long);
    gp = o;    o += (size_t)bp * sizeof(double);
    state = o; o += (size_t)R * sizeof(int);
    o = (o + 15) & ~(size_t)15;
    mbar = o;  o += 2 * sizeof(unsigned long long);
    total = o + 64;
  }
};

// Warp argmax of (key, idx): largest key, ties -> lowest idx; plus the runner-up key.
// REDUX-based (32-bit halves), no shuffles of doubles.
__device__ __forceinline__ void warp_argmax(unsigned long long key, unsigned idx, unsigned long long sec,
                                            unsigned long long& wkey, unsigned& widx,
                                            unsigned long long& wsec, bool want_sec) {
  const unsigned FULL = 0xffffffffu;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_max_sync(FULL, hi);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  wkey = ((unsigned long long)mh << 32) | ml;
  widx = __reduce_min_sync(FULL, (key == wkey && key != 0ull) ? idx : 0xffffffffu);
  wsec = 0ull;
  if (want_sec) {
    const unsigned long long own = (key == wkey && idx == widx) ? sec : key;
    const unsigned sh = __reduce_max_sync(FULL, (unsigned)(own >> 32));
    const unsigned sl = __reduce_max_sync(FULL, (unsigned)(own >> 32) == sh ? (unsigned)own : 0u);
    wsec = ((unsigned long long)sh << 32) | sl;
  }
}

__device__ __forceinline__ void cand_push(unsigned long long k, long long i, unsigned long long& key, long long& idx,
                                          unsigned long long& sec) {
  if (k > key || (k == key && k != 0ull && i < idx)) {
    sec = key > sec ? key : sec;
    key = k; idx = i;
  } else {
    sec = k > sec ? k : sec;
  }
}

__device__ __forceinline__ unsigned long long mag_key(double v) {
  return (unsigned long long)__double_as_longlong(fabs(v)) + 1ull;
}

// ---- cluster mailbox: st.async into a peer CTA's shared memory, completing bytes on the
// peer's mbarrier; the receiver waits on its own mbarrier (no cluster-wide barrier).
__device__ __forceinline__ unsigned mapa(unsigned local_addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v2(unsigned raddr, unsigned long long a, unsigned long long b,
                                            unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "l"(a), "l"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned addr, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned addr, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned addr, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// One thread per row (RPT = ceil(R / PNT) rows per thread), the CTA's block of rows in
// shared memory.  Pivot step s, per warp, with no CTA-wide barrier:
//   A  wait on this CTA's mailbox (mbarrier) for the CS*PNW warp candidates of step s;
//      reduce them (REDUX) to the winner -- identical in every warp of every CTA;
//   F  fetch the winner's published row copy from its owner's shared memory (DSMEM) and
//      apply the one update it lacks (step s-1 on columns >= s+1);
//   B  critical part: multipliers L(i,s) and column s+1 of own rows -> warp argmax ->
//      copy of the candidate row into this warp's publish buffer -> st.async of the
//      candidate into every CTA's mailbox (completes bytes on that CTA's mbarrier);
//   C  bulk Schur update of columns >= s+2, overlapping the exchange of step s+1.
template <bool GAPS>
__global__ void __launch_bounds__(PNT, 1) k_lupp_panel(PanelParams p) {
  dev::griddep_wait();
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  extern __shared__ __align__(16) unsigned char smraw[];
  const PanelSmem L(p.R, p.bp);
  double* P = reinterpret_cast<double*>(smraw + L.P);                 // [R][stride]
  Slot* slots = reinterpret_cast<Slot*>(smraw + L.slots);             // [2][MAXCS*PNW]
  double* ub = reinterpret_cast<double*>(smraw + L.ub);               // [bp][bp]
  long long* js = reinterpret_cast<long long*>(smraw + L.js);         // [bp]
  double* gp = reinterpret_cast<double*>(smraw + L.gp);               // [bp]
  int* state = reinterpret_cast<int*>(smraw + L.state);               // [R]
  const unsigned mbar0 = dev::smem_u32(smraw + L.mbar);                // 2 mbarriers (step parity)
  const unsigned slots_u32 = dev::smem_u32(slots);
  __shared__ int s_stop;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bp = p.bp, ps = L.stride, rs = L.rs;
  double* urow0 = reinterpret_cast<double*>(smraw + L.urow);                           // + par*rs
  double* wrow0 = reinterpret_cast<double*>(smraw + L.wrow) + (size_t)warp * rs;
  const unsigned wrow_u32 = dev::smem_u32(smraw + L.wrow);
  const int64_t r0 = (int64_t)crank * p.R;
  const int Rc = (int)std::max<int64_t>(0, std::min<int64_t>(p.R, p.n - r0));
  const int nslots = csize * PNW;

  if (tid == 0) {
    s_stop = (*p.status != 0);
    mbar_init(mbar0, 1);
    mbar_init(mbar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int e = tid; e < Rc * bp; e += PNT) {          // async copy, coalesced along rows
    const int li = e % Rc, s = e / Rc;
    dev::cp_async8(P + (size_t)li * ps + s, p.W + (r0 + li) + (int64_t)(p.c0 + s) * p.n, true);
  }
  dev::cp_async_commit();
  for (int li = tid; li < Rc; li += PNT) state[li] = p.rowstate[r0 + li];
  const double tol = 1e-14 * __longlong_as_double((long long)*p.maxbits);
  dev::cp_async_wait<0>();
  cluster.sync();    // rows staged, mbarriers initialised cluster-wide
  const int s_end = s_stop ? 0 : bp;

  // publish this warp's candidate for step `sn`: rows' column sn, copy of the winning row
  auto publish = [&](int sn, unsigned long long ckey, long long cidx, unsigned long long csec) {
    const int par = sn & 1;
    if (tid == 0) mbar_arm(mbar0 + 8 * par, (unsigned)(nslots * sizeof(Slot)));
    __syncwarp();   // the lanes' row updates are visible to the lanes copying the candidate row
    unsigned long long wk, ws;
    unsigned wi;
    warp_argmax(ckey, (unsigned)cidx, csec, wk, wi, ws, GAPS);
    if (wk) {   // copy row wi, columns sn-1 .. bp-1 (multiplier of step sn-1 included)
      const double* src = P + (size_t)wi * ps;
      double* dst = wrow0 + (size_t)par * PNW * rs;
      for (int j = max(sn - 1, 0) + lane; j < bp; j += 32) dst[j] = src[j];
    }
    __syncwarp();
    const double lpc = (wk && sn > 0) ? P[(size_t)wi * ps + sn - 1] : 0.0;
    if (lane < csize) {
      const unsigned off = (unsigned)((par * (MAXCS * PNW) + crank * PNW + warp) * sizeof(Slot));
      const unsigned ra = mapa(slots_u32 + off, (unsigned)lane);
      const unsigned rb = mapa(mbar0 + 8 * par, (unsigned)lane);
      const long long gi = wk ? (long long)(r0 + wi) : 0x7fffffffffffffffLL;
      st_async_v2(ra, wk, (unsigned long long)gi, rb);
      st_async_v2(ra + 16, ws, (unsigned long long)__double_as_longlong(lpc), rb);
    }
  };

  if (s_end > 0) {   // candidate for step 0
    unsigned long long ckey = 0ull, csec = 0ull;
    long long cidx = 0x7fffffffffffffffLL;
    for (int li = tid; li < Rc; li += PNT)
      if (state[li] < 0) cand_push(mag_key(P[(size_t)li * ps]), li, ckey, cidx, csec);
    publish(0, ckey, cidx, csec);
  }
  int s_done = s_end;
  for (int s = 0; s < s_end; ++s) {
    const int t = p.c0 + s, par = s & 1;
    // (A) mailbox -> winner
    mbar_wait(mbar0 + 8 * par, (unsigned)((s >> 1) & 1));
    unsigned long long bk = 0ull, bs = 0ull;
    long long bi = 0x7fffffffffffffffLL;
    double blp = 0.0;
    for (int e = lane; e < nslots; e += 32) {
      const Slot sl = slots[par * (MAXCS * PNW) + e];
      if (sl.key && (sl.key > bk || (sl.key == bk && sl.idx < bi))) blp = sl.lp;
      if (sl.key) cand_push(sl.key, sl.idx, bk, bi, bs);
      if (GAPS) bs = sl.sec > bs ? sl.sec : bs;
    }
    unsigned long long wk, ws;
    unsigned wi;
    warp_argmax(bk, bk ? (unsigned)bi : 0xffffffffu, bs, wk, wi, ws, GAPS);
    const double a1 = wk ? __longlong_as_double((long long)(wk - 1ull)) : -1.0;
    if (!(a1 > tol)) {   // rank failure (R7): the same decision in every warp of every CTA
      if (crank == 0 && tid == 0) {
        *p.status = t + 1;
        for (int tt = t; tt < p.k; ++tt) p.Js[tt] = -1;
      }
      s_done = s;
      break;
    }
    const long long widx = (long long)wi;
    const unsigned wlanes = __ballot_sync(0xffffffffu, bk == wk && bi == widx);
    const double lp = __shfl_sync(0xffffffffu, blp, __ffs(wlanes) - 1);
    // (F) the winner's published row copy (one remote load per thread, the CTA shares it),
    //     fixed up with the step s-1 update it lacks
    double* ucur = urow0 + (size_t)par * rs;
    const double* uprev = urow0 + (size_t)(par ^ 1) * rs;
    {
      const int wr = (int)(widx / p.R);
      const int wl = (int)(widx - (int64_t)wr * p.R);
      const int ww = (wl % PNT) >> 5;
      const unsigned src = mapa(wrow_u32 + (unsigned)(((size_t)par * PNW + ww) * rs * sizeof(double)), (unsigned)wr);
      for (int j = s + tid; j < bp; j += PNT) {
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(src + 8u * j));
        ucur[j] = (s > 0 && j > s) ? fma(-lp, uprev[j], v) : v;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(PNT) : "memory");
    }
    if (crank == 0 && warp == 0) {
      if (lane == 0) {
        js[s] = widx;
        if (GAPS) {
          const double a2 = ws ? __longlong_as_double((long long)(ws - 1ull)) : 0.0;
          gp[s] = (a1 - a2) / a1;
        }
      }
      for (int j = s + lane; j < bp; j += 32) ub[s * bp + j] = ucur[j];
    }
    // (B) multipliers and column s+1 of own rows; candidate for step s+1
    const double piv = ucur[s];
    const bool more = s + 1 < bp;
    const double u1 = more ? ucur[s + 1] : 0.0;
    unsigned long long ckey = 0ull, csec = 0ull;
    long long cidx = 0x7fffffffffffffffLL;
    for (int li = tid; li < Rc; li += PNT) {
      if (state[li] >= 0) continue;
      if (r0 + li == widx) { state[li] = t; continue; }
      double* row = P + (size_t)li * ps;
      const double Lm = row[s] / piv;
      row[s] = Lm;
      if (more) {
        const double v = fma(-Lm, u1, row[s + 1]);
        row[s + 1] = v;
        cand_push(mag_key(v), li, ckey, cidx, csec);
      }
    }
    if (more) publish(s + 1, ckey, cidx, csec);
    // (C) bulk update of columns >= s+2 (off the pivot chain's critical path)
    if (s + 2 < bp) {
      for (int li = tid; li < Rc; li += PNT) {
        if (state[li] != -1) continue;
        double* row = P + (size_t)li * ps;
        const double Lm = row[s];
        int j = s + 2;
        if (j & 1) { row[j] = fma(-Lm, ucur[j], row[j]); ++j; }
        for (; j + 3 < bp; j += 4) {
          double2 x0 = *reinterpret_cast<double2*>(row + j);
          double2 x1 = *reinterpret_cast<double2*>(row + j + 2);
          const double2 y0 = *reinterpret_cast<const double2*>(ucur + j);
          const double2 y1 = *reinterpret_cast<const double2*>(ucur + j + 2);
          x0.x = fma(-Lm, y0.x, x0.x); x0.y = fma(-Lm, y0.y, x0.y);
          x1.x = fma(-Lm, y1.x, x1.x); x1.y = fma(-Lm, y1.y, x1.y);
          *reinterpret_cast<double2*>(row + j) = x0;
          *reinterpret_cast<double2*>(row + j + 2) = x1;
        }
        for (; j < bp; ++j) row[j] = fma(-Lm, ucur[j], row[j]);
      }
    }
  }
  __syncthreads();
  // outputs of the block: pivots, gaps, U rows (CTA 0); the L block and row states (all)
  if (crank == 0) {
    for (int s = tid; s < s_done; s += PNT) {
      p.Js[p.c0 + s] = js[s];
      if (GAPS) p.gaps[p.c0 + s] = gp[s];
    }
    for (int e = tid; e < s_done * bp; e += PNT) {
      const int s = e / bp, j = e % bp;
      if (j >= s) p.Uw[(p.c0 + s) + (int64_t)(p.c0 + j) * p.k] = ub[s * bp + j];
    }
  }
  for (int e = tid; e < Rc * bp; e += PNT) {        // coalesced along rows
    const int li = e % Rc, j = e / Rc;
    const int st = state[li], t = p.c0 + j;
    const double v = (st < 0 || st > t) ? P[(size_t)li * ps + j] : (st == t ? 1.0 : 0.0);
    p.Lf[(r0 + li) + (int64_t)t * p.ldlf] = v;
  }
  for (int li = tid; li < Rc; li += PNT) p.rowstate[r0 + li] = state[li];
  cluster.sync();   // no CTA leaves while a peer may still read its shared memory
}

// ------------------------------------------------------------------------------------------
// v2 panel: CTA-reduced candidates + a row-carrying all-to-all.
// Per pivot step s (measured primitives, profiles/round1/mailbox_lat.txt: a 16-CTA all-to-all
// of 34 x 16 B messages completes in ~890 cycles, a DSMEM load round trip ~265 cycles):
//   (A) every warp: REDUX argmax of column s over its active rows; the owner lane copies its
//       row (block coordinates) to the warp's smem slot; one CTA barrier;
//   (B) every warp reduces the 8 warp candidates to the CTA candidate; warp w st.async's the
//       CTA candidate + its row to CTAs w and w + 8 (one message per CTA pair per step);
//   (C) the deferred bulk Schur update of step s-1 (columns >= s+1) overlaps the exchange;
//   (D) wait for the CS messages; every warp picks the same winner (REDUX, ties -> lowest
//       global index); the winner's row is local; its columns > s lack only the step s-1
//       update (taken before (C) ran on the owner), which is applied on read:
//       U(s, c) = row(c) - row(s-1) * U(s-1, c);
//   (E) multipliers and column s+1 of the own rows (the next step's search column).
// One CTA barrier and one cluster exchange per pivot; no remote loads.
template <int RPT, int NB, bool GAPS, bool MULTI>
__global__ void __launch_bounds__(PNT, 1) k_lupp_panel_v2(PanelParams p) {
  dev::griddep_wait();
  static_assert(NB % 8 == 0 && RPT * NB <= 64, "register window");
  constexpr int MSGD = 4 + NB;                       // doubles per message: key, idx, sec, L(s-1), row[NB]
  constexpr int MSG = MSGD / 2;                      // 16-byte chunks
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int csize = (int)cluster.num_blocks();
  extern __shared__ __align__(16) unsigned char smraw[];
  double* ub = reinterpret_cast<double*>(smraw);                         // [NB][NB]
  double* wrow = ub + NB * NB;                                           // [2][PNW][NB]
  unsigned long long* wck = reinterpret_cast<unsigned long long*>(wrow + 2 * PNW * NB);   // [2][PNW]
  long long* wci = reinterpret_cast<long long*>(wck + 2 * PNW);          // [2][PNW]
  unsigned long long* wcs = reinterpret_cast<unsigned long long*>(wci + 2 * PNW);         // [2][PNW]
  double* wlp = reinterpret_cast<double*>(wcs + 2 * PNW);                // [2][PNW] candidate's L(s-1)
  double* mbox = reinterpret_cast<double*>(wlp + 2 * PNW);               // [2][MAXCS][MSGD]
  long long* js = reinterpret_cast<long long*>(mbox + 2 * MAXCS * MSGD); // [NB]
  double* gp = reinterpret_cast<double*>(js + NB);                       // [NB]
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(gp + NB);   // [2]
  const unsigned mbar0 = dev::smem_u32(mbar);
  const unsigned mbox_u = dev::smem_u32(mbox);
  __shared__ int s_stop;
  __shared__ int s_late;
  __shared__ __align__(16) double gall[MULTI ? kMaxG * (4 + NB) : 2];   // G > 1: every cluster's winning message
  const int g = (int)blockIdx.x / csize;             // cluster index (G > 1)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bp = p.bp;
  const int64_t r0 = ((int64_t)g * csize + crank) * p.R;
  const int Rc = (int)std::max<int64_t>(0, std::min<int64_t>(p.R, p.n - r0));

  if (tid == 0) {
    s_late = 0;
    s_stop = (*p.status != 0);
    mbar_init(mbar0, 1);
    mbar_init(mbar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  double v[RPT][NB];
  int st[RPT];
  double lprev[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = tid + PNT * r;
    const bool in = li < Rc;
    st[r] = in ? p.rowstate[r0 + li] : -2;
    lprev[r] = 0.0;
#pragma unroll
    for (int q = 0; q < NB; ++q)
      v[r][q] = (in && q < bp) ? p.W[(r0 + li) + (int64_t)(p.c0 + q) * p.n] : 0.0;   // coalesced along rows
  }
  const double tol = 1e-14 * __longlong_as_double((long long)*p.maxbits);
  __syncthreads();
  cluster.sync();    // mbarriers initialised cluster-wide before any message
  const int s_end = s_stop ? 0 : bp;
  int s_done = s_end;
  bool stop = false;

  // Steps run in chunks of 8 with the chunk unrolled, so the register window (v[r][q] =
  // block column cb + q) is indexed statically; the window slides by 8 after each chunk.
  // (A per-step slide with a rolled loop was measured 1.5x slower: predicated full-width
  // updates and longer dependency chains, profiles/round1/lupp_probe.txt.)
  for (int cb = 0; cb < s_end && !stop; cb += 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int s = cb + i;
      if (s >= s_end) break;
      const int t = p.c0 + s, par = s & 1;
      // (A) local candidate of column s, owner copies its row (block coordinates)
      unsigned long long ckey = 0ull, csec = 0ull;
      long long cidx = 0x7fffffffffffffffLL;
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (st[r] == -1) cand_push(mag_key(v[r][i]), tid + PNT * r, ckey, cidx, csec);
      unsigned long long wk, ws;
      unsigned wi;
      warp_argmax(ckey, (unsigned)cidx, csec, wk, wi, ws, GAPS);
      if (lane == 0) {
        wck[par * PNW + warp] = wk;
        wci[par * PNW + warp] = wk ? (long long)(r0 + wi) : 0x7fffffffffffffffLL;
        wcs[par * PNW + warp] = ws;
      }
      // message = header (2 chunks) + the row's live chunks (columns >= s, rounded to pairs)
      const int jrow0 = 2 + (s >> 1);
      const int nchunk = 2 + (MSG - jrow0);
      if (tid == 0) mbar_arm(mbar0 + 8 * par, (unsigned)(csize * nchunk * 16));
      asm volatile("bar.sync 1, %0;" ::"n"(PNT) : "memory");
      // (B) CTA candidate -> every CTA of the cluster
      {
        const unsigned long long k8 = lane < PNW ? wck[par * PNW + lane] : 0ull;
        const long long i8 = lane < PNW ? wci[par * PNW + lane] : 0x7fffffffffffffffLL;
        const unsigned long long s8 = lane < PNW ? wcs[par * PNW + lane] : 0ull;
        unsigned long long bk, bs;
        unsigned bl;
        warp_argmax(k8, k8 ? (unsigned)(i8 - r0) : 0xffffffffu, s8, bk, bl, bs, GAPS);
        const unsigned wl = __ballot_sync(0xffffffffu, k8 == bk && k8 != 0ull && (unsigned)(i8 - r0) == bl);
        const int cw = wl ? __ffs(wl) - 1 : 0;
        const long long gidx = bk ? r0 + (long long)bl : 0x7fffffffffffffffLL;
        // only the CTA-winning warp's owner lane copies its row (one warp's 16-byte stores instead
        // of all 8 warps'), then every warp sends to its 2 destination CTAs
        if (warp == cw && bk && (int)(bl & 31u) == lane) {
          double* dst = wrow + (size_t)(par * PNW + cw) * NB + cb;
#pragma unroll
          for (int r = 0; r < RPT; ++r)
            if ((int)bl == tid + PNT * r) {
              wlp[par * PNW + cw] = lprev[r];
#pragma unroll
              for (int q = (i & ~1); q + 1 < NB; q += 2)   // live columns, 16-byte stores
                if (cb + q + 1 < NB) *reinterpret_cast<double2*>(dst + q) = make_double2(v[r][q], v[r][q + 1]);
            }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(PNT) : "memory");
        const double* src = wrow + (size_t)(par * PNW + cw) * NB;
        const unsigned slot = mbox_u + (unsigned)(((par * MAXCS) + crank) * MSGD * 8);
        const double lpw = wlp[par * PNW + cw];
        for (int d = warp; d < csize; d += PNW) {
          const unsigned rslot = mapa(slot, (unsigned)d);
          const unsigned rbar = mapa(mbar0 + 8 * par, (unsigned)d);
          for (int jj = lane; jj < nchunk; jj += 32) {
            const int j = jj < 2 ? jj : jrow0 + (jj - 2);
            unsigned long long x, y;
            if (j == 0) { x = bk; y = (unsigned long long)gidx; }
            else if (j == 1) { x = bs; y = (unsigned long long)__double_as_longlong(lpw); }
            else {
              x = (unsigned long long)__double_as_longlong(src[2 * (j - 2)]);
              y = (unsigned long long)__double_as_longlong(src[2 * (j - 2) + 1]);
            }
            st_async_v2(rslot + 16u * j, x, y, rbar);
          }
        }
      }
      // (C) deferred bulk update of step s-1: columns >= s+1 (window q with cb+q >= s+1)
      if (s > 0) {
        const double* uprev = ub + (size_t)(s - 1) * NB + cb;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const double lm = lprev[r];
          if (lm != 0.0) {
            if ((i + 1) & 1) {   // odd start column, then 16-byte pairs of U(s-1, :)
              if (cb + i + 1 < NB) v[r][i + 1] = fma(-lm, uprev[i + 1], v[r][i + 1]);
            }
#pragma unroll
            for (int q = (i + 2) & ~1; q + 1 < NB; q += 2)
              if (cb + q + 1 < NB) {
                const double2 u2 = *reinterpret_cast<const double2*>(uprev + q);
                v[r][q] = fma(-lm, u2.x, v[r][q]);
                v[r][q + 1] = fma(-lm, u2.y, v[r][q + 1]);
              }
          }
        }
      }
      // (D) the cluster's winner and its row
      mbar_wait(mbar0 + 8 * par, (unsigned)((s >> 1) & 1));
      const double* box = mbox + (size_t)par * MAXCS * MSGD;
      const unsigned long long gk = lane < csize ? __double_as_longlong(box[lane * MSGD]) : 0ull;
      const long long gi8 = lane < csize ? __double_as_longlong(box[lane * MSGD + 1]) : 0x7fffffffffffffffLL;
      const unsigned long long gs8 = lane < csize ? __double_as_longlong(box[lane * MSGD + 2]) : 0ull;
      // ties -> lowest global index: CTA row ranges are ordered by rank, so the lowest lane
      unsigned long long wkey, wsec;
      unsigned wlane;
      warp_argmax(gk, gk ? (unsigned)lane : 0xffffffffu, gs8, wkey, wlane, wsec, GAPS);
      // no active row left in this cluster (every key 0, possible when G > 1 and k exceeds the
      // cluster's rows): take slot 0's message so every read below stays in bounds; its key 0
      // never wins the cross-cluster reduction unless every cluster is exhausted (rank failure)
      if (!wkey) wlane = 0;
      long long widx = __shfl_sync(0xffffffffu, gi8, (int)wlane);
      const double* row = box + (size_t)wlane * MSGD + 4;
      double lp = s > 0 ? box[(size_t)wlane * MSGD + 3] : 0.0;
      if (MULTI && p.G > 1) {
        // (D') the G cluster winners meet in global memory: CTA 0 of each cluster publishes its
        // cluster's winning message (release at gpu scope), every CTA waits for all G flags of this
        // step and takes the same winner (max key, ties -> lowest cluster = lowest rows).  Double
        // buffering by parity is safe for the same reason as the cluster mailbox: a cluster publishes
        // step s+2 only after every cluster has published step s+1, i.e. finished reading step s.
        double* gb = p.gbox + (size_t)par * p.G * MSGD;
        const unsigned long long seq = (unsigned long long)t + 1ull;
        if (crank == 0 && tid == 0) {     // one thread writes the message, then releases its flag
          double* dst = gb + (size_t)g * MSGD;
          dst[0] = __longlong_as_double((long long)wkey);
          dst[1] = __longlong_as_double(widx);
          dst[2] = __longlong_as_double((long long)wsec);
          dst[3] = lp;
          for (int j = (s & ~1); j < NB; j += 2)    // live columns, 16-byte stores
            *reinterpret_cast<double2*>(dst + 4 + j) = *reinterpret_cast<const double2*>(row + j);
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.gflag + g), "l"(seq) : "memory");
        }
        if (tid < p.G) {
          const unsigned long long t0 = dev::globaltimer_ns();
          unsigned long long f;
          do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(f) : "l"(p.gflag + tid) : "memory");
            if (f < seq && dev::globaltimer_ns() - t0 > p.timeout_ns) { s_late = 1; break; }
          } while (f < seq);
        }
        asm volatile("bar.sync 4, %0;" ::"n"(PNT) : "memory");
        if (s_late) {
          if (tid == 0) atomicCAS(reinterpret_cast<unsigned long long*>(p.status), 0ull,
                                  (unsigned long long)(-(long long)(t + 1)));
          if (g == 0 && crank == 0)   // as on a rank failure: the undecided pivots read -1
            for (int tt = t + tid; tt < p.k; tt += PNT) p.Js[tt] = -1;
          s_done = s;
          stop = true;
          break;
        }
        // all G messages in one round trip (16-byte loads, every one in flight), then the reduction
        for (int j = tid; j < p.G * (MSGD / 2); j += PNT)
          reinterpret_cast<double2*>(gall)[j] = __ldcg(reinterpret_cast<const double2*>(gb) + j);
        asm volatile("bar.sync 5, %0;" ::"n"(PNT) : "memory");
        const unsigned long long hk = lane < p.G ? (unsigned long long)__double_as_longlong(gall[lane * MSGD]) : 0ull;
        const unsigned long long hs = lane < p.G ? (unsigned long long)__double_as_longlong(gall[lane * MSGD + 2]) : 0ull;
        unsigned wg;
        warp_argmax(hk, hk ? (unsigned)lane : 0xffffffffu, hs, wkey, wg, wsec, GAPS);
        const double* gwin = gall + (size_t)wg * MSGD;
        widx = __double_as_longlong(gwin[1]);
        row = gwin + 4;
        lp = s > 0 ? gwin[3] : 0.0;
      }
      const double a1 = wkey ? __longlong_as_double((long long)(wkey - 1ull)) : -1.0;
      if (!(a1 > tol)) {
        if (g == 0 && crank == 0 && tid == 0) {
          *p.status = t + 1;
          for (int tt = t; tt < p.k; ++tt) p.Js[tt] = -1;
        }
        s_done = s;
        stop = true;
        break;
      }
      const double* uprev = ub + (size_t)(s > 0 ? s - 1 : 0) * NB;
      const double piv = row[s];
      const double u1 = s + 1 < bp ? (s > 0 ? fma(-lp, uprev[s + 1], row[s + 1]) : row[s + 1]) : 0.0;
      if (warp == PNW - 1) {   // U(s, :) for the bulk update of the next step, fix-ups and the output
        double* ucur = ub + (size_t)s * NB;
        for (int c = s + lane; c < bp; c += 32) ucur[c] = (s > 0 && c > s) ? fma(-lp, uprev[c], row[c]) : row[c];
      }
      if (crank == 0 && tid == 0) {
        js[s] = widx;
        if (GAPS) {
          const double a2 = wsec ? __longlong_as_double((long long)(wsec - 1ull)) : 0.0;
          gp[s] = (a1 - a2) / a1;
        }
      }
      // (E) multipliers, the next search column, the L column of step s
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int li = tid + PNT * r;
        double lout = 0.0;
        lprev[r] = 0.0;
        if (st[r] == -1) {
          if (r0 + li == widx) {
            st[r] = t;
            lout = 1.0;
          } else {
            const double lm = v[r][i] / piv;
            v[r][i] = lm;
            if (i + 1 < NB) v[r][i + 1] = fma(-lm, u1, v[r][i + 1]);
            lprev[r] = lm;
            lout = lm;
          }
        }
        if (li < Rc) p.Lf[(r0 + li) + (int64_t)t * p.ldlf] = lout;
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int q = 0; q < NB; ++q) v[r][q] = (q + 8 < NB) ? v[r][q + 8] : 0.0;
  }
  __syncthreads();
  if (g == 0 && crank == 0) {
    for (int s = tid; s < s_done; s += PNT) {
      p.Js[p.c0 + s] = js[s];
      if (GAPS) p.gaps[p.c0 + s] = gp[s];
    }
    for (int e = tid; e < s_done * bp; e += PNT) {
      const int s = e / bp, j = e % bp;
      if (j >= s) p.Uw[(p.c0 + s) + (int64_t)(p.c0 + j) * p.k] = ub[(size_t)s * NB + j];
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = tid + PNT * r;
    if (li < Rc) p.rowstate[r0 + li] = st[r];
  }
  cluster.sync();
}

template <int NB>
constexpr size_t v2_smem_bytes() {
  return sizeof(double) * ((size_t)NB * NB + 2 * PNW * NB) + 4 * 2 * PNW * 8 +
         sizeof(double) * 2 * MAXCS * (4 + NB) + NB * 8 + NB * 8 + 16 + 64;
}

// U(c0+s, j) = M(piv_s, j) - sum_{s'<s} L11(s, s') U(c0+s', j), j in [c1, k).
// One thread per column, the column of U in registers (bp <= U12_BP), L11 broadcast from smem.
// Right-looking: step sp subtracts L11(:, sp) u[sp] from every later row -- the row updates of a step
// are independent (no accumulator chains, the shared-memory loads of a step all in flight at once),
// only u[sp + 1] of the next step waits for one FMA.  L11 is held transposed (L11T[sp][s], rows padded
// to U12_LS) so that one 16-byte broadcast load feeds two rows.
constexpr int U12_LS = U12_BP + 2;
template <int BP>
__device__ __forceinline__ void u12_subst(double (&u)[U12_BP], const double (*L11T)[U12_LS]) {
  static_assert(BP % 2 == 0, "pairs");
#pragma unroll
  for (int sp = 0; sp + 1 < BP; ++sp) {
    const double us = u[sp];
    if ((sp + 1) & 1) u[sp + 1] = fma(-L11T[sp][sp + 1], us, u[sp + 1]);
#pragma unroll
    for (int s = (sp + 2) & ~1; s + 1 < BP; s += 2) {
      const double2 l2 = *reinterpret_cast<const double2*>(&L11T[sp][s]);
      u[s] = fma(-l2.x, us, u[s]);
      u[s + 1] = fma(-l2.y, us, u[s + 1]);
    }
  }
}

__global__ void __launch_bounds__(256) k_lupp_u12(const double* W, int64_t n, int k, int c0, int bp,
                                                  const int64_t* Js, const double* Lf, int64_t ldlf,
                                                  double* Uw, const int64_t* status) {
  dev::griddep_wait();
  if (*status != 0) return;
  extern __shared__ __align__(16) double u12sm[];
  double (*L11T)[U12_LS] = reinterpret_cast<double (*)[U12_LS]>(u12sm);      // L11T[sp][s] = L11(s, sp)
  double (*Wv)[33] = reinterpret_cast<double (*)[33]>(u12sm + U12_BP * U12_LS);
  int64_t* piv = reinterpret_cast<int64_t*>(u12sm + U12_BP * U12_LS + U12_BP * 33);
  const int j0 = c0 + bp + blockIdx.x * 32;
  for (int s = threadIdx.x; s < bp; s += blockDim.x) piv[s] = Js[c0 + s];
  __syncthreads();
  for (int e = threadIdx.x; e < bp * bp; e += blockDim.x) {      // async gathers: all in flight
    const int s = e % bp, sp = e / bp;
    if (sp < s) dev::cp_async8(&L11T[sp][s], Lf + piv[s] + (int64_t)(c0 + sp) * ldlf, true);
  }
  for (int e = threadIdx.x; e < bp * 32; e += blockDim.x) {
    const int s = e % bp, cc = e / bp;
    const int j = j0 + cc;
    dev::cp_async8(&Wv[s][cc], j < k ? W + piv[s] + (int64_t)j * n : W, j < k);
  }
  dev::cp_async_commit();
  dev::cp_async_wait<0>();
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int j = j0 + threadIdx.x;
  if (j >= k) return;
  double u[U12_BP];
#pragma unroll
  for (int s = 0; s < U12_BP; ++s) u[s] = s < bp ? Wv[s][threadIdx.x] : 0.0;
  if (bp == U12_BP) u12_subst<U12_BP>(u, L11T);
  else if (bp == 32) u12_subst<32>(u, L11T);
  else if (bp == 16) u12_subst<16>(u, L11T);
  else {
#pragma unroll
    for (int sp = 0; sp + 1 < U12_BP; ++sp) {
      if (sp + 1 < bp) {
        const double us = u[sp];
#pragma unroll
        for (int s = sp + 1; s < U12_BP; ++s)
          if (s < bp) u[s] = fma(-L11T[sp][s], us, u[s]);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < U12_BP; ++s)
    if (s < bp) Uw[(c0 + s) + (int64_t)j * k] = u[s];
}

constexpr size_t kU12Smem = sizeof(double) * (U12_BP * U12_LS + U12_BP * 33 + U12_BP);

__global__ void k_copy_u(const double* Uw, int k, double* U, int64_t ldu) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % k), j = (int)(e / k);
    U[i + j * ldu] = i <= j ? Uw[e] : 0.0;
  }
}

using PanelFn = void (*)(PanelParams);

struct ClusterCfg {
  int cs = 0;
  bool ok = false;
  int max_dyn = 0;
  std::string why;
};

ClusterCfg pick_cluster(sk_ctx* c) {
  static ClusterCfg cfg_dev[kMaxDevices];                  // function attributes are per device
  static bool done_dev[kMaxDevices] = {};
  ClusterCfg& cfg = cfg_dev[c->device % kMaxDevices];
  bool& done = done_dev[c->device % kMaxDevices];
  if (done) return cfg;
  done = true;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k_lupp_panel<true>);
  cfg.max_dyn = c->max_smem_optin - (int)fa.sharedSizeBytes - 64;
  for (PanelFn fn : {k_lupp_panel<true>, k_lupp_panel<false>}) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.max_dyn);
  }
  for (PanelFn fn : {k_lupp_panel_v2<1, 64, true, false>, k_lupp_panel_v2<1, 64, false, false>,
                     k_lupp_panel_v2<2, 32, true, false>, k_lupp_panel_v2<2, 32, false, false>,
                     k_lupp_panel_v2<4, 16, true, false>, k_lupp_panel_v2<4, 16, false, false>,
                     k_lupp_panel_v2<1, 64, true, true>, k_lupp_panel_v2<1, 64, false, true>,
                     k_lupp_panel_v2<2, 32, true, true>, k_lupp_panel_v2<2, 32, false, true>,
                     k_lupp_panel_v2<4, 16, true, true>, k_lupp_panel_v2<4, 16, false, true>}) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v2_smem_bytes<64>());
  }
  cudaFuncSetAttribute(k_lupp_u12, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kU12Smem);
  for (int cs : {16, 8, 4, 2, 1}) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(PNT);
    lc.dynamicSmemBytes = (size_t)cfg.max_dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    lc.attrs = at; lc.numAttrs = 1;
    int nclusters = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, k_lupp_panel<true>, &lc);
    if (e == cudaSuccess && nclusters > 0) {
      cfg.cs = cs; cfg.ok = true;
      break;
    }
    cfg.why += "cs=" + std::to_string(cs) + ": " + cudaGetErrorString(e) + " (" + std::to_string(nclusters) + "); ";
    cudaGetLastError();
  }
  return cfg;
}

}  // namespace

int64_t lupp_max_rows(sk_ctx* c) {
  const ClusterCfg cfg = pick_cluster(c);
  return cfg.ok ? (int64_t)cfg.cs * 16 * PNT : 0;
}

sk_status ensure_aux(sk_ctx* c) {
  if (c->aux) return SK_OK;
  int lo = 0, hi = 0;
  SK_CUDA(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  SK_CUDA(c, cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, lo));   // lo = least priority
  SK_CUDA(c, cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming));
  SK_CUDA(c, cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming));
  return SK_OK;
}

sk_status lupp(sk_ctx* c, const double* Pin, bool row_major, int64_t n, int64_t k, int64_t ld,
               int64_t* Js, double* Lf, int64_t ldlf, double* U, int64_t ldu, double* gaps,
               int64_t* status_dev) {
  const ClusterCfg cfg = pick_cluster(c);
  if (!cfg.ok) return fail(c, SK_E_CUDA, "no thread-block cluster configuration for the LUPP panel: " + cfg.why);
  int cs = cfg.cs;
  int64_t R = cdiv(n, cs);
  // Tall panels (more than 4 rows per thread in one cluster): G co-resident clusters of the
  // register-resident v2 kernel, whose winners meet in global memory once per step, instead of
  // one cluster streaming thousands of rows per CTA.  For k >= 512 the fewest rows per thread
  // first (wider column blocks, fewer block transitions: C5 columns 10.5 vs 11.4 us/step), else the
  // fewest clusters (cheaper per-step exchange: C4 rows 6.0 vs 7.0 us/step); then the larger cluster.
  int G = 1;
  if (cdiv(R, PNT) > 4) {
    bool found = false;
    const int order_wide[3] = {1, 2, 4}, order_few[3] = {4, 2, 1};
    const int* order = k >= 512 ? order_wide : order_few;
    for (int oi = 0; oi < 3; ++oi) {
      const int target = order[oi];
      for (int ccs : {cfg.cs, cfg.cs / 2, cfg.cs / 4}) {
        if (ccs < 2) continue;
        const int gg = (int)cdiv(n, (int64_t)ccs * PNT * target);
        if (gg < 2 || gg > kMaxG) continue;
        PanelFn f = target == 1 ? k_lupp_panel_v2<1, 64, true, true> : target == 2 ? k_lupp_panel_v2<2, 32, true, true>
                                                                                   : k_lupp_panel_v2<4, 16, true, true>;
        cudaLaunchConfig_t oc{};
        oc.gridDim = dim3((unsigned)(ccs * gg));
        oc.blockDim = dim3(PNT);
        oc.dynamicSmemBytes = v2_smem_bytes<64>();
        cudaLaunchAttribute oa[1];
        oa[0].id = cudaLaunchAttributeClusterDimension;
        oa[0].val.clusterDim.x = ccs; oa[0].val.clusterDim.y = 1; oa[0].val.clusterDim.z = 1;
        oc.attrs = oa; oc.numAttrs = 1;
        int active = 0;
        if (cudaOccupancyMaxActiveClusters(&active, f, &oc) != cudaSuccess) { cudaGetLastError(); active = 0; }
        if (gg <= active) {
          G = gg;
          cs = ccs;
          R = cdiv(n, (int64_t)cs * G);
          found = true;
          break;
        }
      }
      if (found) break;
    }
  }
  if (R > 16 * PNT) return fail(c, SK_E_ARG, "LUPP panel too tall for one cluster (n too large)");
  // register-resident kernel when a thread's rows x block fit 64 doubles, else the
  // shared-memory kernel with the widest block whose rows fit the cluster's shared memory
  PanelFn fn = nullptr;
  int64_t bp = 0;
  size_t smem_bytes = 0;
  const int rpt = (int)cdiv(R, PNT);
  if (rpt <= 4) {
    const int nb = rpt == 1 ? 64 : rpt == 2 ? 32 : 16;
    bp = std::min<int64_t>(k, nb);
    const bool multi = G > 1;      // the cross-cluster exchange is compiled only into the G > 1 variants
    if (rpt == 1) {
      fn = multi ? (gaps ? k_lupp_panel_v2<1, 64, true, true> : k_lupp_panel_v2<1, 64, false, true>)
                 : (gaps ? k_lupp_panel_v2<1, 64, true, false> : k_lupp_panel_v2<1, 64, false, false>);
      smem_bytes = v2_smem_bytes<64>();
    } else if (rpt == 2) {
      fn = multi ? (gaps ? k_lupp_panel_v2<2, 32, true, true> : k_lupp_panel_v2<2, 32, false, true>)
                 : (gaps ? k_lupp_panel_v2<2, 32, true, false> : k_lupp_panel_v2<2, 32, false, false>);
      smem_bytes = v2_smem_bytes<32>();
    } else {
      fn = multi ? (gaps ? k_lupp_panel_v2<4, 16, true, true> : k_lupp_panel_v2<4, 16, false, true>)
                 : (gaps ? k_lupp_panel_v2<4, 16, true, false> : k_lupp_panel_v2<4, 16, false, false>);
      smem_bytes = v2_smem_bytes<16>();
    }
  } else {
    bp = std::min<int64_t>(k, 1024);
    while (bp > 1 && (int64_t)PanelSmem((int)R, (int)bp).total > cfg.max_dyn) bp = (bp > 64) ? bp / 2 : bp - 1;
    if (bp < k) bp = std::min<int64_t>(bp, U12_BP);
    fn = gaps ? k_lupp_panel<true> : k_lupp_panel<false>;
    smem_bytes = PanelSmem((int)R, (int)bp).total;
  }
  if ((int64_t)smem_bytes > cfg.max_dyn) return fail(c, SK_E_ARG, "LUPP panel staging exceeds shared memory");

  DBuf Wb, Ub, stateb, maxb, Lfb;
  DBuf gxb;
  const size_t gbox_doubles = (size_t)2 * G * (4 + 64);
  if (G > 1) {
    SK_TRY(gxb.alloc(c, gbox_doubles * sizeof(double) + (size_t)G * sizeof(unsigned long long)));
    SK_CUDA(c, cudaMemsetAsync(gxb.p, 0, gbox_doubles * sizeof(double) + (size_t)G * sizeof(unsigned long long),
                               c->stream));
  }
  SK_TRY(Wb.alloc(c, (size_t)n * k * sizeof(double)));
  SK_TRY(Ub.alloc(c, (size_t)k * k * sizeof(double)));
  SK_TRY(stateb.alloc(c, (size_t)n * sizeof(int)));
  SK_TRY(maxb.alloc(c, sizeof(unsigned long long)));
  if (!Lf) {
    SK_TRY(Lfb.alloc(c, (size_t)n * k * sizeof(double)));
    Lf = Lfb.as<double>();
    ldlf = n;
  }
  SK_CUDA(c, cudaMemsetAsync(maxb.p, 0, sizeof(unsigned long long), c->stream));
  SK_CUDA(c, cudaMemsetAsync(status_dev, 0, sizeof(int64_t), c->stream));
  {
    k_lupp_init<<<dim3((unsigned)cdiv(n, 1024), (unsigned)k), 256, 0, c->stream>>>(Pin, row_major, n, (int)k, ld, Wb.as<double>(),
                                               stateb.as<int>(), maxb.as<unsigned long long>());
    SK_TRY(launched(c));
  }
  // programmatic dependent launch along the panel -> u12 -> next-block GEMM -> panel chain
  constexpr bool pdl = true;
  const bool lookahead = bp < k;
  if (lookahead) SK_TRY(ensure_aux(c));
  bool rest_pending = false;
  for (int64_t c0 = 0; c0 < k; c0 += bp) {
    const int b = (int)std::min<int64_t>(bp, k - c0);
    PanelParams pp{};
    pp.W = Wb.as<double>(); pp.n = n; pp.k = (int)k;
    pp.c0 = (int)c0; pp.bp = b; pp.R = (int)R;
    pp.rowstate = stateb.as<int>();
    pp.Js = Js; pp.Lf = Lf; pp.ldlf = ldlf; pp.Uw = Ub.as<double>(); pp.gaps = gaps;
    pp.maxbits = maxb.as<unsigned long long>(); pp.status = status_dev;
    pp.G = G;
    pp.gbox = G > 1 ? gxb.as<double>() : nullptr;
    pp.gflag = G > 1 ? reinterpret_cast<unsigned long long*>(gxb.as<double>() + gbox_doubles) : nullptr;
    pp.timeout_ns = 10ull * 1000 * 1000 * 1000;      // a cluster that never publishes: SK_E_STATE, not a hang
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)(cs * G));
    lc.blockDim = dim3(PNT);
    lc.dynamicSmemBytes = smem_bytes;
    lc.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at; lc.numAttrs = pdl ? 2 : 1;             // block 0: the predecessor is k_lupp_init
    SK_CUDA(c, cudaLaunchKernelEx(&lc, fn, pp));
    SK_TRY(launched(c));
    const int64_t c1 = c0 + b;
    if (c1 < k) {
      // look-ahead: the next block's columns are updated on the main stream; the rest of the
      // trailing update runs on the low-priority aux stream, overlapping the next panel
      const bool waited = rest_pending;
      if (rest_pending) SK_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_b, 0));   // before u12 reads W(piv, c1:)
      rest_pending = false;
      {
        cudaLaunchConfig_t lu{};
        lu.gridDim = dim3((unsigned)cdiv(k - c1, 32));
        lu.blockDim = dim3(256);
        lu.dynamicSmemBytes = kU12Smem;
        lu.stream = c->stream;
        cudaLaunchAttribute au[1];
        au[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        au[0].val.programmaticStreamSerializationAllowed = 1;
        lu.attrs = au; lu.numAttrs = (pdl && !waited) ? 1 : 0;      // an event wait keeps full ordering
        SK_CUDA(c, cudaLaunchKernelEx(&lu, k_lupp_u12, (const double*)Wb.as<double>(), n, (int)k, (int)c0, b,
                                      (const int64_t*)Js, (const double*)Lf, ldlf, Ub.as<double>(),
                                      (const int64_t*)status_dev));
        SK_TRY(launched(c));
      }
      const int64_t nn = lookahead ? std::min<int64_t>(bp, k - c1) : k - c1;
      c->pdl = pdl;
      const sk_status gs = gemm(c, false, false, n, nn, b, -1.0, Lf + c0 * ldlf, ldlf, Ub.as<double>() + c0 + c1 * k,
                                k, 1.0, Wb.as<double>() + c1 * n, n);
      c->pdl = false;
      SK_TRY(gs);
      if (c1 + nn < k) {
        SK_CUDA(c, cudaEventRecord(c->ev_a, c->stream));
        SK_CUDA(c, cudaStreamWaitEvent(c->aux, c->ev_a, 0));
        cudaStream_t main_stream = c->stream;
        c->stream = c->aux;
        const sk_status st = gemm(c, false, false, n, k - c1 - nn, b, -1.0, Lf + c0 * ldlf, ldlf,
                                  Ub.as<double>() + c0 + (c1 + nn) * k, k, 1.0, Wb.as<double>() + (c1 + nn) * n, n);
        c->stream = main_stream;
        SK_TRY(st);
        SK_CUDA(c, cudaEventRecord(c->ev_b, c->aux));
        rest_pending = true;
      }
    }
  }
  if (rest_pending) SK_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_b, 0));
  if (U) {
    const int blocks = (int)std::min<int64_t>(cdiv(k * k, 256), 4LL * c->num_sms);
    k_copy_u<<<blocks, 256, 0, c->stream>>>(Ub.as<double>(), (int)k, U, ldu);
    SK_TRY(launched(c));
  }
  return SK_OK;
}

}  // namespace skel
