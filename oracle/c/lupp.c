/* lupp.c -- the oracle's k-step swap-free LUPP in plain C (TEST INFRASTRUCTURE ONLY).
 *
 * The same algorithm, step for step and rounding for rounding, as oracle/lupp.py::lupp_panel
 * (eq:def_LUPP and the pivot rule; readings R5-R7 of DESIGN.md section 3), written as
 * plain loops so that panels of 65536-131072 rows and k = 1000 (BASELINE C5) finish in seconds:
 *
 *   for t = 0 .. k-1:
 *     p_t = argmax over active rows i of |W(i, t)|, ties to the lowest original index (R6)
 *     gap_t = (a1 - a2) / a1 with a2 the largest |W(i, t)| over the other active rows
 *     (forced[t] >= 0 replaces p_t: the parity harness's near-tie rule)
 *     rank failure if !(a1 > 1e-14 * max|W(:, 0:k)|)  -> return t + 1 (R7)
 *     U(t, t:) = W(p_t, t:);  Lf(p_t, t) = 1;  row p_t leaves the active set
 *     every active row i:  L = W(i, t) / W(p_t, t);  Lf(i, t) = L;
 *                          W(i, c) = W(i, c) - L * U(t, c)   for c = t+1 .. k-1
 *
 * Compiled with -ffp-contract=off, so each update is a rounded product followed by a rounded
 * subtraction -- exactly numpy's `W[rows, t+1:] -= np.outer(mult, U[t, t+1:])`.  The loops over
 * rows are split across OpenMP threads; the argmax merges per-thread candidates with the
 * lowest-index tie rule, so the result does not depend on the thread count.
 * Shares no code with the CUDA path (paper_2104_05877_b200/csrc).
 *
 * W: n x k row-major (overwritten).  Outputs: piv[k], Lf n x k row-major (zero-initialised by the
 * caller), U k x k row-major (zero-initialised), gaps[k].  Returns 0 or the 1-based failing step.
 */
#include <math.h>
#include <stdint.h>

typedef struct { double v1; int64_t i1; double v2; } top2;

static top2 merge(top2 a, top2 b) {
  top2 r;
  if (b.v1 > a.v1 || (b.v1 == a.v1 && b.i1 < a.i1 && b.i1 >= 0)) {
    r.v1 = b.v1; r.i1 = b.i1;
    r.v2 = fmax(a.v1, fmax(a.v2, b.v2));
  } else {
    r.v1 = a.v1; r.i1 = a.i1;
    r.v2 = fmax(b.v1, fmax(a.v2, b.v2));
  }
  return r;
}

int64_t or_lupp_panel(double* W, int64_t n, int64_t k, const int64_t* forced, int64_t* piv, double* Lf,
                      double* U, double* gaps, unsigned char* active) {
  double scale = 0.0;
#pragma omp parallel for reduction(max : scale)
  for (int64_t e = 0; e < n * k; ++e) scale = fmax(scale, fabs(W[e]));
  for (int64_t i = 0; i < n; ++i) active[i] = 1;
  for (int64_t t = 0; t < k; ++t) {
    top2 best = {-1.0, -1, -1.0};
#pragma omp parallel
    {
      top2 loc = {-1.0, -1, -1.0};
#pragma omp for schedule(static) nowait
      for (int64_t i = 0; i < n; ++i) {
        if (!active[i]) continue;
        const double a = fabs(W[i * k + t]);
        if (a > loc.v1) { loc.v2 = loc.v1; loc.v1 = a; loc.i1 = i; }
        else if (a > loc.v2) loc.v2 = a;
      }
#pragma omp critical
      best = merge(best, loc);
    }
    int64_t p = best.i1;
    double a1 = best.v1;
    const double a2 = best.v2 > 0.0 ? best.v2 : 0.0;
    gaps[t] = a1 > 0.0 ? (a1 - a2) / a1 : 0.0;
    if (forced && forced[t] >= 0) {
      p = forced[t];
      a1 = fabs(W[p * k + t]);
    }
    if (!(a1 > 1e-14 * scale)) return t + 1;
    piv[t] = p;
    for (int64_t c = t; c < k; ++c) U[t * k + c] = W[p * k + c];
    active[p] = 0;
    Lf[p * k + t] = 1.0;
    const double pv = W[p * k + t];
    const double* u = U + t * k;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      if (!active[i]) continue;
      double* w = W + i * k;
      const double L = w[t] / pv;
      Lf[i * k + t] = L;
      for (int64_t c = t + 1; c < k; ++c) w[c] = w[c] - L * u[c];
    }
  }
  return 0;
}
