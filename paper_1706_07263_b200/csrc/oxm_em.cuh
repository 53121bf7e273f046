// K4 core: the iterative shape-prior ("Bayes") estimator for one low-pass
// coefficient, in fp64.  Device-inline so the fused hybrid kernel and the
// standalone estimate_lowpass kernel share one implementation.
//
// Reference: bayes.py:185-207 (_iterate_block), bayes.py:241-250 (start),
// bayes.py:96-111 (_BeerLambertFit), bayes.py:114-135 (_ShapePriorSolver).
// Per coefficient, with y the unit-scale RGB:
//   s  = max(solve y, eps)            (or max(init, eps))
//   x  = -F log(s)                    fit #1
//   repeat while fits < max_iters:
//     e  = exp(-xi x)
//     s' = max(N^-1 (C^T y + P e), eps)       evaluated as  e + G (y - C e)
//     x' = -F log(s')                 fit #k
//     rel = |x' - x| / max(|x|, 1e-8);  s, x <- s', x';  stop if rel < tol
// N^-1 P = I - N^-1 C^T C (N = C^T C + P) makes the 26x26 prior solve a
// rank-3 update: 78+78 FMAs instead of a 676-FMA dense matvec.
#pragma once

#include "oxm_common.cuh"

namespace oxm {

template <int KL>
struct BandCount {
  static constexpr int kMax = KL > 0 ? KL : kMaxBands;
  __device__ __forceinline__ static int get(const DevOps& ops) { return KL > 0 ? KL : ops.L; }
};

// Runs the estimator for one coefficient.  `init` (stride 1) may be null.
// On return x[] holds the final concentrations, fits the fit count and s_out
// receives the final spectrum through the functor `store(l, value)`.
template <int KL, typename Store>
__device__ __forceinline__ void em_coefficient(const DevOps& ops, const double y0, const double y1,
                                               const double y2, const double* init, double& x0,
                                               double& x1, double& x2, int& fits, Store store) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  const double eps = ops.eps;

  // fit #1 of the (clamped) start spectrum
  x0 = 0.0;
  x1 = 0.0;
  x2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
  for (int l = 0; l < LM; ++l) {
    if (KL == 0 && l >= L) break;
    double s;
    if (init) {
      s = init[l];
    } else {
      s = fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0));
    }
    s = fmax(s, eps);
    const double lg = log(s);
    x0 = fma(ops.fitm[0][l], lg, x0);
    x1 = fma(ops.fitm[1][l], lg, x1);
    x2 = fma(ops.fitm[2][l], lg, x2);
  }
  x0 = -x0;
  x1 = -x1;
  x2 = -x2;

  double e[LM];
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  int nfit = 1;
  for (int it = 1; it < ops.max_iters; ++it) {
    // expected spectrum e = exp(-xi x) and its RGB projection C e
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      const double arg = fma(ops.xi[l][2], x2, fma(ops.xi[l][1], x1, ops.xi[l][0] * x0));
      const double el = exp(-arg);
      e[l] = el;
      c0 = fma(ops.sens[0][l], el, c0);
      c1 = fma(ops.sens[1][l], el, c1);
      c2 = fma(ops.sens[2][l], el, c2);
    }
    r0 = y0 - c0;
    r1 = y1 - c1;
    r2 = y2 - c2;
    // shape-prior update and fit
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      const double s = fmax(fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, e[l]))), eps);
      const double lg = log(s);
      n0 = fma(ops.fitm[0][l], lg, n0);
      n1 = fma(ops.fitm[1][l], lg, n1);
      n2 = fma(ops.fitm[2][l], lg, n2);
    }
    n0 = -n0;
    n1 = -n1;
    n2 = -n2;
    ++nfit;
    // relative change, as np.linalg.norm(new - prev) / max(norm(prev), 1e-8)
    const double d0 = n0 - x0, d1 = n1 - x1, d2 = n2 - x2;
    const double dn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
    const double xn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)), __dmul_rn(x2, x2)));
    const double rel = dn / fmax(xn, 1e-8);
    x0 = n0;
    x1 = n1;
    x2 = n2;
    if (rel < ops.rel_tol) break;
  }
  fits = nfit;

  // final spectrum: the last update (recomputed from e, r) or the start
  if (nfit > 1) {
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      store(l, fmax(fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, e[l]))), eps));
    }
  } else {
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      double s = init ? init[l] : fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0));
      store(l, fmax(s, eps));
    }
  }
}

}  // namespace oxm
