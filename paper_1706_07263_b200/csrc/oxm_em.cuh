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
//
// Performance shape (fp64-pipe bound): the expected spectrum e (L doubles)
// lives in shared memory, not registers, and the band loops are only 2-way
// unrolled around the table-driven exp/log of oxm_math.cuh, so the kernel is
// ~70 registers (>= 7 warps / scheduler) and its loop fits the instruction
// cache.  The stopping test compares squared norms (no sqrt/div); it differs
// from the reference's rel < tol only when rel is within ~1e-16 of tol.
#pragma once

#include "oxm_common.cuh"
#include "oxm_math.cuh"

namespace oxm {

template <int KL>
struct BandCount {
  static constexpr int kMax = KL > 0 ? KL : kMaxBands;
  __device__ __forceinline__ static int get(const DevOps& ops) { return KL > 0 ? KL : ops.L; }
};

// Runs the estimator for one coefficient.  `init` (stride 1) may be null.
// `e` is this thread's shared-memory column (element l at e[l * es]).
// On return x[] holds the final concentrations, fits the fit count, and the
// final spectrum has been passed to `store(l, value)`.
template <int KL, typename Store>
__device__ __forceinline__ void em_coefficient(const DevOps& ops, const MathSmem& mt, double* __restrict__ e,
                                               const int es, const double y0, const double y1, const double y2,
                                               const double* init, double& x0, double& x1, double& x2, int& fits,
                                               Store store) {
  const int L = BandCount<KL>::get(ops);
  const double eps = ops.eps;

  // fit #1 of the (clamped) start spectrum
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll 2
  for (int l = 0; l < L; ++l) {
    double s = init ? init[l] : fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0));
    const double lg = log_tab(fmax(s, eps), mt);
    a0 = fma(ops.fitm[0][l], lg, a0);
    a1 = fma(ops.fitm[1][l], lg, a1);
    a2 = fma(ops.fitm[2][l], lg, a2);
  }
  x0 = -a0;
  x1 = -a1;
  x2 = -a2;

  const double tol2 = ops.rel_tol * ops.rel_tol;
  double r0 = 0.0, r1 = 0.0, r2 = 0.0;
  int nfit = 1;
  for (int it = 1; it < ops.max_iters; ++it) {
    // expected spectrum e = exp(-xi x) and its RGB projection C e
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll 2
    for (int l = 0; l < L; ++l) {
      // xi[:, 2] == 1 by the ChromophoreBasis contract (core.py:152-153)
      const double arg = fma(ops.xi[l][0], x0, fma(ops.xi[l][1], x1, x2));
      const double el = exp_tab(-arg, mt);
      e[l * es] = el;
      c0 = fma(ops.sens[0][l], el, c0);
      c1 = fma(ops.sens[1][l], el, c1);
      c2 = fma(ops.sens[2][l], el, c2);
    }
    r0 = y0 - c0;
    r1 = y1 - c1;
    r2 = y2 - c2;
    // shape-prior update and fit
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;
#pragma unroll 2
    for (int l = 0; l < L; ++l) {
      const double s = fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, e[l * es])));
      const double lg = log_tab(fmax(s, eps), mt);
      n0 = fma(ops.fitm[0][l], lg, n0);
      n1 = fma(ops.fitm[1][l], lg, n1);
      n2 = fma(ops.fitm[2][l], lg, n2);
    }
    n0 = -n0;
    n1 = -n1;
    n2 = -n2;
    ++nfit;
    const double d0 = n0 - x0, d1 = n1 - x1, d2 = n2 - x2;
    const double dn2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
    const double xn2 = __dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)), __dmul_rn(x2, x2));
    x0 = n0;
    x1 = n1;
    x2 = n2;
    if (dn2 < tol2 * fmax(xn2, 1e-16)) break;  // rel < rel_tol (bayes.py:200-204)
  }
  fits = nfit;

  // final spectrum: the last update (recomputed from e, r) or the start
  if (nfit > 1) {
    for (int l = 0; l < L; ++l)
      store(l, fmax(fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, e[l * es]))), eps));
  } else {
    for (int l = 0; l < L; ++l) {
      const double s = init ? init[l] : fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0));
      store(l, fmax(s, eps));
    }
  }
}

// Dynamic shared memory of an EM kernel: tables + one e column per thread.
__host__ __device__ constexpr size_t em_smem_bytes(int L, int threads) {
  return sizeof(MathSmem) + sizeof(double) * (size_t)L * (size_t)threads;
}

}  // namespace oxm
