// Table-driven fp64 exp / log for the EM kernel.
//
// CUDA's exp()/log() for double are ~35 fp64-pipe instructions each once the
// range checks and polynomial are counted; the EM evaluates 52 of them per
// coefficient per iteration and is fp64-pipe bound.  These versions use a
// 64-entry 2^(j/64) table (exp) and a 128-entry reciprocal table (log), held
// in shared memory, so each costs ~13 fp64 instructions with ~1 ulp error:
//   exp(z) = 2^m * 2^(j/64) * (1 + p(r)),  z = (64m + j) ln2/64 + r, |r| <= ln2/128
//   log(x) = e ln2 - ln(c_j) + log1p(r),   r = m c_j - 1 (one FMA), |r| <= 2^-8
// The EM's discrete decisions (fit counts) need only ~1e-12 relative
// fidelity to the reference's libm (bayes.py:106-111); these are ~1e-16.
// Domain: exp for |z| < 700 (results normal), log for normal x > 0 -- the EM
// clamps every spectrum at epsilon > 0 before the log (bayes.py:107).
#pragma once

#include "oxm_common.cuh"
#include "oxm_tables.h"

namespace oxm {

// ln 2 split with a 42-bit high part so e * kLn2Hi42 is exact for |e| < 2^11
constexpr double kLn2Hi42 = 0.693147180559890330187045037746;  // 0x3FE62E42FEFA3800
constexpr double kLn2Lo42 = 5.4979230187083711552420206e-14;   // ln2 - kLn2Hi42

// One shared-memory access per transcendental: exp reads 2^(j/64) (the lo
// correction is dropped: +0.5 ulp), log reads (c_j, -ln c_j) as one 16-byte
// word (the lo part of -ln c_j is below 2^-60 absolute and is dropped too).
struct MathSmem {
  double expt[64];   // 2^(j/64)
  double2 logt[128]; // (c_j, -ln(c_j))
};

__device__ __forceinline__ void load_math_tables(MathSmem& t) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    if (i < 64) t.expt[i] = kExpTable[i][0];
    t.logt[i] = make_double2(kLogTable[i][0], kLogTable[i][1] + kLogTable[i][2]);
  }
}

__device__ __forceinline__ double exp_tab(const double z, const MathSmem& t) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest integer trick
  const double km = fma(z, k64OverLn2, magic);
  const int k = __double2loint(km);
  const double kd = km - magic;
  double r = fma(-kd, kLn2Over64Hi, z);
  r = fma(-kd, kLn2Over64Lo, r);
  double q = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  q = fma(q, r, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  const double p = fma(q, r * r, r);  // exp(r) - 1
  const double T = t.expt[k & 63];
  const double res = fma(T, p, T);
  const int m = k >> 6;  // floor(k / 64)
  return __hiloint2double(__double2hiint(res) + (m << 20), __double2loint(res));
}

__device__ __forceinline__ double log_tab(const double x, const MathSmem& t) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);  // [1, 2)
  const double2 cj = t.logt[j];
  const double r = fma(m, cj.x, -1.0);
  double q = fma(r, 1.0 / 7.0, -1.0 / 6.0);
  q = fma(q, r, 0.2);
  q = fma(q, r, -0.25);
  q = fma(q, r, 1.0 / 3.0);
  q = fma(q, r, -0.5);
  const double ed = (double)e;
  const double h = fma(ed, kLn2Hi42, cj.y);
  return h + (r + fma(q, r * r, ed * kLn2Lo42));
}

}  // namespace oxm
