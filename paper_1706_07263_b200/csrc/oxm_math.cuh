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

// fp64 SASS instructions take 32-bit immediates (the high word of a double
// whose low word is zero) but no constant-bank operands, so every other
// constant must be (re)materialised in registers inside the loop.  Constants
// below are therefore split or rounded to 20-bit-mantissa "immediate" doubles
// wherever the accuracy budget allows; only four full-precision constants
// remain (kExpLo, kInv6, kInv3, kLn2Lo20).
constexpr double k64OverLn2I = 92.33245849609375;        // 0x4057154700000000 (rounding only)
constexpr double kLn2Over64I = 0.010830417275428772;     // 0x3F862E4200000000 = hi part of ln2/64
constexpr double kExpLo = 7.420820373486988e-09;         // ln2/64 - kLn2Over64I
constexpr double kLn2I = 0.6931467056274414;             // 0x3FE62E4200000000 = hi part of ln2
constexpr double kLn2Lo20 = 4.7493250390316726e-07;      // ln2 - kLn2I
constexpr double kInv6 = 1.0 / 6.0;
constexpr double kInv3 = 1.0 / 3.0;
// 20-bit-mantissa polynomial tail coefficients: |error| contributions below
// 1e-17 relative for |r| <= ln2/128 (exp) and |r| <= 2^-8 (log)
constexpr double kC720 = 0.00138888880610466;
constexpr double kC120 = 0.00833333283662796;
constexpr double kC24 = 0.041666656732559204;
constexpr double kC7 = 0.14285719394683838;
constexpr double kCm6 = -0.16666662693023682;
constexpr double kC5 = 0.20000004768371582;

// One shared-memory access per transcendental: exp reads 2^(j/64) (the lo
// correction is dropped: +0.5 ulp), log reads (c_j, -ln c_j) as one 16-byte
// word (the lo part of -ln c_j is below 2^-60 absolute and is dropped too).
struct MathSmem {
  double expt[64];   // 2^(j/64)
  double2 logt[128]; // (c_j, -ln(c_j))
  double expt2[64];  // 2^(j/4096) (2-level exp)
};

__device__ __forceinline__ void load_math_tables(MathSmem& t) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    if (i < 64) {
      t.expt[i] = kExpTable[i][0];
      t.expt2[i] = kExpTable2[i];
    }
    t.logt[i] = make_double2(kLogTable[i][0], kLogTable[i][1] + kLogTable[i][2]);
  }
}

__device__ __forceinline__ double exp_tab(const double z, const MathSmem& t) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest integer trick
  const double km = fma(z, k64OverLn2I, magic);
  const int k = __double2loint(km);
  const double kd = km - magic;
  double r = fma(-kd, kLn2Over64I, z);  // exact: kd * kLn2Over64I has <= 32 significant bits
  r = fma(-kd, kExpLo, r);
  double q = fma(r, kC720, kC120);
  q = fma(q, r, kC24);
  q = fma(q, r, kInv6);
  q = fma(q, r, 0.5);
  const double p = fma(q, r * r, r);  // exp(r) - 1
  const double T = t.expt[k & 63];
  const double res = fma(T, p, T);
  const int m = k >> 6;  // floor(k / 64)
  return __hiloint2double(__double2hiint(res) + (m << 20), __double2loint(res));
}

// 2-level variant: z = (4096 m + 64 j1 + j2) ln2/4096 + r, |r| <= ln2/8192,
// exp(r) - 1 = r + r^2/2 + r^3/6 (next term 2e-18): 9 fp64 ops + 2 lookups.
__device__ __forceinline__ double exp_tab2(const double z, const MathSmem& t) {
  const double magic = 6755399441055744.0;
  const double km = fma(z, k4096OverLn2I, magic);
  const int k = __double2loint(km);
  const double kd = km - magic;
  double r = fma(-kd, kLn2Over4096I, z);  // exact: kd * kLn2Over4096I has <= 40 significant bits
  r = fma(-kd, kExp2Lo, r);
  const double q = fma(r, kInv6, 0.5);
  const double p = fma(q, r * r, r);
  const double T = t.expt[(k >> 6) & 63] * t.expt2[k & 63];
  const double res = fma(T, p, T);
  const int m = k >> 12;
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
  double q = fma(r, kC7, kCm6);
  q = fma(q, r, kC5);
  q = fma(q, r, -0.25);
  q = fma(q, r, kInv3);
  q = fma(q, r, -0.5);
  const double ed = (double)e;
  const double h = fma(ed, kLn2I, cj.y);  // ed * kLn2I exact (20 x 11 bits)
  return h + (r + fma(q, r * r, ed * kLn2Lo20));
}

}  // namespace oxm
