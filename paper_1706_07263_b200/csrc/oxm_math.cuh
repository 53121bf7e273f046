// Table-driven fp64 exp / log for the EM kernel.
//
// CUDA's exp()/log() for double are ~35 fp64-pipe instructions each once the
// range checks and polynomial are counted; the EM evaluates 52 of them per
// coefficient per iteration and is fp64-pipe bound.  These versions use a
// 256-entry 2^(j/256) table (exp) and a 256-entry reciprocal table (log), held
// in shared memory, so each costs 8-10 fp64 instructions with ~1 ulp error:
//   exp:  zs = z * 256/ln2 = 256 m + j + rs, |rs| <= 1/2
//         exp(z) = 2^m * 2^(j/256) * (1 + p(rs)),  p: degree 4, Horner in rs
//   log:  log(x) = e ln2 - ln(c_j) + log1p(r),  r = m c_j - 1 (one FMA), |r| <= 2^-9
// The EM passes zs directly (its xi columns are pre-scaled by 256/ln2 on the
// host, DevOps::xis), which folds the argument scaling into the operator and
// makes the reduction rs = zs - round(zs) exact.  Polynomial truncation errors
// are < 5e-18 (tools/gen_math_tables.py fits them at Chebyshev nodes).
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
// constant is (re)materialised in registers.  Polynomial tail coefficients
// are rounded to such 20-bit-mantissa immediates where the accuracy budget
// allows (oxm_tables.h); the full-precision ones are kExpA1..A3, kLogB3 and
// kLn2Lo20.

// One table access per transcendental: exp reads 2^(j/256) (the lo
// correction is dropped: +0.5 ulp), log reads (c_j, -ln c_j) as one 16-byte
// word (the lo part of -ln c_j is below 2^-60 absolute and is dropped too).
struct MathSmem {
  double expt[256];   // 2^(j/256)
  double2 logt[256];  // (c_j, -ln(c_j))
};

__device__ __forceinline__ void load_math_tables(MathSmem& t) {
  const double2* lg = reinterpret_cast<const double2*>(kLogPair);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.expt[i] = kExpTable[i];
    t.logt[i] = lg[i];
  }
}

// the log table in global memory, for kernels too short-lived to stage it
__device__ __forceinline__ const double2* log_table_global() { return reinterpret_cast<const double2*>(kLogPair); }

// MUFU (XU pipe) fp32 transcendentals: ~2 ulp, no range handling
__device__ __forceinline__ float ex2_approx(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float lg2_approx(float v) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// 2^t for a pair on the FMA pipe (FADD2/FFMA2 + two integer adds), < 2 ulp like
// ex2.approx: t clamped to [-125, 127] (the lead-in's e feeds sums with the eps
// clamp downstream, so 2^-125 for an underflowing band is as good as 0), rounded
// with the 1.5 * 2^23 trick, 2^r on [-1/2, 1/2] by a degree-5 fit at Chebyshev
// nodes, then n added to the exponent field ((0x4B400000 + n) << 23 == n << 23
// mod 2^32).  Lets the MUFU-bound fp32 EM lead-in move a share of its ex2s off
// the XU pipe.
__device__ __forceinline__ float2 ex2_poly2(float2 t) {
  t.x = fminf(fmaxf(t.x, -125.f), 127.f);
  t.y = fminf(fmaxf(t.y, -125.f), 127.f);
  const float2 k = __fadd2_rn(t, make_float2(12582912.f, 12582912.f));
  const float2 n = __fadd2_rn(k, make_float2(-12582912.f, -12582912.f));  // round(t), exact
  const float2 r = __ffma2_rn(n, make_float2(-1.f, -1.f), t);                // t - n, exact
  float2 p = __ffma2_rn(r, make_float2(1.3400432653725147e-3f, 1.3400432653725147e-3f),
                        make_float2(9.676037356257439e-3f, 9.676037356257439e-3f));
  p = __ffma2_rn(p, r, make_float2(5.550327152013779e-2f, 5.550327152013779e-2f));
  p = __ffma2_rn(p, r, make_float2(2.402210682630539e-1f, 2.402210682630539e-1f));
  p = __ffma2_rn(p, r, make_float2(6.931471824645996e-1f, 6.931471824645996e-1f));
  p = __ffma2_rn(p, r, make_float2(1.0000001192092896f, 1.0000001192092896f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(k.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(k.y) << 23)));
}

// exp(zs * ln2/256) for a pre-scaled argument zs
__device__ __forceinline__ double exp_scaled(const double zs, const MathSmem& t) {
  // round-to-nearest via F2I/I2F: conversions run on the XU pipe, which the
  // EM leaves mostly idle, instead of two fp64 adds with a 1.5*2^52 shifter
  const int k = __double2int_rn(zs);
  const double rs = zs - (double)k;  // exact
  double q = fma(rs, kExpA4, kExpA3);
  q = fma(q, rs, kExpA2);
  q = fma(q, rs, kExpA1);
  const double p = q * rs;  // exp(rs ln2/256) - 1
  const double T = t.expt[k & 255];
  const double res = fma(T, p, T);
  // hi word += floor(k / 256) << 20, as one arithmetic shift + one IMAD
  int m, hi;
  asm("shr.s32 %0, %1, 8;" : "=r"(m) : "r"(k));
  asm("mad.lo.s32 %0, %1, 1048576, %2;" : "=r"(hi) : "r"(m), "r"(__double2hiint(res)));
  return __hiloint2double(hi, __double2loint(res));
}

__device__ __forceinline__ double exp_tab(const double z, const MathSmem& t) { return exp_scaled(z * kExpScale, t); }

// logt: shared-memory (MathSmem::logt) or global (log_table_global) table
__device__ __forceinline__ double log_tab(const double x, const double2* __restrict__ logt) {
  const int hi = __double2hiint(x);
  const int lo = __double2loint(x);
  const int e = (hi >> 20) - 1023;
  const int j = (hi >> 12) & 255;
  const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);  // [1, 2)
  const double2 cj = logt[j];
  const double r = fma(m, cj.x, -1.0);
  double q = fma(r, kLogB5, kLogB4);
  q = fma(q, r, kLogB3);
  q = fma(q, r, -0.5);  // log1p(r) - r = r^2 q
#ifdef OXM_LOG_SPLIT_LN2
  const double ed = (double)e;
  const double h = fma(ed, kLn2I, cj.y);  // ed * kLn2I exact (20 x 11 bits)
  return h + (r + fma(q, r * r, ed * kLn2Lo20));
#else
  // e ln2 - ln c_j rounded once (<= 0.5 ulp of |log x| <= ~15), then + log1p(r)
  const double h = fma((double)e, kLn2Hi, cj.y);
  return h + fma(q, r * r, r);
#endif
}

}  // namespace oxm
