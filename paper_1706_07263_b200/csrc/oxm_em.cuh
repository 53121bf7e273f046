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
// lives in shared memory, not registers, and both band loops are fully
// unrolled around the table-driven exp/log of oxm_math.cuh (96 registers, 5
// CTAs per SM).  The stopping test compares squared norms (no sqrt/div); it
// differs from the reference's rel < tol only when rel is within ~1e-16 of tol.
//
// Kernels here: em_init_kernel (fit #1), em_persistent_kernel (all-fp64, or
// the fp64 tail of the fp32 map path), em_lead_kernel (fp32 lead-in) and
// em_exact_kernel (all-fp64 on a short coefficient list, 4 lanes each); the
// precision schedule that combines them is described at em_lead_kernel.
#pragma once

#include "oxm_common.cuh"
#include "oxm_math.cuh"

// band-loop unroll of the EM step (tuned on B200; build knob for experiments)
#ifndef OXM_EM_UNROLL
#define OXM_EM_UNROLL 26
#endif
#ifndef OXM_EM_UNROLL_B
#define OXM_EM_UNROLL_B 26
#endif
#ifndef OXM_TAIL_MIN_BLOCKS
#define OXM_TAIL_MIN_BLOCKS 5
#endif
#ifndef OXM_X_MIN_BLOCKS
#define OXM_X_MIN_BLOCKS 1
#endif
#ifndef OXM_LEAD_REVERSE
#define OXM_LEAD_REVERSE 1  // lead-in takes coefficients last-first (L2 reuse of the low-pass outputs)
#endif
#ifndef OXM_EM_MIN_BLOCKS
#define OXM_EM_MIN_BLOCKS 5
#endif

namespace oxm {

// max(s, eps) for finite s (no NaN handling: 3 instructions instead of ~8)
__device__ __forceinline__ double clamp_eps(double s, double eps) { return s > eps ? s : eps; }

template <int KL>
struct BandCount {
  static constexpr int kMax = KL > 0 ? KL : kMaxBands;
  __device__ __forceinline__ static int get(const DevOps& ops) { return KL > 0 ? KL : ops.L; }
};

// Dynamic shared memory of the persistent EM kernel: tables + one column per
// thread.  Columns are strided by threads + 1 doubles per row: rows (one band,
// consecutive threads) stay contiguous, and a column (one thread, consecutive
// bands -- write_spectra) walks the banks instead of hitting one bank 26 times.
// Rows of a lane's column after its L bands (which hold e during phase A and
// s = max(e + G r, eps) after phase B):
constexpr int kColOff = 0;     // element offset of the lane's output row (write_spectra)
constexpr int kColY = 1;       // 3 rows: y of the current coefficient
constexpr int kColPre = 4;     // 6 rows: cp.async prefetch of the next coefficient --
                               // y (3 rows), then x_init (3 rows; all-fp64 kernel) or
                               // {xh0, xh1}, {xh2, fits} (tail)
constexpr int kEmColExtra = 10;
__host__ __device__ constexpr size_t em_smem_bytes(int L, int threads) {
  return sizeof(MathSmem) + sizeof(double) * (size_t)(L + kEmColExtra) * (size_t)(threads + 1);
}

// cp.async (LDGSTS) of 4 / 8 bytes into shared memory, and its group waits
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Persistent, warp-refilled EM kernel.
//
// A one-thread-per-coefficient loop would leave a warp running until its
// slowest lane converges (fit counts vary 11..15 per coefficient) and a CTA
// until its slowest warp.  Here every warp advances all its lanes one *fit*
// per step; a lane whose coefficient has converged records it and immediately
// takes the next one from the warp's current chunk of kEmChunk consecutive
// coefficients.  Chunks are handed out by one global counter (one atomic per
// chunk, issued by lane 0): fit counts are spatially correlated (smooth
// regions converge in fewer fits), so static per-warp slices left the SMs
// unevenly loaded at the end of a launch.
//
// Fit #1 (the Tikhonov start) runs beforehand in em_init_kernel, so every
// persistent step is the same exp/prior/log/fit step and control flow is
// warp-uniform: the band counter stays in a uniform register and operator
// entries are uniform-datapath constants (ULDC / UR operands) rather than
// per-thread indexed LDCs feeding every DFMA.
//
// The final spectrum is not written by its own lane (a 26-store divergent
// branch in almost every step): phase B leaves s = max(e + G r, eps) in the
// lane's shared-memory column, and when lanes finish the whole warp writes
// their rows out together (write_spectra: coalesced).  The next coefficient's
// inputs are already in the lane's column (cp.async prefetch), so a refill
// does not wait on global memory.
enum class SpecOut { kSoaF64, kAosF32HiLo, kAosF64 };

struct EmIO {
  const double* y;     // unit-scale low-pass data: SoA [3][n] (y_soa) or AoS (n, 3)
  int y_soa;
  const double* init;  // AoS (n, L) start spectra, or null (Tikhonov start)
  int64_t n;
  double* S;           // kSoaF64: [L][n];  kAosF64: (n, L)
  float* Shi;          // kAosF32HiLo: (n, Lp) hi parts, then (n, Lp) lo parts:
  float* Slo;          //   hi + lo = s to 48 bits (Lp = L rounded up to 4)
  int Lp;
  SpecOut fmt;         // set by launch_em from its OUT parameter
  double* x;           // (n, 3) final concentrations, or null
  double* xinit;       // [3][n] fit #1 of the start spectrum (em_init_kernel output, required)
  int32_t* fits;       // (n) fit counts (required)
  unsigned long long* work;  // chunk counter, zero at launch (zeroed by em_init_kernel when it runs)
  int xinit_ready;     // x_init already computed (fused into the low-pass kernel)
  int em_reserve;      // CTA slots per SM left free for a concurrent kernel
  // fp32 lead-in (kAosF32HiLo only, when ops.lead_thr_f > 0): em_lead_kernel
  // writes each coefficient's hand-over state x to xh ([3][n] fp32) and its
  // fit count to fits; the fp64 tail continues from there
  float* xh;
  unsigned long long* lead_work;  // lead-in chunk counter, zero at launch
  // optional work counters (zero at launch): [0] fp32 fits committed by the
  // lead-in, [1] fp64 fits of the tail, [2] tail restarts in exact mode
  unsigned long long* stats;
  // optional coefficient selection: the kernel runs coefficients sel[0 ..
  // *sel_count) (device-side count) instead of 0 .. n; n stays the stride of
  // the SoA arrays
  const uint32_t* sel;
  const uint32_t* sel_count;
};

// warp-aggregated add of each lane's v into *ctr (one atomic per warp)
__device__ __forceinline__ void warp_count(unsigned long long* ctr, unsigned v, int lane) {
  const unsigned t = __reduce_add_sync(0xffffffffu, v);
  if (ctr && lane == 0 && t) atomicAdd(ctr, (unsigned long long)t);
}

constexpr int kEmThreads = 128;  // fp32 lead-in and fit #1 kernels
#ifndef OXM_PERS_THREADS
#define OXM_PERS_THREADS 128
#endif
constexpr int kPersThreads = OXM_PERS_THREADS;  // persistent fp64 EM kernel (tail / all-fp64 / exact list)
constexpr int kEmUnroll = OXM_EM_UNROLL;
constexpr int kEmUnrollB = OXM_EM_UNROLL_B;
#ifndef OXM_EM_CHUNK
#define OXM_EM_CHUNK 32
#endif
constexpr int kEmChunk = OXM_EM_CHUNK;  // coefficients per dynamically assigned chunk (>= 32)
#ifndef OXM_LEAD_RESID64
#define OXM_LEAD_RESID64 0  // 1: the lead-in's residual y - C e in fp64 (tools/lead_noise_study.py)
#endif
#ifndef OXM_LEAD_POLY_PAIRS
#define OXM_LEAD_POLY_PAIRS 0
#endif
constexpr int kLeadPolyPairs = OXM_LEAD_POLY_PAIRS;  // lead-in band pairs whose ex2 runs on the FMA pipe
static_assert(kEmChunk >= 32, "a refill may need up to 32 fresh coefficients");

// Fit #1 of one coefficient (bayes.py:241-250, 193): x = -F log(max(start, eps))
// with start = solve y (or ini[0..L) when given).
template <int KL>
__device__ __forceinline__ void start_fit(const DevOps& ops, const double2* logt, double y0, double y1, double y2,
                                          const double* ini, double& x0, double& x1, double& x2) {
  const int L = BandCount<KL>::get(ops);
  double n0 = 0.0, n1 = 0.0, n2 = 0.0;
#pragma unroll(KL > 0 ? KL : 2)
  for (int l = 0; l < L; ++l) {
    const double st = ini ? ini[l] : fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0));
    const double lg = log_tab(clamp_eps(st, ops.eps), logt);
    n0 = fma(ops.fitm[0][l], lg, n0);
    n1 = fma(ops.fitm[1][l], lg, n1);
    n2 = fma(ops.fitm[2][l], lg, n2);
  }
  x0 = -n0;
  x1 = -n1;
  x2 = -n2;
}

// Fit #1 for every coefficient, fully parallel, before the persistent loop
// (the fused video path does this inside its low-pass kernel instead).
template <int KL>
__global__ void __launch_bounds__(kEmThreads) em_init_kernel(const __grid_constant__ DevOps ops, EmIO io) {
  const int64_t i = (int64_t)blockIdx.x * kEmThreads + threadIdx.x;
  if (i == 0 && io.work) *io.work = 0ull;
  if (i >= io.n) return;
  const int L = BandCount<KL>::get(ops);
  double y0, y1, y2;
  if (io.y_soa) {
    y0 = io.y[i];
    y1 = io.y[io.n + i];
    y2 = io.y[2 * io.n + i];
  } else {
    y0 = io.y[3 * i];
    y1 = io.y[3 * i + 1];
    y2 = io.y[3 * i + 2];
  }
  const double* ini = io.init ? io.init + i * L : nullptr;
  double n0, n1, n2;
  start_fit<KL>(ops, log_table_global(), y0, y1, y2, ini, n0, n1, n2);
  n0 = -n0;
  n1 = -n1;
  n2 = -n2;
  io.xinit[i] = -n0;
  io.xinit[io.n + i] = -n1;
  io.xinit[2 * io.n + i] = -n2;
  if (ops.max_iters <= 1) {  // bayes.py:195 runs no iteration: fit #1 and the start spectrum are final
    io.fits[i] = 1;
    if (io.x) {
      io.x[3 * i] = -n0;
      io.x[3 * i + 1] = -n1;
      io.x[3 * i + 2] = -n2;
    }
    for (int l = 0; l < L; ++l) {
      const double st = clamp_eps(ini ? ini[l] : fma(ops.solve[l][2], y2, fma(ops.solve[l][1], y1, ops.solve[l][0] * y0)), ops.eps);
      if (io.fmt == SpecOut::kSoaF64) {
        io.S[(int64_t)l * io.n + i] = st;
      } else if (io.fmt == SpecOut::kAosF64) {
        io.S[i * L + l] = st;
      } else {
        const float h = __double2float_rn(st);
        io.Shi[i * io.Lp + l] = h;
        io.Slo[i * io.Lp + l] = __double2float_rn(st - (double)h);
      }
    }
  }
}

// Write the spectra s of the lanes in `done_mask` to global memory.  Phase B
// leaves each lane's s_l in its shared-memory column (column j holds lane j's
// s_l at c0[l * es + j]) and row kColOff holds the element offset of its
// output row, so a finished lane costs the warp one broadcast read of the
// offset, one read of s per band and one coalesced store: one finished lane
// at a time (warp-uniform loop, ~9 lanes finish per tail step), lane l
// storing band l.  lterm is the lane's part of the element index (band
// `lane` of the output row).  Slo == nullptr: hi parts only (the exact-block
// pass rewrites every block whose lo parts the fp64 pixel fallback reads).
template <SpecOut OUT>
__device__ __forceinline__ void store_band(const EmIO& io, int64_t e, double s) {
  if constexpr (OUT == SpecOut::kAosF32HiLo) {
    const float h = __double2float_rn(s);
    io.Shi[e] = h;
    if (io.Slo) io.Slo[e] = __double2float_rn(s - (double)h);
  } else {
    io.S[e] = s;
  }
}

template <SpecOut OUT>
__device__ __forceinline__ int64_t out_row_offset(const EmIO& io, int64_t i, int L) {
  return OUT == SpecOut::kSoaF64 ? i : (OUT == SpecOut::kAosF64 ? i * L : i * io.Lp);
}

template <SpecOut OUT>
__device__ __forceinline__ int64_t out_band_term(const EmIO& io, int l) {
  return OUT == SpecOut::kSoaF64 ? (int64_t)l * io.n : (int64_t)l;
}

template <int KL, SpecOut OUT, int es>
__device__ __forceinline__ void write_spectra(const EmIO& io, const double* c0, int L, unsigned done_mask, int lane,
                                              int64_t lterm) {
  if constexpr (KL > 0 && KL <= 32) {
    if (lane >= KL) return;  // lanes without a band
    while (done_mask) {
      const int owner = __ffs(done_mask) - 1;
      done_mask &= done_mask - 1;
      const int64_t off = __double_as_longlong(c0[(KL + kColOff) * es + owner]);
      store_band<OUT>(io, off + lterm, c0[lane * es + owner]);
    }
  } else {
    while (done_mask) {
      const int owner = __ffs(done_mask) - 1;
      done_mask &= done_mask - 1;
      const int64_t off = __double_as_longlong(c0[(L + kColOff) * es + owner]);
      for (int l = lane; l < L; l += 32) store_band<OUT>(io, off + out_band_term<OUT>(io, l), c0[l * es + owner]);
    }
  }
}

// TAIL: continue from the fp32 lead-in's hand-over (x from io.xh, or x_init
// when the hand-over came at fit #1; fit count from io.fits).  A tail step
// whose rel lands within the guard band around tol, or a tail that runs into
// max_iters, restarts its coefficient from fit #1 in exact fp64 mode.
//
// Refill: every lane holds its next coefficient's data (y and x_init, or the
// hand-over state) in the prefetch rows of its column, copied there by
// cp.async when the lane took its current one; a lane whose coefficient
// converges takes the prefetched one (its copies landed steps ago) and issues
// the next prefetch.  Invariant: a lane without a current coefficient
// (idx < 0) has none prefetched either (pidx < 0).
template <int KL, SpecOut OUT, bool TAIL = false>
__global__ void __launch_bounds__(kPersThreads, TAIL ? OXM_TAIL_MIN_BLOCKS : OXM_EM_MIN_BLOCKS)
    em_persistent_kernel(const __grid_constant__ DevOps ops, EmIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MathSmem& mt = *reinterpret_cast<MathSmem*>(smem_raw);
  constexpr int es = kPersThreads + 1;  // row stride of the columns (see em_smem_bytes)
  double* const col = reinterpret_cast<double*>(smem_raw + sizeof(MathSmem)) + threadIdx.x;  // this lane's column
  load_math_tables(mt);
  __syncthreads();

  const int L = BandCount<KL>::get(ops);
  double* const xrow = col + L * es;  // the rows after the bands
  auto row = [&](int r) -> double& { return xrow[r * es]; };
  const double eps = ops.eps;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t warp = ((int64_t)blockIdx.x * kPersThreads + threadIdx.x) >> 5;
  // first 32 coefficients statically per warp, then kEmChunk-sized chunks
  // from io.work, numbered from dyn0
  const int64_t dyn0 = (int64_t)gridDim.x * kPersThreads;
  // positions 0 .. count are coefficients, or indices into io.sel
  const int64_t count = io.sel ? (int64_t)*io.sel_count : io.n;
  auto coef = [&](int64_t pos) -> int64_t { return io.sel ? (int64_t)io.sel[pos] : pos; };
  int64_t next = warp * 32;               // next unassigned position of the current chunk
  int64_t stop = min64(next + 32, count);  // end of the current chunk
  bool exhausted = false;

  if (ops.max_iters <= 1) return;  // fit #1 is the answer: written by em_init_kernel

  // y layout is fixed per output format (hybrid path: SoA; estimate_lowpass
  // API: AoS), so the prefetch has no runtime branch for it
  constexpr bool kYSoa = OUT != SpecOut::kAosF64;
  const int64_t lterm = out_band_term<OUT>(io, lane);
  int64_t idx = -1, pidx = -1;
  int nfit = 1;
  // TAIL state: 0 = exact (runs the coefficient from fit #1, no guard), j >= 1 =
  // the next step is tail step j of a hand-over (j = 1: the fp64 redo of the
  // lead-in's uncommitted fit), guarded by max(guard, guard1 2^(-(j-1) shift))
  int mode = 0;
  unsigned wsteps = 0, wrestarts = 0;  // TAIL work counters of this warp (io.stats; < 2^32 per warp)
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;

  auto prefetch = [&](int64_t i) {
#pragma unroll
    for (int k = 0; k < 3; ++k) cp_async8(&row(kColPre + k), kYSoa ? io.y + k * io.n + i : io.y + 3 * i + k);
    if constexpr (TAIL) {
      float* a = reinterpret_cast<float*>(&row(kColPre + 3));
      float* b = reinterpret_cast<float*>(&row(kColPre + 4));
      cp_async4(a, io.xh + i);
      cp_async4(a + 1, io.xh + io.n + i);
      cp_async4(b, io.xh + 2 * io.n + i);
      cp_async4(b + 1, io.fits + i);
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async8(&row(kColPre + 3 + k), io.xinit + k * io.n + i);
    }
    cp_async_commit();
  };
  // make the prefetched coefficient (pidx >= 0) the current one
  auto take = [&]() {
    cp_async_wait_all();
    idx = pidx;
    double yv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) yv[k] = row(kColPre + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) row(kColY + k) = yv[k];
    if constexpr (TAIL) {
      const float2 a = *reinterpret_cast<const float2*>(&row(kColPre + 3));
      const float2 b = *reinterpret_cast<const float2*>(&row(kColPre + 4));
      const int f = __float_as_int(b.y);
      nfit = f;
      mode = f <= 1 ? 0 : 1;
      if (f > 1) {
        x0 = a.x;
        x1 = a.y;
        x2 = b.x;
      } else {  // hand-over at fit #1 (rare): exact fp64 from x_init
        x0 = io.xinit[idx];
        x1 = io.xinit[io.n + idx];
        x2 = io.xinit[2 * io.n + idx];
      }
    } else {
      x0 = row(kColPre + 3);
      x1 = row(kColPre + 4);
      x2 = row(kColPre + 5);
      nfit = 1;
      mode = 0;
    }
  };
  // hand out the next positions to the lanes of mask m (warp-uniform call;
  // `want`: this lane is in m): rest of the current chunk, then a new one
  auto assign = [&](unsigned m, bool want) -> int64_t {
    const int need = __popc(m);
    const int64_t avail = stop - next;  // warp-uniform
    int64_t fresh = count, fresh_end = count;
    if (avail < need && !exhausted) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(io.work, (unsigned long long)kEmChunk);
      fresh = dyn0 + (int64_t)__shfl_sync(0xffffffffu, b, 0);
      fresh_end = min64(fresh + kEmChunk, count);
      exhausted = fresh >= count;
    }
    int64_t got = -1;
    if (want) {
      const int r = __popc(m & lt_mask);
      const int64_t pos = r < avail ? next + r : fresh + (r - avail);
      got = pos < (r < avail ? stop : fresh_end) ? coef(pos) : -1;
    }
    if (avail < need) {
      next = fresh_end > fresh ? min64(fresh + (need - avail), fresh_end) : fresh_end;
      stop = fresh_end;
    } else {
      next += need;
    }
    return got;
  };

  // start: the static chunk's coefficient is fetched and taken at once, then
  // every lane that got one prefetches its next
  pidx = assign(0xffffffffu, true);
  if (pidx >= 0) {
    prefetch(pidx);
    take();
    row(kColOff) = __longlong_as_double(out_row_offset<OUT>(io, idx, L));
  }
  pidx = -1;
  {
    const unsigned m = __ballot_sync(0xffffffffu, idx >= 0);
    if (m) {
      pidx = assign(m, idx >= 0);
      if (pidx >= 0) prefetch(pidx);
    }
  }

  while (__any_sync(0xffffffffu, idx >= 0)) {
    if constexpr (TAIL) wsteps += __popc(__ballot_sync(0xffffffffu, idx >= 0));
    // ---- phase A: expected spectrum e = exp(-xi x) and residual r = y - C e
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    const double x2s = x2 * kExpScale;  // xi[:, 2] == 1 (core.py:152-153); xis = xi[:, 0:2] * kExpScale
#pragma unroll(KL > 0 ? kEmUnroll : 2)
    for (int l = 0; l < L; ++l) {
      const double el = exp_scaled(-fma(ops.xis[l][0], x0, fma(ops.xis[l][1], x1, x2s)), mt);
      col[l * es] = el;
      c0 = fma(ops.sens[0][l], el, c0);
      c1 = fma(ops.sens[1][l], el, c1);
      c2 = fma(ops.sens[2][l], el, c2);
    }
    const double r0 = row(kColY) - c0, r1 = row(kColY + 1) - c1, r2 = row(kColY + 2) - c2;
    // ---- phase B: s = max(e + G r, eps) (kept in the column for
    // write_spectra), Beer-Lambert fit of log s
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll(KL > 0 ? kEmUnrollB : 2)
    for (int l = 0; l < L; ++l) {
      const double sv = clamp_eps(fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, col[l * es]))), eps);
      col[l * es] = sv;
      const double lg = log_tab(sv, mt.logt);
      m0 = fma(ops.fitm[0][l], lg, m0);
      m1 = fma(ops.fitm[1][l], lg, m1);
      m2 = fma(ops.fitm[2][l], lg, m2);
    }
    // ---- bookkeeping: stopping rule of bayes.py:195-205, then write-out and refill
    const double n0 = -m0, n1 = -m1, n2 = -m2;
    bool done = false, restart = false;
    if (idx >= 0) {
      ++nfit;
      const double d0 = n0 - x0, d1 = n1 - x1, d2 = n2 - x2;
      const double dn2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
      const double xn2 = __dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)), __dmul_rn(x2, x2));
      const double xm2 = fmax(xn2, 1e-16);
      done = dn2 < ops.rel_tol2 * xm2 || nfit >= ops.max_iters;
      if (ops.dbg_rel && nfit < 24) {
        ops.dbg_rel[idx * 24 + nfit] = (float)sqrt(dn2 / xm2);
        ops.dbg_step[idx * 24 + nfit] = (uint8_t)min(TAIL ? mode : 0, 255);
      }
      if constexpr (TAIL) {
        // the state still carries the lead-in's fp32 perturbation: a stop
        // decision near the threshold (or one forced by max_iters) is not
        // trusted -- redo the coefficient in exact fp64 from fit #1.  The
        // first tail step redoes the lead-in's uncommitted fit from the fp32
        // state itself, so its decision sees that perturbation undamped: a
        // stop there is never trusted either (rare: rel must fall from
        // > K tol to < tol in one fit), and the guard band starts wider
        // (oxm_ctx_set_em_first_guard, default +-10%) and shrinks 4x per tail step
        const int j = mode;
        if (j) {
          const double lo = j == 1 ? ops.band_lo[0] : (j == 2 ? ops.band_lo[1] : ops.band_lo[2]);
          const double hi = j == 1 ? ops.band_hi[0] : (j == 2 ? ops.band_hi[1] : ops.band_hi[2]);
          restart = (dn2 > lo * xm2 && dn2 < hi * xm2) || nfit >= ops.max_iters || (j == 1 && done);
        }
        mode = restart || !j ? 0 : min(j + 1, 3);
        if (restart) {
          done = false;
          nfit = 1;
        }
      }
      if (done) {
        io.fits[idx] = nfit;
        if (io.x) {
          io.x[3 * idx] = n0;
          io.x[3 * idx + 1] = n1;
          io.x[3 * idx + 2] = n2;
        }
      }
    }
    if (TAIL && restart) {
      x0 = io.xinit[idx];
      x1 = io.xinit[io.n + idx];
      x2 = io.xinit[2 * io.n + idx];
    } else {
      x0 = n0;
      x1 = n1;
      x2 = n2;
    }
    if constexpr (TAIL) wrestarts += __popc(__ballot_sync(0xffffffffu, restart));
    const unsigned m = __ballot_sync(0xffffffffu, done);
    if (m) {
      // finished lanes take their prefetched coefficient and prefetch the
      // next; then the whole warp streams the finished spectra out (their s
      // rows and output offsets are still in the columns), and only then are
      // the new offsets stored
      const bool more = done && pidx >= 0;
      const unsigned mm = __ballot_sync(0xffffffffu, more);
      int64_t np = -1;
      if (mm) np = assign(mm, more);
      if (done) {
        if (more) {
          take();
          pidx = np;
          if (np >= 0) prefetch(np);
        } else {
          idx = -1;
        }
      }
      __syncwarp();  // every lane's phase-B stores of s are visible to the warp
      write_spectra<KL, OUT, es>(io, col - lane, L, m, lane, lterm);
      __syncwarp();
      if (done && idx >= 0) row(kColOff) = __longlong_as_double(out_row_offset<OUT>(io, idx, L));
    }
  }
  if (TAIL && io.stats && lane == 0) {
    atomicAdd(io.stats + 1, (unsigned long long)wsteps);
    atomicAdd(io.stats + 2, (unsigned long long)wrestarts);
  }
}

// ---------------------------------------------------------------------------
// fp32 lead-in of the EM (hybrid fp32-map path).
//
// The iteration of bayes.py:185-207 contracts (rel shrinks ~2x per fit), and a
// "not converged" decision taken while rel is far above tol is insensitive to
// fp32 error.  So the first fits run here in fp32 -- MUFU ex2/lg2 and FFMA
// instead of the fp64 pipe -- for as long as |dx| > K tol |x| (K = 16 by
// default: ops.lead_thr_f = (K tol)^2) and the next fit is not the last
// allowed one.  The step that fails the test is not committed: the state
// before it (x after fit k, and k) is handed to the fp64 tail
// (em_persistent_kernel<..., TAIL>), which redoes fit k+1 onwards exactly as
// the reference does.  The tail damps the hand-over perturbation at the
// iteration's contraction rate while rel falls from ~K tol to tol, so final
// spectra differ from the all-fp64 ones by ~1e-8 relative
// (tools/mixed_em_study.py); stop decisions that land within the guard band
// around tol are redone from fit #1 in exact fp64 (~2% of coefficients), so
// fit counts stay bit-exact.  A hand-over at fit #1 passes x_init itself.
template <int KL>
__global__ void __launch_bounds__(kEmThreads) em_lead_kernel(const __grid_constant__ DevOps ops, EmIO io) {
  static_assert(KL > 0, "the fp32 lead-in keeps e in registers: fixed band count only");
  constexpr float kLog2e = 1.44269504088896340736f;
  const float eps = ops.eps_f, thr = ops.lead_thr_f;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t warp = ((int64_t)blockIdx.x * kEmThreads + threadIdx.x) >> 5;
  const int64_t dyn0 = (int64_t)gridDim.x * kEmThreads;
  int64_t next = warp * 32;
  int64_t stop = min64(next + 32, io.n);
  bool exhausted = false;

  int64_t idx = next + lane < stop ? next + lane : -1;
  int nfit = 1;
#if OXM_LEAD_RESID64
  using YT = double;
#else
  using YT = float;
#endif
  YT y0 = 0, y1 = 0, y2 = 0;
  float x0 = 0.f, x1 = 0.f, x2 = 0.f;
  auto load = [&](int64_t i) {
    y0 = (YT)io.y[i];
    y1 = (YT)io.y[io.n + i];
    y2 = (YT)io.y[2 * io.n + i];
    x0 = (float)io.xinit[i];
    x1 = (float)io.xinit[io.n + i];
    x2 = (float)io.xinit[2 * io.n + i];
    nfit = 1;
  };
  // positions map to coefficients last-first (OXM_LEAD_REVERSE): the low-pass
  // kernel wrote the last frames' ybar / x_init last, so those are the ones
  // still in L2 when this kernel starts (128 frames: 18.75 -> 18.11 us/frame);
  // the fp64 tail then walks forward and starts on the hand-over states this
  // kernel wrote last
  auto cof = [&](int64_t p) -> int64_t { return OXM_LEAD_REVERSE ? io.n - 1 - p : p; };
  if (idx >= 0) load(cof(idx));
  next = stop;

  // bands l, l+1 share one packed FFMA2 (two partial sums per accumulator,
  // added at the end: the lead-in needs no particular summation order)
  static_assert(KL % 2 == 0, "band pairs");
  auto pair = [](const float* row, int l) { return *reinterpret_cast<const float2*>(row + l); };
  auto dup = [](float v) { return make_float2(v, v); };
  while (__any_sync(0xffffffffu, idx >= 0)) {
    float2 e[KL / 2];
    float2 c0 = dup(0.f), c1 = c0, c2 = c0;
#if OXM_LEAD_RESID64
    double cd0 = 0.0, cd1 = 0.0, cd2 = 0.0;
#endif
    const float2 X0 = dup(x0), X1 = dup(x1), X2 = dup(-kLog2e * x2);  // xi[:, 2] == 1
#pragma unroll
    for (int q = 0; q < KL / 2; ++q) {
      const int l = 2 * q;
      const float2 t = __ffma2_rn(pair(ops.xl2_t[0], l), X0, __ffma2_rn(pair(ops.xl2_t[1], l), X1, X2));
      // the first kLeadPolyPairs band pairs take their ex2 on the FMA pipe
      e[q] = q < kLeadPolyPairs ? ex2_poly2(t) : make_float2(ex2_approx(t.x), ex2_approx(t.y));
#if OXM_LEAD_RESID64
      const double ex = e[q].x, ey = e[q].y;
      cd0 = fma(ops.sens[0][l + 1], ey, fma(ops.sens[0][l], ex, cd0));
      cd1 = fma(ops.sens[1][l + 1], ey, fma(ops.sens[1][l], ex, cd1));
      cd2 = fma(ops.sens[2][l + 1], ey, fma(ops.sens[2][l], ex, cd2));
#else
      c0 = __ffma2_rn(pair(ops.sens_f[0], l), e[q], c0);
      c1 = __ffma2_rn(pair(ops.sens_f[1], l), e[q], c1);
      c2 = __ffma2_rn(pair(ops.sens_f[2], l), e[q], c2);
#endif
    }
#if OXM_LEAD_RESID64
    const float2 R0 = dup((float)(y0 - cd0)), R1 = dup((float)(y1 - cd1)), R2 = dup((float)(y2 - cd2));
#else
    const float2 R0 = dup(y0 - (c0.x + c0.y)), R1 = dup(y1 - (c1.x + c1.y)), R2 = dup(y2 - (c2.x + c2.y));
#endif
    float2 m0 = dup(0.f), m1 = m0, m2 = m0;
#pragma unroll
    for (int q = 0; q < KL / 2; ++q) {
      const int l = 2 * q;
      const float2 sv = __ffma2_rn(pair(ops.gain_t[2], l), R2,
                                   __ffma2_rn(pair(ops.gain_t[1], l), R1, __ffma2_rn(pair(ops.gain_t[0], l), R0, e[q])));
      const float2 lg = make_float2(lg2_approx(fmaxf(sv.x, eps)), lg2_approx(fmaxf(sv.y, eps)));
      m0 = __ffma2_rn(pair(ops.fitl2_f[0], l), lg, m0);
      m1 = __ffma2_rn(pair(ops.fitl2_f[1], l), lg, m1);
      m2 = __ffma2_rn(pair(ops.fitl2_f[2], l), lg, m2);
    }
    const float n0 = m0.x + m0.y, n1 = m1.x + m1.y, n2 = m2.x + m2.y;
    bool done = false;
    if (idx >= 0) {
      const float d0 = n0 - x0, d1 = n1 - x1, d2 = n2 - x2;
      const float dn2 = d0 * d0 + d1 * d1 + d2 * d2;
      const float xn2 = fmaxf(x0 * x0 + x1 * x1 + x2 * x2, 1e-16f);
      // commit fit nfit+1 only when the reference surely continues after it;
      // NaN / inf (fp32 overflow) fail the test and hand over the last finite state
      if (dn2 > thr * xn2 && dn2 <= 3.0e38f && nfit + 1 < ops.max_iters) {
        x0 = n0;
        x1 = n1;
        x2 = n2;
        ++nfit;
      } else {
        done = true;
        const int64_t c = cof(idx);
        if (nfit > 1) {
          io.xh[c] = x0;
          io.xh[io.n + c] = x1;
          io.xh[2 * io.n + c] = x2;
        }
        io.fits[c] = nfit;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, done);
    if (m) {
      if (io.stats) warp_count(io.stats, done ? (unsigned)(nfit - 1) : 0u, lane);
      // refill finished lanes: rest of the current chunk, then a new one
      const int need = __popc(m);
      const int64_t avail = stop - next;
      int64_t fresh = io.n, fresh_end = io.n;
      if (avail < need && !exhausted) {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(io.lead_work, (unsigned long long)kEmChunk);
        fresh = dyn0 + (int64_t)__shfl_sync(0xffffffffu, b, 0);
        fresh_end = min64(fresh + kEmChunk, io.n);
        exhausted = fresh >= io.n;
      }
      if (done) {
        const int r = __popc(m & lt_mask);
        const int64_t mine = r < avail ? next + r : fresh + (r - avail);
        idx = mine < (r < avail ? stop : fresh_end) ? mine : -1;
        if (idx >= 0) load(cof(idx));
      }
      if (avail < need) {
        next = fresh_end > fresh ? min64(fresh + (need - avail), fresh_end) : fresh_end;
        stop = fresh_end;
      } else {
        next += need;
      }
    }
  }
}

template <typename K>
inline int persistent_blocks(K kern, size_t smem, int reserve, int64_t need_ctas, int64_t& blocks,
                             int threads = kEmThreads) {
  cudaError_t err = cudaSuccess;
  if (smem > 48 * 1024) err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 0, per_sm = 0;
  if (err == cudaSuccess) err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (err != cudaSuccess) {
    set_last_error("em launch configuration", err);
    return OXM_ERR_CUDA;
  }
  if (sms < 1) sms = 1;
  // leave `reserve` CTA slots per SM free so a concurrent per-pixel kernel
  // (split launch, other stream) can co-reside with the persistent EM
  per_sm -= reserve;
  if (per_sm < 1) per_sm = 1;
  blocks = (int64_t)sms * per_sm;
  if (blocks > need_ctas) blocks = need_ctas;
  return OXM_OK;
}

// Persistent EM launch (enough CTAs to fill every SM once).  io.work must be
// zero when the persistent kernel starts: em_init_kernel zeroes it when it
// runs, otherwise (x_init fused upstream) the caller does; likewise
// io.lead_work for the fp32 lead-in.  `split` (optional) is recorded between
// the lead-in and the fp64 kernel.
template <int KL, SpecOut OUT>
inline int launch_em(const DevOps& ops, EmIO io, cudaStream_t s, cudaEvent_t split = nullptr) {
  if (io.n <= 0) return OXM_OK;
  if (!io.fits || !io.xinit || !io.work) return OXM_ERR_ARGUMENT;
  if ((io.y_soa != 0) != (OUT != SpecOut::kAosF64)) return OXM_ERR_ARGUMENT;  // see em_persistent_kernel
  io.fmt = OUT;
  const size_t smem = em_smem_bytes(ops.L, kPersThreads);
  const int64_t need = ceil_div(io.n, kEmThreads);
  const int64_t need_p = ceil_div(io.n, kPersThreads);
  if (!io.xinit_ready || ops.max_iters <= 1) {
    em_init_kernel<KL><<<(unsigned)need, kEmThreads, 0, s>>>(ops, io);
    int st0 = check_launch("em_init");
    if (st0) return st0;
  }
  constexpr bool kCanLead = KL > 0 && OUT == SpecOut::kAosF32HiLo;
  const bool lead = kCanLead && ops.lead_thr_f > 0.0f && ops.max_iters > 2 && io.xh && io.lead_work;
  int64_t blocks = 0;
  int st = OXM_OK;
  if constexpr (kCanLead) {
    if (lead) {
      auto lk = em_lead_kernel<(KL > 0 ? KL : 1)>;
      if ((st = persistent_blocks(lk, 0, io.em_reserve, need, blocks))) return st;
      lk<<<(unsigned)blocks, kEmThreads, 0, s>>>(ops, io);
      if ((st = check_launch("em_lead"))) return st;
    }
  }
  if (split) cudaEventRecord(split, s);
  if constexpr (kCanLead) {
    if (lead) {
      auto tk = em_persistent_kernel<KL, OUT, true>;
      if ((st = persistent_blocks(tk, smem, io.em_reserve, need_p, blocks, kPersThreads))) return st;
      tk<<<(unsigned)blocks, kPersThreads, smem, s>>>(ops, io);
      return check_launch("em_tail");
    }
  }
  auto kern = em_persistent_kernel<KL, OUT>;
  if ((st = persistent_blocks(kern, smem, io.em_reserve, need_p, blocks, kPersThreads))) return st;
  kern<<<(unsigned)blocks, kPersThreads, smem, s>>>(ops, io);
  return check_launch("em_persistent");
}

// Exact fp64 EM over a device-side coefficient list (sel, *sel_count), e.g.
// the low-pass blocks whose pixels need the fp64 map fallback: their spectra
// must be the all-fp64 ones, not the lead-in/tail ones.  The list is short
// (~6% of the coefficients), so one lane per coefficient would leave most of
// the GPU idle and each warp waiting for its slowest lanes; here a group of
// kXLanes lanes shares a coefficient (bands sub, sub + kXLanes, ...; the
// C e and fit sums are reduced with xor shuffles, which leave bit-identical
// sums in every lane of the group) and takes the next list entry from a
// global counter when it finishes.  Same fp64 table exp/log and the same
// per-band arithmetic as em_persistent_kernel; only the order of the 26-term
// sums differs (~1 ulp, like any other summation order of the reference's
// BLAS products).  The count is device-side, so the grid is the resident
// one; io.work must be zero at launch.
constexpr int kXLanes = 4;
constexpr int64_t kExactSeqMinN = int64_t(1) << 21;  // low-pass coefficients (~16 1080p n=2 frames)
constexpr int kXThreads = 128;
struct alignas(16) XBand {  // per-band operator row, staged in shared memory (lanes read different bands)
  double xs0, xs1, c0, c1, c2, g0, g1, g2, f0, f1, f2, pad;
};

template <int KL, SpecOut OUT>
__global__ void __launch_bounds__(kXThreads, OXM_X_MIN_BLOCKS) em_exact_kernel(const __grid_constant__ DevOps ops, EmIO io) {
  static_assert(KL > 0, "fixed band count");
  constexpr int NB = (KL + kXLanes - 1) / kXLanes;  // bands per lane
  __shared__ MathSmem mt;
  __shared__ XBand ob[KL];
  load_math_tables(mt);
  for (int l = threadIdx.x; l < KL; l += kXThreads) {
    ob[l] = XBand{ops.xis[l][0], ops.xis[l][1], ops.sens[0][l], ops.sens[1][l], ops.sens[2][l], ops.gain[l][0],
                  ops.gain[l][1], ops.gain[l][2], ops.fitm[0][l], ops.fitm[1][l], ops.fitm[2][l], 0.0};
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, sub = lane & (kXLanes - 1), lead = lane & ~(kXLanes - 1);
  const double eps = ops.eps, tol2 = ops.rel_tol2;
  const int64_t count = io.sel ? (int64_t)*io.sel_count : io.n;
  int64_t idx = -1;
  int nfit = 1;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0, x0 = 0.0, x1 = 0.0, x2 = 0.0;
  bool want = true;  // this group needs its next coefficient
  for (;;) {
    if (want) {  // group-uniform
      unsigned long long j = 0;
      if (sub == 0) j = atomicAdd(io.work, 1ull);
      j = __shfl_sync(((1u << kXLanes) - 1u) << lead, j, lead);
      idx = (int64_t)j < count ? (io.sel ? (int64_t)io.sel[j] : (int64_t)j) : -1;
      if (idx >= 0) {
        y0 = io.y[idx];
        y1 = io.y[io.n + idx];
        y2 = io.y[2 * io.n + idx];
        x0 = io.xinit[idx];
        x1 = io.xinit[io.n + idx];
        x2 = io.xinit[2 * io.n + idx];
        nfit = 1;
      }
      want = false;
    }
    if (!__any_sync(0xffffffffu, idx >= 0)) break;
    // phase A: e = exp(-xi x) for this lane's bands, C e reduced over the group
    double e[NB];
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
    const double x2s = x2 * kExpScale;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int l = sub + kXLanes * k;
      if (l < KL) {
        const XBand& b = ob[l];
        e[k] = exp_scaled(-fma(b.xs0, x0, fma(b.xs1, x1, x2s)), mt);
        c0 = fma(b.c0, e[k], c0);
        c1 = fma(b.c1, e[k], c1);
        c2 = fma(b.c2, e[k], c2);
      }
    }
#pragma unroll
    for (int o = 1; o < kXLanes; o <<= 1) {
      c0 += __shfl_xor_sync(0xffffffffu, c0, o);
      c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    }
    const double r0 = y0 - c0, r1 = y1 - c1, r2 = y2 - c2;
    // phase B: s = max(e + G r, eps), fit of log s reduced over the group
    double sv[NB];
    double n0 = 0.0, n1 = 0.0, n2 = 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int l = sub + kXLanes * k;
      if (l < KL) {
        const XBand& b = ob[l];
        sv[k] = clamp_eps(fma(b.g2, r2, fma(b.g1, r1, fma(b.g0, r0, e[k]))), eps);
        const double lg = log_tab(sv[k], mt.logt);
        n0 = fma(b.f0, lg, n0);
        n1 = fma(b.f1, lg, n1);
        n2 = fma(b.f2, lg, n2);
      }
    }
#pragma unroll
    for (int o = 1; o < kXLanes; o <<= 1) {
      n0 += __shfl_xor_sync(0xffffffffu, n0, o);
      n1 += __shfl_xor_sync(0xffffffffu, n1, o);
      n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    }
    n0 = -n0;
    n1 = -n1;
    n2 = -n2;
    if (idx >= 0) {  // group-uniform from here on
      ++nfit;
      const double d0 = n0 - x0, d1 = n1 - x1, d2 = n2 - x2;
      const double dn2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
      const double xn2 = __dadd_rn(__dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1)), __dmul_rn(x2, x2));
      x0 = n0;
      x1 = n1;
      x2 = n2;
      if (dn2 < tol2 * fmax(xn2, 1e-16) || nfit >= ops.max_iters) {
#pragma unroll
        for (int k = 0; k < NB; ++k) {
          const int l = sub + kXLanes * k;
          if (l < KL) {
            if constexpr (OUT == SpecOut::kSoaF64) {
              io.S[(int64_t)l * io.n + idx] = sv[k];
            } else if constexpr (OUT == SpecOut::kAosF64) {
              io.S[idx * KL + l] = sv[k];
            } else {
              const float h = __double2float_rn(sv[k]);
              io.Shi[idx * io.Lp + l] = h;
              io.Slo[idx * io.Lp + l] = __double2float_rn(sv[k] - (double)h);
            }
          }
        }
        if (sub == 0) {
          io.fits[idx] = nfit;
          if (io.x) {
            io.x[3 * idx] = n0;
            io.x[3 * idx + 1] = n1;
            io.x[3 * idx + 2] = n2;
          }
        }
        want = true;
      }
    }
  }
}

template <int KL, SpecOut OUT>
inline int launch_em_selected(const DevOps& ops, EmIO io, cudaStream_t s) {
  if (io.n <= 0) return OXM_OK;
  if (!io.fits || !io.xinit || !io.work || !io.sel || !io.sel_count) return OXM_ERR_ARGUMENT;
  if (ops.max_iters <= 1) return OXM_ERR_ARGUMENT;  // fit #1 would be final: nothing to redo
  io.fmt = OUT;
  int64_t blocks = 0;
  int st = OXM_OK;
  // The list is ~1% of the coefficients.  Large batches give it enough
  // coefficients per warp for the one-lane-per-coefficient persistent kernel
  // (cheaper per fit); small ones leave that kernel latency-bound, where the
  // 4-lane groups finish each coefficient ~3x sooner (tools/em_variants.py:
  // 8 frames 10.3 vs 10.6 us/frame, 32 frames 5.6 vs 5.2, 64 frames 5.3 vs 4.7).
  if (io.n >= kExactSeqMinN) {
    io.stats = nullptr;
    const size_t smem = em_smem_bytes(ops.L, kPersThreads);
    auto kern = em_persistent_kernel<KL, OUT>;
    if ((st = persistent_blocks(kern, smem, 0, ceil_div(io.n, kPersThreads), blocks, kPersThreads)))
      return st;
    kern<<<(unsigned)blocks, kPersThreads, smem, s>>>(ops, io);
  } else {
    auto kern = em_exact_kernel<KL, OUT>;
    if ((st = persistent_blocks(kern, 0, 0, ceil_div(io.n * kXLanes, kXThreads), blocks))) return st;
    kern<<<(unsigned)blocks, kXThreads, 0, s>>>(ops, io);
  }
  return check_launch("em_exact");
}

}  // namespace oxm
