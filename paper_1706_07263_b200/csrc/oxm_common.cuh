// Shared definitions for the sm_100a kernels behind include/oximap_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "oximap_b200.h"

namespace oxm {

constexpr int kMaxBands = OXM_MAX_BANDS;

// Operator set passed BY VALUE as a __grid_constant__ kernel parameter, so it
// lives in constant bank 0 and every FMA below takes its matrix entry as a
// c[0x0][...] operand (uniform across the warp, no LDS/LDG).  ~9.3 KB, well
// under the 32 KB kernel-parameter limit of CUDA >= 12.1.
struct DevOps {
  // fp32 copies first: low parameter-bank offsets encode directly in FFMA
  float solve_f[kMaxBands][3];
  float fitl2_f[3][kMaxBands];  // -ln(2) * fit_mat: x = sum_l fitl2 * log2(s)
  float2 solve_f2[kMaxBands][3];   // the same, duplicated into both halves for FFMA2
  float2 fitl2_f2[3][kMaxBands];
  // fp32 lead-in of the EM (oxm_em.cuh, em_lead_kernel)
  // (band-major rows: bands l, l+1 form one float2 FFMA2 operand)
  float xl2_t[2][kMaxBands];  // -xi[:, 0:2]^T * log2(e): e = 2^(xl2 . x - log2(e) x2)
  float sens_f[3][kMaxBands];
  float gain_t[3][kMaxBands];  // gain^T
  float lead_thr_f;  // (K tol)^2: fp32 steps continue while |dx|^2 > lead_thr |x|^2; 0 = no lead-in
  float eps_f;
  int L;
  int max_iters;
  double eps;
  double rel_tol;
  double rel_tol2;  // rel_tol^2 (the stopping test compares squared norms)
  double fallback_below;
  double exact_below;  // with the lead-in: fallback pixels with a band below this get their block's EM redone all-fp64
  // fp64 tail guard bands: tail step j (1 = the redo of the lead-in's uncommitted
  // fit) with |rel/tol - 1| < g_j = max(guard, guard1 * 2^(-(j-1) guard_shift))
  // redoes its coefficient; band_lo/hi[k] = ((1 -+ g_j) tol)^2 for j = 1, 2 and
  // j >= 3 (g_j has reached guard by step 3 for every shift >= 2)
  double guard, guard1;
  int guard_shift;
  double band_lo[3], band_hi[3];
  double solve[kMaxBands][3];  // Tikhonov ridge inverse, unmix.py:53-65
  double fitm[3][kMaxBands];   // (xi^T xi)^-1 xi^T, bayes.py:102
  double xi[kMaxBands][3];     // chromophore basis, core.py:134-158
  double sens[3][kMaxBands];   // camera matrix C, core.py:112-131
  double gain[kMaxBands][3];   // N^-1 C^T, N = C^T C + beta D2^T D2 (bayes.py:117-129)
  double xis[kMaxBands][2];    // xi[:, 0:2] * 256/ln2: EM exp arguments pre-scaled (oxm_math.cuh)
  // device copy of the per-band rows {solve[l][0..2], fitm[0..2][l], 0, 0}
  // (L x 8 doubles, 64 B per band): code that indexes bands by lane reads
  // them with coalesced loads instead of serialised indexed constant loads
  const double* band_rows;
  // diagnostics (oxm_ctx_set_em_debug_log, normally null): the persistent EM
  // kernels record rel of every fit m of coefficient i at dbg_rel[i * 24 + m]
  // and the tail step index j (0 = exact fp64 trajectory) at dbg_step[i * 24 + m]
  float* dbg_rel;
  uint8_t* dbg_step;
};

struct oxm_ctx_impl {
  int device;
  DevOps ops;
};

// Per-thread error text for OXM_ERR_CUDA.
void set_last_error(const char* where, cudaError_t err);

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = (cudaSetDevice(dev) == cudaSuccess);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

inline int check_launch(const char* where) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_last_error(where, err);
    return OXM_ERR_CUDA;
  }
  return OXM_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SM count of the current device (cached per device): grids of kernels that
// stride over a device-side count are sized from it, not from a constant.
inline int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) return 148;
  if (dev < 64) cache[dev] = sms;
  return sms;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

inline unsigned grid_1d(int64_t n, int threads) {
  int64_t g = ceil_div(n, threads);
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// Quiet NaN used for the SO2 "THb == 0" sentinel (core.py:202-209).
__device__ __forceinline__ float qnan_f() { return __int_as_float(0x7fc00000); }

// ld.global.nc: read-only streaming loads for frames / cubes.
template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

}  // namespace oxm

struct oxm_ctx : oxm::oxm_ctx_impl {};
