// K3 (per-coefficient 3 -> L unmix) and K5 (per-pixel Beer-Lambert fit),
// plus the Beer-Lambert forward model used by expected_spectrum.
//
// K3 replaces tikhonov_unmix (unmix.py:77-82) / lsq_unmix (unmix.py:21-37):
//   out[i, l] = sum_k M[l, k] rgb[i, k]        (rgb @ M.T)
// K5 replaces fit_cube (pipeline.py:66-94) / fit_concentration (bayes.py:138-151):
//   x[i] = -fit_mat @ log(max(cube[i], eps));  x *= (cal, cal, 1)
// Both are HBM-bound streaming kernels: each CTA moves a contiguous slab of
// (n, L) rows through shared memory so every global access is coalesced.
#include "oxm_common.cuh"
#include "oxm_tma.cuh"

namespace oxm {
namespace {

constexpr int kRows = 128;  // coefficients / pixels per CTA

struct Mat3 {
  int L;
  double m[kMaxBands][3];
  float mf[kMaxBands][3];
};

template <typename T>
__device__ __forceinline__ T dot3(const Mat3& M, int l, T y0, T y1, T y2);

template <>
__device__ __forceinline__ double dot3<double>(const Mat3& M, int l, double y0, double y1, double y2) {
  return fma(M.m[l][2], y2, fma(M.m[l][1], y1, M.m[l][0] * y0));
}
template <>
__device__ __forceinline__ float dot3<float>(const Mat3& M, int l, float y0, float y1, float y2) {
  return fmaf(M.mf[l][2], y2, fmaf(M.mf[l][1], y1, M.mf[l][0] * y0));
}

template <typename T>
__global__ void __launch_bounds__(kRows) unmix_kernel(const __grid_constant__ Mat3 M, const T* __restrict__ rgb,
                                                      int64_t n, T* __restrict__ out) {
  extern __shared__ unsigned char smem_raw[];
  T* sin = reinterpret_cast<T*>(smem_raw);  // [kRows*3]
  T* sout = sin + kRows * 3;                // [kRows*L]
  const int L = M.L;
  const int64_t base = (int64_t)blockIdx.x * kRows;
  const int64_t cnt = min64(kRows, n - base);
  for (int64_t k = threadIdx.x; k < cnt * 3; k += kRows) sin[k] = ldg(rgb + base * 3 + k);
  __syncthreads();
  if (threadIdx.x < cnt) {
    const T y0 = sin[3 * threadIdx.x], y1 = sin[3 * threadIdx.x + 1], y2 = sin[3 * threadIdx.x + 2];
    T* row = sout + threadIdx.x * L;
    for (int l = 0; l < L; ++l) row[l] = dot3<T>(M, l, y0, y1, y2);
  }
  __syncthreads();
  T* dst = out + base * L;
  for (int64_t k = threadIdx.x; k < cnt * L; k += kRows) dst[k] = sout[k];
}

// KL > 0: band count fixed at compile time (staging index math by constant
// division, band loop unrolled); KL == 0: generic L.  32-bit index math
// inside a CTA slab (cnt * L <= kRows * kMaxBands).
// BULK: the CTA's slab of kRows x L values is contiguous in global memory and
// arrives by one cp.async.bulk (TMA) copy into shared memory (row stride L);
// otherwise (partial last slab, unaligned cube) per-thread coalesced loads fill
// rows of odd stride L | 1.
template <typename T, int KL, bool BULK>
__global__ void __launch_bounds__(kRows) fit_kernel(const __grid_constant__ DevOps ops, const T* __restrict__ cube,
                                                    int64_t n, double cal, T* __restrict__ hbo, T* __restrict__ hb,
                                                    T* __restrict__ off) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);
  __shared__ __align__(8) uint64_t bar;
  const int L = KL > 0 ? KL : ops.L;
  const int64_t base = (int64_t)blockIdx.x * kRows;
  const int cnt = (int)min64(kRows, n - base);
  const T* src = cube + base * L;
  int LS;
  if constexpr (BULK) {
    LS = L;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_fence_init();
      mbar_expect_tx(&bar, (uint32_t)(sizeof(T) * kRows * L));
      bulk_load_1d(stage, src, (uint32_t)(sizeof(T) * kRows * L), &bar);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&bar, 0);
  } else {
    LS = L | 1;  // odd row stride: conflict-free per-thread row walks
    for (int k = threadIdx.x; k < cnt * L; k += kRows) {
      const int r = k / L, l = k - r * L;
      stage[r * LS + l] = ldg(src + k);
    }
    __syncthreads();
  }
  if ((int)threadIdx.x >= cnt) return;
  const T* row = stage + threadIdx.x * LS;
  T x0, x1, x2;
  if constexpr (sizeof(T) == 8) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll(KL > 0 ? KL : 1)
    for (int l = 0; l < L; ++l) {
      const double lg = log(fmax((double)row[l], ops.eps));
      a0 = fma(ops.fitm[0][l], lg, a0);
      a1 = fma(ops.fitm[1][l], lg, a1);
      a2 = fma(ops.fitm[2][l], lg, a2);
    }
    x0 = -a0;
    x1 = -a1;
    x2 = -a2;
  } else {
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll(KL > 0 ? KL : 1)
    for (int l = 0; l < L; ++l) {
      const float lg = __log2f(fmaxf((float)row[l], ops.eps_f));
      a0 = fmaf(ops.fitl2_f[0][l], lg, a0);
      a1 = fmaf(ops.fitl2_f[1][l], lg, a1);
      a2 = fmaf(ops.fitl2_f[2][l], lg, a2);
    }
    x0 = a0;
    x1 = a1;
    x2 = a2;
  }
  const int64_t i = base + threadIdx.x;
  if (hbo) hbo[i] = x0 * (T)cal;
  if (hb) hb[i] = x1 * (T)cal;
  if (off) off[i] = x2;
}

__global__ void __launch_bounds__(kRows) expected_kernel(const __grid_constant__ DevOps ops,
                                                         const double* __restrict__ x, int64_t n,
                                                         double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kRows + threadIdx.x;
  if (i >= n) return;
  const int L = ops.L;
  const double x0 = x[3 * i], x1 = x[3 * i + 1], x2 = x[3 * i + 2];
  for (int l = 0; l < L; ++l) {
    const double arg = fma(ops.xi[l][2], x2, fma(ops.xi[l][1], x1, ops.xi[l][0] * x0));
    out[i * L + l] = exp(-arg);
  }
}

int build_mat(int L, const double* matrix, Mat3& M) {
  if (L < 1 || L > kMaxBands || !matrix) return OXM_ERR_ARGUMENT;
  M.L = L;
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < 3; ++k) {
      M.m[l][k] = matrix[3 * l + k];
      M.mf[l][k] = (float)matrix[3 * l + k];
    }
  return OXM_OK;
}

template <typename T>
int unmix_impl(int L, const double* matrix, const T* rgb, int64_t n, T* out, cudaStream_t s) {
  Mat3 M{};
  int st = build_mat(L, matrix, M);
  if (st) return st;
  if (n < 0 || (n > 0 && (!rgb || !out))) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  const size_t smem = sizeof(T) * kRows * (3 + L);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(unmix_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unmix_kernel<T><<<grid_1d(n, kRows), kRows, smem, s>>>(M, rgb, n, out);
  return check_launch("unmix");
}

template <typename T>
int fit_impl(const oxm_ctx* ctx, const T* cube, int64_t n, double cal, T* hbo, T* hb, T* off, cudaStream_t s) {
  if (!ctx || n < 0 || (n > 0 && !cube)) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  const int L = ctx->ops.L;
  const size_t smem = sizeof(T) * kRows * (L | 1);
  const int64_t full = n / kRows;  // CTAs with a whole slab
  // whole slabs by bulk copy when every slab start is 16-byte aligned
  const bool bulk = (reinterpret_cast<uintptr_t>(cube) & 15) == 0 && (sizeof(T) * kRows * L) % 16 == 0 && full > 0;
  auto launch = [&](auto kern, int64_t first, int64_t cnt) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t off_px = first * kRows;
    kern<<<(unsigned)cnt, kRows, smem, s>>>(ctx->ops, cube + off_px * L, n - off_px, cal, hbo ? hbo + off_px : nullptr,
                                            hb ? hb + off_px : nullptr, off ? off + off_px : nullptr);
  };
  if (bulk) {
    if (L == 26)
      launch(fit_kernel<T, 26, true>, 0, full);
    else
      launch(fit_kernel<T, 0, true>, 0, full);
  }
  const int64_t first = bulk ? full : 0;
  const int64_t rest = (int64_t)grid_1d(n - first * kRows, kRows);
  if (n > first * kRows) {
    if (L == 26)
      launch(fit_kernel<T, 26, false>, first, rest);
    else
      launch(fit_kernel<T, 0, false>, first, rest);
  }
  return check_launch("fit");
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_unmix_f32(int n_bands, const double* matrix, const float* rgb, int64_t n, float* out,
                             void* stream) {
  return unmix_impl<float>(n_bands, matrix, rgb, n, out, as_stream(stream));
}

extern "C" int oxm_unmix_f64(int n_bands, const double* matrix, const double* rgb, int64_t n, double* out,
                             void* stream) {
  return unmix_impl<double>(n_bands, matrix, rgb, n, out, as_stream(stream));
}

extern "C" int oxm_fit_f32(const oxm_ctx* ctx, const float* cube, int64_t n, double calibration, float* hbo,
                           float* hb, float* offset, void* stream) {
  return fit_impl<float>(ctx, cube, n, calibration, hbo, hb, offset, as_stream(stream));
}

extern "C" int oxm_fit_f64(const oxm_ctx* ctx, const double* cube, int64_t n, double calibration, double* hbo,
                           double* hb, double* offset, void* stream) {
  return fit_impl<double>(ctx, cube, n, calibration, hbo, hb, offset, as_stream(stream));
}

extern "C" int oxm_expected_spectrum_f64(const oxm_ctx* ctx, const double* x, int64_t n, double* out,
                                         void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!x || !out))) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  expected_kernel<<<grid_1d(n, kRows), kRows, 0, as_stream(stream)>>>(ctx->ops, x, n, out);
  return check_launch("expected_spectrum");
}
