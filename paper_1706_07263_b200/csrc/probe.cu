// Roofline probes: measured pipe peaks for the non-GEMM kernels.
//
// MEASURED_PEAKS.json carries HBM copy bandwidth and cuBLAS bf16 throughput,
// neither of which bounds the EM (fp64 FMA pipe) or the per-pixel fit (MUFU).
// These two kernels saturate those pipes with 8 independent dependency
// chains per thread (enough ILP to cover the pipe latency at full occupancy)
// so bench.py can report achieved / measured-peak for them.
#include "oxm_common.cuh"
#include "oxm_math.cuh"

namespace oxm {
namespace {

constexpr int kProbeThreads = 256;

__global__ void __launch_bounds__(kProbeThreads) fp64_fma_probe(int iters, double* sink) {
  double a[8];
  const double m = 1.0 + 1e-12 * threadIdx.x, c = 1e-9;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + k * 1e-3 + blockIdx.x * 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], m, c);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) sink[threadIdx.x] = s;  // keeps the chains live
}

__global__ void __launch_bounds__(kProbeThreads) mufu_lg2_probe(int iters, float* sink) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.5f + k * 0.1f + threadIdx.x * 1e-4f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = __log2f(a[k]) + 2.0f;  // stays in [2, 3]
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678f) sink[threadIdx.x] = s;
}

__global__ void __launch_bounds__(kProbeThreads) math_selftest_kernel(const double* __restrict__ in, int64_t n,
                                                                        int which, double* __restrict__ out) {
  __shared__ MathSmem mt;
  load_math_tables(mt);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kProbeThreads + threadIdx.x;
  if (i >= n) return;
  out[i] = which == 0 ? exp_scaled(in[i], mt) : log_tab(in[i], mt.logt);
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_probe_fp64_fma(int blocks, int iters, double* sink, double* ops, void* stream) {
  if (blocks < 1 || iters < 1 || !sink) return OXM_ERR_ARGUMENT;
  fp64_fma_probe<<<blocks, kProbeThreads, 0, as_stream(stream)>>>(iters, sink);
  if (ops) *ops = (double)blocks * kProbeThreads * (double)iters * 16.0 * 8.0;
  return check_launch("probe_fp64_fma");
}

extern "C" int oxm_probe_mufu_lg2(int blocks, int iters, float* sink, double* ops, void* stream) {
  if (blocks < 1 || iters < 1 || !sink) return OXM_ERR_ARGUMENT;
  mufu_lg2_probe<<<blocks, kProbeThreads, 0, as_stream(stream)>>>(iters, sink);
  if (ops) *ops = (double)blocks * kProbeThreads * (double)iters * 16.0 * 8.0;
  return check_launch("probe_mufu_lg2");
}

extern "C" int oxm_selftest_math(const double* in, int64_t n, int which, double* out, void* stream) {
  if (n < 0 || (which != 0 && which != 1) || (n > 0 && (!in || !out))) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  math_selftest_kernel<<<grid_1d(n, kProbeThreads), kProbeThreads, 0, as_stream(stream)>>>(in, n, which, out);
  return check_launch("selftest_math");
}
