// K4: standalone low-pass estimator (estimate_lowpass, bayes.py:210-272) and
// the shape-prior update for arbitrary (y, e) (expectation_step, bayes.py:162-182).
//
// The estimator is em_persistent_kernel (oxm_em.cuh); here it writes spectra
// row-major (n, L) like the reference's return value (the drop-in API path;
// the video path in hybrid.cu writes them SoA).
#include "oxm_em.cuh"

namespace oxm {
namespace {


template <int KL>
__global__ void __launch_bounds__(kEmThreads) expectation_kernel(const __grid_constant__ DevOps ops,
                                                                 const double* __restrict__ y,
                                                                 const double* __restrict__ e, int64_t n,
                                                                 double* __restrict__ out) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  const int64_t i = (int64_t)blockIdx.x * kEmThreads + threadIdx.x;
  if (i >= n) return;
  const double* ei = e + i * L;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
  for (int l = 0; l < LM; ++l) {
    if (KL == 0 && l >= L) break;
    const double el = ei[l];
    c0 = fma(ops.sens[0][l], el, c0);
    c1 = fma(ops.sens[1][l], el, c1);
    c2 = fma(ops.sens[2][l], el, c2);
  }
  const double r0 = y[3 * i] - c0, r1 = y[3 * i + 1] - c1, r2 = y[3 * i + 2] - c2;
#pragma unroll(KL > 0 ? LM : 1)
  for (int l = 0; l < LM; ++l) {
    if (KL == 0 && l >= L) break;
    out[i * L + l] = fma(ops.gain[l][2], r2, fma(ops.gain[l][1], r1, fma(ops.gain[l][0], r0, ei[l])));
  }
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_em_lowpass(const oxm_ctx* ctx, const double* y, const double* init, int64_t n, double* spectra,
                              double* x, int32_t* fits, void* stream) {
  if (!ctx || n < 0 || (n > 0 && !y)) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  if (!spectra) return OXM_ERR_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  void* scratch = nullptr;
  // scratch: EM chunk counter (zeroed by em_init_kernel), x_init [3][n]
  // (+ fit counts when the caller does not want them)
  const size_t bytes = 256 + sizeof(double) * 3 * (size_t)n + (fits ? 0 : sizeof(int32_t) * (size_t)n);
  cudaError_t err = cudaMallocAsync(&scratch, bytes, s);
  if (err != cudaSuccess) {
    set_last_error("em_lowpass scratch", err);
    return OXM_ERR_CUDA;
  }
  EmIO io{};
  io.y = y;
  io.y_soa = 0;
  io.init = init;
  io.n = n;
  io.S = spectra;
  io.x = x;
  io.work = static_cast<unsigned long long*>(scratch);
  io.xinit = reinterpret_cast<double*>(static_cast<unsigned char*>(scratch) + 256);
  io.fits = fits ? fits : reinterpret_cast<int32_t*>(io.xinit + 3 * n);
  const int st = ctx->ops.L == 26 ? launch_em<26, SpecOut::kAosF64>(ctx->ops, io, s)
                                  : launch_em<0, SpecOut::kAosF64>(ctx->ops, io, s);
  cudaFreeAsync(scratch, s);
  return st;
}

extern "C" int oxm_expectation_step(const oxm_ctx* ctx, const double* y, const double* e, int64_t n, double* out,
                                    void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!y || !e || !out))) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  const unsigned grid = grid_1d(n, kEmThreads);
  cudaStream_t s = as_stream(stream);
  if (ctx->ops.L == 26)
    expectation_kernel<26><<<grid, kEmThreads, 0, s>>>(ctx->ops, y, e, n, out);
  else
    expectation_kernel<0><<<grid, kEmThreads, 0, s>>>(ctx->ops, y, e, n, out);
  return check_launch("expectation_step");
}
