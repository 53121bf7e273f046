// Off-path helpers on either side of the hot path (SURVEY.md §8f "next"):
//
//  * oxm_synth_frames_f32 -- synthetic RGB frames on the device (synth.py:150-184):
//      cube = exp(-xi x) per band, + N(0, sigma) reflectance noise, floored at
//      1e-6 (synth.py:25, 180-183), rgb = exposure * C cube (synth.py:156-163).
//    Noise comes from a counter-based Philox4x32-10 stream keyed by `seed`
//    and indexed by (frame, pixel, band), so any frame of a long video is
//    reproducible independently (statistically equivalent to the reference's
//    numpy generator, not bit-identical).  Feeds BASELINE config 4 (4096-frame
//    batches) without host generation or PCIe.
//  * oxm_patch_mean_f32 -- per-frame sum / count of finite THb inside a
//    rectangle (timeseries.py:44-73 patch_mean); the NaN-frame interpolation
//    is done on the host like the reference.
#include "oxm_common.cuh"

namespace oxm {
namespace {

constexpr int kSynthThreads = 256;
constexpr int kMeanThreads = 256;

struct SynthOps {
  int L;
  float xi[kMaxBands][3];
  float c[3][kMaxBands];
};

// Philox4x32-10 (Salmon et al., SC'11), one 128-bit block per call.
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * ctr.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * ctr.z;
    const unsigned hi0 = (unsigned)(p0 >> 32), lo0 = (unsigned)p0;
    const unsigned hi1 = (unsigned)(p1 >> 32), lo1 = (unsigned)p1;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

__device__ __forceinline__ float u01(unsigned v) {  // (0, 1]
  return ((float)(v >> 8) + 1.0f) * (1.0f / 16777216.0f);
}

__global__ void __launch_bounds__(kSynthThreads) synth_kernel(const __grid_constant__ SynthOps ops,
                                                              const float* __restrict__ truth, int64_t npx,
                                                              int64_t count, float sigma, float exposure,
                                                              uint2 key, unsigned long long frame0,
                                                              double amplitude, double pulse_hz, double fps,
                                                              float* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * kSynthThreads + threadIdx.x;
  if (t >= npx * count) return;
  const int64_t f = t / npx, p = t - f * npx;
  const unsigned long long fr = frame0 + (unsigned long long)f;
  // pulse_sequence (synth.py:218-222): frame fr scales both haemoglobin planes by
  // m = 1 + amplitude sin(2 pi f fr / fps), same expression order, fp64
  const float m = amplitude != 0.0 ? (float)(1.0 + amplitude * sin(2.0 * 3.141592653589793 * pulse_hz * (double)fr / fps))
                                   : 1.0f;
  const float x0 = ldg(truth + 3 * p) * m, x1 = ldg(truth + 3 * p + 1) * m, x2 = ldg(truth + 3 * p + 2);
  float r0 = 0.f, r1 = 0.f, r2 = 0.f;
  const int L = ops.L;
  for (int l0 = 0; l0 < L; l0 += 4) {
    // 4 uniforms -> 4 normals (two Box-Muller pairs) per Philox block
    const uint4 u = philox(make_uint4((unsigned)p, (unsigned)(p >> 32), (unsigned)fr, (unsigned)(fr >> 32) ^ (unsigned)l0),
                           key);
    float z[4];
    {
      const float ra = sqrtf(-2.f * __logf(u01(u.x))), rb = sqrtf(-2.f * __logf(u01(u.z)));
      float sa, ca, sb, cb;
      __sincosf(6.2831853071795865f * u01(u.y), &sa, &ca);
      __sincosf(6.2831853071795865f * u01(u.w), &sb, &cb);
      z[0] = ra * ca;
      z[1] = ra * sa;
      z[2] = rb * cb;
      z[3] = rb * sb;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = l0 + q;
      if (l < L) {
        float s = __expf(-fmaf(ops.xi[l][0], x0, fmaf(ops.xi[l][1], x1, ops.xi[l][2] * x2)));
        if (sigma > 0.f) s = fmaxf(fmaf(sigma, z[q], s), 1e-6f);
        r0 = fmaf(ops.c[0][l], s, r0);
        r1 = fmaf(ops.c[1][l], s, r1);
        r2 = fmaf(ops.c[2][l], s, r2);
      }
    }
  }
  float* o = out + 3 * t;
  o[0] = exposure * r0;
  o[1] = exposure * r1;
  o[2] = exposure * r2;
}

// One CTA per (frame, row slab): fp64 partial sums in a fixed tree order;
// a second pass adds the slabs of each frame in order -> deterministic.
__global__ void __launch_bounds__(kMeanThreads) patch_mean_kernel(const float* __restrict__ thb, int64_t H, int64_t W,
                                                                  int x, int y, int w, int h, int rows_per_cta,
                                                                  double* __restrict__ psum,
                                                                  unsigned long long* __restrict__ pcnt) {
  __shared__ double ssum[kMeanThreads / 32];
  __shared__ unsigned long long scnt[kMeanThreads / 32];
  const int64_t f = blockIdx.y;
  const int r0 = y + blockIdx.x * rows_per_cta;
  const int r1 = min(r0 + rows_per_cta, y + h);
  double acc = 0.0;
  unsigned long long n = 0;
  for (int r = r0; r < r1; ++r) {
    const float* row = thb + (f * H + r) * W + x;
    for (int c = threadIdx.x; c < w; c += kMeanThreads) {
      const float v = ldg(row + c);
      if (isfinite(v)) {
        acc += (double)v;
        ++n;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    n += __shfl_xor_sync(0xffffffffu, n, o);
  }
  if ((threadIdx.x & 31) == 0) {
    ssum[threadIdx.x >> 5] = acc;
    scnt[threadIdx.x >> 5] = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    unsigned long long c = 0;
    for (int k = 0; k < kMeanThreads / 32; ++k) {
      s += ssum[k];
      c += scnt[k];
    }
    psum[f * gridDim.x + blockIdx.x] = s;
    pcnt[f * gridDim.x + blockIdx.x] = c;
  }
}

__global__ void patch_mean_finish(const double* __restrict__ psum, const unsigned long long* __restrict__ pcnt,
                                  int slabs, int64_t batch, double* __restrict__ sums,
                                  unsigned long long* __restrict__ counts) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= batch) return;
  double s = 0.0;
  unsigned long long c = 0;
  for (int k = 0; k < slabs; ++k) {
    s += psum[f * slabs + k];
    c += pcnt[f * slabs + k];
  }
  sums[f] = s;
  counts[f] = c;
}

// SPC1 map payload (io.py:34-39, 79-80): (H, W, 3) little-endian fp32 in
// (hbo, hb, offset) order, interleaved from the three planes on the device.
__global__ void pack_hwc3_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                 const float* __restrict__ c, int64_t n, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[3 * i] = ldg(a + i);
  out[3 * i + 1] = ldg(b + i);
  out[3 * i + 2] = ldg(c + i);
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_pack_hwc3_f32(const float* a, const float* b, const float* c, int64_t n, float* out,
                                 void* stream) {
  if (n < 0 || (n > 0 && (!a || !b || !c || !out))) return OXM_ERR_ARGUMENT;
  if (n == 0) return OXM_OK;
  pack_hwc3_kernel<<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(a, b, c, n, out);
  return check_launch("pack_hwc3");
}

extern "C" int oxm_synth_pulse_frames_f32(const oxm_ctx* ctx, const float* truth, int64_t height, int64_t width,
                                          int64_t count, double noise_sigma, double exposure, uint64_t seed,
                                          uint64_t frame0, double fps, double pulse_hz, double amplitude, float* out,
                                          void* stream) {
  if (!ctx || height < 1 || width < 1 || count < 0 || noise_sigma < 0 || !(exposure > 0)) return OXM_ERR_ARGUMENT;
  // synth.py:209-216 argument checks (amplitude 0 = static phantom frames)
  if (amplitude < 0 || (amplitude > 0 && !(fps > 0 && pulse_hz > 0 && pulse_hz < fps / 2))) return OXM_ERR_ARGUMENT;
  if (count == 0) return OXM_OK;
  if (!truth || !out) return OXM_ERR_ARGUMENT;
  DeviceGuard dg(ctx->device);
  SynthOps s{};
  s.L = ctx->ops.L;
  for (int l = 0; l < s.L; ++l)
    for (int k = 0; k < 3; ++k) {
      s.xi[l][k] = (float)ctx->ops.xi[l][k];
      s.c[k][l] = (float)ctx->ops.sens[k][l];
    }
  const int64_t npx = height * width;
  const uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  synth_kernel<<<grid_1d(npx * count, kSynthThreads), kSynthThreads, 0, as_stream(stream)>>>(
      s, truth, npx, count, (float)noise_sigma, (float)exposure, key, (unsigned long long)frame0, amplitude, pulse_hz,
      amplitude > 0 ? fps : 1.0, out);
  return check_launch("synth_frames");
}

extern "C" int oxm_synth_frames_f32(const oxm_ctx* ctx, const float* truth, int64_t height, int64_t width,
                                    int64_t count, double noise_sigma, double exposure, uint64_t seed,
                                    uint64_t frame0, float* out, void* stream) {
  return oxm_synth_pulse_frames_f32(ctx, truth, height, width, count, noise_sigma, exposure, seed, frame0, 1.0, 0.0,
                                    0.0, out, stream);
}

extern "C" int oxm_patch_mean_f32(const float* thb, int64_t batch, int64_t height, int64_t width, int x, int y,
                                  int w, int h, double* sums, unsigned long long* counts, void* stream) {
  if (w < 1 || h < 1) return OXM_ERR_ARGUMENT;  // timeseries.py:53-54
  if (x < 0 || y < 0 || x + (int64_t)w > width || y + (int64_t)h > height) return OXM_ERR_ARGUMENT;  // :57-60
  if (batch < 0 || (batch > 0 && (!thb || !sums || !counts))) return OXM_ERR_ARGUMENT;
  if (batch == 0) return OXM_OK;
  if (batch > 65535) return OXM_ERR_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const int rows = 16;
  const int slabs = (int)ceil_div(h, rows);
  void* scratch = nullptr;
  cudaError_t err = cudaMallocAsync(&scratch, (size_t)batch * slabs * 16, s);
  if (err != cudaSuccess) {
    set_last_error("patch_mean scratch", err);
    return OXM_ERR_CUDA;
  }
  double* psum = static_cast<double*>(scratch);
  unsigned long long* pcnt = reinterpret_cast<unsigned long long*>(psum + batch * slabs);
  dim3 grid((unsigned)slabs, (unsigned)batch);
  patch_mean_kernel<<<grid, kMeanThreads, 0, s>>>(thb, height, width, x, y, w, h, rows, psum, pcnt);
  int st = check_launch("patch_mean");
  if (!st) {
    patch_mean_finish<<<grid_1d(batch, 128), 128, 0, s>>>(psum, pcnt, slabs, batch, sums, counts);
    st = check_launch("patch_mean_finish");
  }
  cudaFreeAsync(scratch, s);
  return st;
}
