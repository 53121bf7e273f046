// K6: fused hybrid estimator = estimate_frame(mode="hybrid") for a batch of
// frames (pipeline.py:176-217 + fit_cube pipeline.py:66-94 + THb/SO2
// core.py:197-209).
//
// The hybrid path is linear everywhere except the low-pass EM, and the
// inverse Haar of a low-pass-only pyramid is block constant, so for a pixel p
// in low-pass block b = (py >> n, px >> n)
//     cube(p) = S[b] + solve (rgb(p) - LL_n[b] / 2^n)
// exactly (SURVEY.md §8a "collapse identity"), where LL_n is the reference's
// recursively edge-replicated low-pass (haar.py:80-101) and S the EM spectra
// of LL_n / 2^n (bayes.py:185-207).  Three launches per batch:
//   1. ll_kernel      one thread per low-pass coefficient: the LL chain in
//                     fp64 with the reference's add order (bit-exact LL),
//                     non-finite / negative checks -> flags
//   2. em_soa_kernel  one thread per coefficient: K4 in fp64 -> S (SoA)
//   3. px kernel      one thread per pixel column segment: reconstruct the
//                     26-band spectrum in registers, log, 3x26 fit, THb/SO2.
//                     fp32 variant: MUFU lg2 with S split hi/lo in shared
//                     memory; pixels whose smallest band < fallback_below
//                     are recomputed in fp64 (cancellation guard).
//                     fp64 variant: everything fp64, optional (H,W,L) cube.
// Neither the directional planes nor the 26-channel cube touch HBM on the
// fp32 path: HBM traffic is the frame read twice + the maps written once.
#include <algorithm>

#include "oxm_em.cuh"

namespace oxm {
namespace {

constexpr int kMaxLevels = 24;
constexpr int kLlThreads = 128;
constexpr int kEmThreads = 128;
constexpr int kPxCols = 256;  // pixel columns per CTA in the map kernels

struct LevelDims {
  int n;
  int64_t h[kMaxLevels + 1], w[kMaxLevels + 1];  // [0] = frame
};

// Low-pass value at level K, position (i, j), channel c, with the per-level
// edge replication of haar.py:80-85 (the odd partner falls back to its twin).
template <typename TIn, int K>
struct LowPass {
  __device__ __forceinline__ static double at(const TIn* img, const LevelDims& d, int64_t i, int64_t j, int c,
                                              bool& bad) {
    const int64_t i1 = min(2 * i + 1, d.h[K - 1] - 1);
    const int64_t j1 = min(2 * j + 1, d.w[K - 1] - 1);
    const double a = LowPass<TIn, K - 1>::at(img, d, 2 * i, 2 * j, c, bad);
    const double b = LowPass<TIn, K - 1>::at(img, d, 2 * i, j1, c, bad);
    const double cc = LowPass<TIn, K - 1>::at(img, d, i1, 2 * j, c, bad);
    const double dd = LowPass<TIn, K - 1>::at(img, d, i1, j1, c, bad);
    return 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b), cc), dd);
  }
};

template <typename TIn>
struct LowPass<TIn, 0> {
  __device__ __forceinline__ static double at(const TIn* img, const LevelDims& d, int64_t i, int64_t j, int c,
                                              bool& bad) {
    const double v = (double)ldg(img + (i * d.w[0] + j) * 3 + c);
    bad |= !isfinite(v);
    return v;
  }
};

// Same recursion with a runtime depth (n > 4; rare, correctness path).
template <typename TIn>
__device__ __noinline__ double low_pass_rt(const TIn* img, const LevelDims& d, int k, int64_t i, int64_t j, int c,
                                           bool& bad) {
  if (k == 0) {
    const double v = (double)ldg(img + (i * d.w[0] + j) * 3 + c);
    bad |= !isfinite(v);
    return v;
  }
  const int64_t i1 = min(2 * i + 1, d.h[k - 1] - 1);
  const int64_t j1 = min(2 * j + 1, d.w[k - 1] - 1);
  const double a = low_pass_rt(img, d, k - 1, 2 * i, 2 * j, c, bad);
  const double b = low_pass_rt(img, d, k - 1, 2 * i, j1, c, bad);
  const double cc = low_pass_rt(img, d, k - 1, i1, 2 * j, c, bad);
  const double dd = low_pass_rt(img, d, k - 1, i1, j1, c, bad);
  return 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b), cc), dd);
}

// ybar[c][idx] = LL_n[b, c] / 2^n for every coefficient of every frame.
template <typename TIn, int NLV>
__global__ void __launch_bounds__(kLlThreads) ll_kernel(const TIn* __restrict__ frames, int64_t batch,
                                                        LevelDims d, double* __restrict__ ybar, int64_t nll,
                                                        uint32_t* flags) {
  const int64_t idx = (int64_t)blockIdx.x * kLlThreads + threadIdx.x;
  if (idx >= nll) return;
  const int n = d.n;
  const int64_t hL = d.h[n], wL = d.w[n];
  const int64_t per = hL * wL;
  const int64_t f = idx / per;
  const int64_t rem = idx - f * per;
  const int64_t by = rem / wL, bx = rem - by * wL;
  const TIn* img = frames + f * d.h[0] * d.w[0] * 3;
  const double inv = ldexp(1.0, -n);  // exact
  bool bad = false;
  bool neg = false;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v;
    if constexpr (NLV > 0)
      v = LowPass<TIn, NLV>::at(img, d, by, bx, c, bad);
    else
      v = low_pass_rt<TIn>(img, d, n, by, bx, c, bad);
    v *= inv;
    neg |= v < 0.0;
    ybar[c * nll + idx] = v;
  }
  if (flags && (bad || neg)) atomicOr(flags, (bad ? OXM_FLAG_NONFINITE : 0u) | (neg ? OXM_FLAG_NEGATIVE_LL : 0u));
}

// S[l][idx] = EM spectra of ybar[:, idx]  (SoA, coalesced per band).
template <int KL>
__global__ void __launch_bounds__(kEmThreads) em_soa_kernel(const __grid_constant__ DevOps ops,
                                                            const double* __restrict__ ybar, int64_t nll,
                                                            double* __restrict__ S, int32_t* __restrict__ fits) {
  const int64_t idx = (int64_t)blockIdx.x * kEmThreads + threadIdx.x;
  if (idx >= nll) return;
  const double y0 = ybar[idx], y1 = ybar[nll + idx], y2 = ybar[2 * nll + idx];
  double x0, x1, x2;
  int nf;
  em_coefficient<KL>(ops, y0, y1, y2, nullptr, x0, x1, x2, nf,
                     [&](int l, double v) { S[(int64_t)l * nll + idx] = v; });
  if (fits) fits[idx] = nf;
}

// Per-pixel fp64 spectrum + fit (used by the fp64 kernel and as the fp32
// kernel's cancellation fallback).  Returns x = (hbo, hb, offset) unscaled.
template <int KL, typename CubeStore>
__device__ __forceinline__ void pixel_fit_f64(const DevOps& ops, const double* __restrict__ S, int64_t nll,
                                              int64_t bidx, double d0, double d1, double d2, double& x0,
                                              double& x1, double& x2, CubeStore cube_store) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
  for (int l = 0; l < LM; ++l) {
    if (KL == 0 && l >= L) break;
    const double s = fma(ops.solve[l][2], d2, fma(ops.solve[l][1], d1, fma(ops.solve[l][0], d0, S[(int64_t)l * nll + bidx])));
    cube_store(l, s);
    const double lg = log(fmax(s, ops.eps));
    a0 = fma(ops.fitm[0][l], lg, a0);
    a1 = fma(ops.fitm[1][l], lg, a1);
    a2 = fma(ops.fitm[2][l], lg, a2);
  }
  x0 = -a0;
  x1 = -a1;
  x2 = -a2;
}

struct PxGeom {
  int64_t H, W, hL, wL, nll;
  int n;
  double cal;
};

// fp32 map kernel.  CTA = kPxCols columns x one low-pass block row (2^n pixel
// rows) of one frame; each thread walks the 2^n rows of its column.
template <int KL>
__global__ void __launch_bounds__(kPxCols) px_f32_kernel(const __grid_constant__ DevOps ops,
                                                         const float* __restrict__ frames, PxGeom g,
                                                         const double* __restrict__ S,
                                                         const double* __restrict__ ybar, float* __restrict__ thb,
                                                         float* __restrict__ so2, float* __restrict__ hbo,
                                                         float* __restrict__ hb, float* __restrict__ off) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  const int LS = L | 1;
  extern __shared__ float sm[];
  const int nbmax = (kPxCols >> g.n) + 1;
  float* shi = sm;                  // [nbmax][LS]
  float* slo = shi + nbmax * LS;    // [nbmax][LS]
  float* yhi = slo + nbmax * LS;    // [nbmax][3]
  float* ylo = yhi + nbmax * 3;     // [nbmax][3]

  const int64_t f = blockIdx.z, by = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kPxCols;
  const int64_t clast = min(c0 + kPxCols, g.W) - 1;
  const int64_t bx0 = c0 >> g.n;
  const int nb = (int)((clast >> g.n) - bx0 + 1);
  const int64_t brow = (f * g.hL + by) * g.wL;  // coefficient index of (f, by, 0)

  // stage this tile's block spectra as (hi, lo) fp32 pairs
  for (int q = threadIdx.x; q < nb * L; q += kPxCols) {
    const int l = q / nb, j = q - l * nb;
    const double v = S[(int64_t)l * g.nll + brow + bx0 + j];
    const float h = __double2float_rn(v);
    shi[j * LS + l] = h;
    slo[j * LS + l] = __double2float_rn(v - (double)h);
  }
  for (int q = threadIdx.x; q < nb * 3; q += kPxCols) {
    const int k = q / nb, j = q - k * nb;
    const double v = ybar[(int64_t)k * g.nll + brow + bx0 + j];
    const float h = __double2float_rn(v);
    yhi[j * 3 + k] = h;
    ylo[j * 3 + k] = __double2float_rn(v - (double)h);
  }
  __syncthreads();

  const int64_t col = c0 + threadIdx.x;
  if (col >= g.W) return;
  const int j = (int)((col >> g.n) - bx0);
  const float* sh = shi + j * LS;
  const float* sl = slo + j * LS;
  const float yh0 = yhi[3 * j], yh1 = yhi[3 * j + 1], yh2 = yhi[3 * j + 2];
  const float yl0 = ylo[3 * j], yl1 = ylo[3 * j + 1], yl2 = ylo[3 * j + 2];
  const int64_t bidx = brow + bx0 + j;
  const float cal = (float)g.cal;
  const int64_t r0 = by << g.n;
  const int64_t r1 = min(r0 + ((int64_t)1 << g.n), g.H);
  for (int64_t row = r0; row < r1; ++row) {
    const int64_t p = (f * g.H + row) * g.W + col;
    const float v0 = ldg(frames + 3 * p), v1 = ldg(frames + 3 * p + 1), v2 = ldg(frames + 3 * p + 2);
    const float d0 = (v0 - yh0) - yl0, d1 = (v1 - yh1) - yl1, d2 = (v2 - yh2) - yl2;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, vmin = 3.0e38f;
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      const float s = fmaf(ops.solve_f[l][2], d2, fmaf(ops.solve_f[l][1], d1, fmaf(ops.solve_f[l][0], d0, sl[l]))) + sh[l];
      vmin = fminf(vmin, s);
      const float lg = __log2f(fmaxf(s, ops.eps_f));
      a0 = fmaf(ops.fitl2_f[0][l], lg, a0);
      a1 = fmaf(ops.fitl2_f[1][l], lg, a1);
      a2 = fmaf(ops.fitl2_f[2][l], lg, a2);
    }
    if (vmin < (float)ops.fallback_below) {
      // cancellation guard: redo this pixel in fp64 from the fp64 spectra
      double x0, x1, x2;
      const double D0 = (double)v0 - ybar[bidx];
      const double D1 = (double)v1 - ybar[g.nll + bidx];
      const double D2 = (double)v2 - ybar[2 * g.nll + bidx];
      pixel_fit_f64<KL>(ops, S, g.nll, bidx, D0, D1, D2, x0, x1, x2, [](int, double) {});
      a0 = (float)(x0);
      a1 = (float)(x1);
      a2 = (float)(x2);
    }
    const float xo = a0 * cal, xd = a1 * cal;
    const float co = fmaxf(xo, 0.f);
    const float t = co + fmaxf(xd, 0.f);
    if (thb) thb[p] = t;
    if (so2) so2[p] = t > 0.f ? __fdiv_rn(co, t) : qnan_f();
    if (hbo) hbo[p] = xo;
    if (hb) hb[p] = xd;
    if (off) off[p] = a2;
  }
}

// fp64 map kernel for the drop-in estimate_frame: one thread per pixel,
// optional (H, W, L) cube, hbo/hb/offset in fp64.
template <int KL>
__global__ void __launch_bounds__(128) px_f64_kernel(const __grid_constant__ DevOps ops,
                                                     const double* __restrict__ frames, PxGeom g, int64_t batch,
                                                     const double* __restrict__ S, const double* __restrict__ ybar,
                                                     double* __restrict__ cube, double* __restrict__ hbo,
                                                     double* __restrict__ hb, double* __restrict__ off) {
  const int64_t p = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t npx = batch * g.H * g.W;
  if (p >= npx) return;
  const int L = BandCount<KL>::get(ops);
  const int64_t f = p / (g.H * g.W);
  const int64_t rem = p - f * g.H * g.W;
  const int64_t row = rem / g.W, col = rem - row * g.W;
  const int64_t bidx = (f * g.hL + (row >> g.n)) * g.wL + (col >> g.n);
  const double D0 = ldg(frames + 3 * p) - ybar[bidx];
  const double D1 = ldg(frames + 3 * p + 1) - ybar[g.nll + bidx];
  const double D2 = ldg(frames + 3 * p + 2) - ybar[2 * g.nll + bidx];
  double x0, x1, x2;
  double* crow = cube ? cube + p * L : nullptr;
  pixel_fit_f64<KL>(ops, S, g.nll, bidx, D0, D1, D2, x0, x1, x2, [&](int l, double s) {
    if (crow) crow[l] = s;
  });
  if (hbo) hbo[p] = x0 * g.cal;
  if (hb) hb[p] = x1 * g.cal;
  if (off) off[p] = x2;
}

int level_dims(int64_t H, int64_t W, int n, LevelDims& d) {
  if (n < 1 || n > kMaxLevels) return OXM_ERR_ARGUMENT;
  d.n = n;
  d.h[0] = H;
  d.w[0] = W;
  for (int k = 1; k <= n; ++k) {
    d.h[k] = (d.h[k - 1] + 1) / 2;
    d.w[k] = (d.w[k - 1] + 1) / 2;
  }
  return OXM_OK;
}

inline void mark(void* const* ev, int i, cudaStream_t s) {
  if (ev && ev[i]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[i]), s);
}

size_t workspace_bytes(int L, int64_t nll) { return sizeof(double) * (size_t)nll * (size_t)(L + 3) + 256; }

template <typename TIn>
int launch_ll(const TIn* frames, int64_t batch, const LevelDims& d, double* ybar, int64_t nll, uint32_t* flags,
              cudaStream_t s) {
  const unsigned grid = grid_1d(nll, kLlThreads);
  switch (d.n) {
    case 1: ll_kernel<TIn, 1><<<grid, kLlThreads, 0, s>>>(frames, batch, d, ybar, nll, flags); break;
    case 2: ll_kernel<TIn, 2><<<grid, kLlThreads, 0, s>>>(frames, batch, d, ybar, nll, flags); break;
    case 3: ll_kernel<TIn, 3><<<grid, kLlThreads, 0, s>>>(frames, batch, d, ybar, nll, flags); break;
    default: ll_kernel<TIn, 0><<<grid, kLlThreads, 0, s>>>(frames, batch, d, ybar, nll, flags); break;
  }
  return check_launch("hybrid_ll");
}

int launch_em_soa(const DevOps& ops, const double* ybar, int64_t nll, double* S, int32_t* fits, cudaStream_t s) {
  const unsigned grid = grid_1d(nll, kEmThreads);
  if (ops.L == 26)
    em_soa_kernel<26><<<grid, kEmThreads, 0, s>>>(ops, ybar, nll, S, fits);
  else
    em_soa_kernel<0><<<grid, kEmThreads, 0, s>>>(ops, ybar, nll, S, fits);
  return check_launch("hybrid_em");
}

template <typename TIn>
int hybrid_prologue(const oxm_ctx* ctx, const TIn* frames, int64_t batch, int64_t H, int64_t W, int n,
                    void* ws, size_t ws_bytes, LevelDims& d, int64_t& nll, double*& S, double*& ybar) {
  if (!ctx || batch < 0 || !frames) return OXM_ERR_ARGUMENT;
  if (n < 1 || n > kMaxLevels) return OXM_ERR_ARGUMENT;
  // pipeline.py:177-181: frame must be at least 2^n in both dimensions
  if (H < ((int64_t)1 << n) || W < ((int64_t)1 << n)) return OXM_ERR_ARGUMENT;
  int st = level_dims(H, W, n, d);
  if (st) return st;
  nll = batch * d.h[n] * d.w[n];
  const int L = ctx->ops.L;
  if (!ws || ws_bytes < workspace_bytes(L, nll)) return OXM_ERR_WORKSPACE;
  uintptr_t p = (reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255);
  ybar = reinterpret_cast<double*>(p);
  S = ybar + 3 * nll;
  return OXM_OK;
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" size_t oxm_hybrid_workspace_bytes(const oxm_ctx* ctx, int64_t batch, int64_t height, int64_t width,
                                             int n_levels) {
  LevelDims d;
  if (!ctx || level_dims(height, width, n_levels, d) != OXM_OK || batch < 0) return 0;
  return workspace_bytes(ctx->ops.L, batch * d.h[n_levels] * d.w[n_levels]);
}

extern "C" int oxm_hybrid_maps_f32(const oxm_ctx* ctx, const float* frames, int64_t batch, int64_t height,
                                   int64_t width, int n_levels, double calibration, void* workspace,
                                   size_t workspace_bytes_, float* thb, float* so2, float* hbo, float* hb,
                                   float* offset, int32_t* fits, uint32_t* flags, void* stream,
                                   void* const* ev) {
  LevelDims d;
  int64_t nll;
  double *S, *ybar;
  int st = hybrid_prologue<float>(ctx, frames, batch, height, width, n_levels, workspace, workspace_bytes_, d, nll,
                                  S, ybar);
  if (st) return st;
  if (batch == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  cudaStream_t s = as_stream(stream);
  mark(ev, 0, s);
  if ((st = launch_ll<float>(frames, batch, d, ybar, nll, flags, s))) return st;
  mark(ev, 1, s);
  if ((st = launch_em_soa(ctx->ops, ybar, nll, S, fits, s))) return st;
  mark(ev, 2, s);
  PxGeom g{height, width, d.h[n_levels], d.w[n_levels], nll, n_levels, calibration};
  const int L = ctx->ops.L;
  const int nbmax = (kPxCols >> n_levels) + 1;
  const size_t smem = sizeof(float) * (size_t)nbmax * (2 * (L | 1) + 6);
  dim3 grid((unsigned)ceil_div(width, kPxCols), (unsigned)d.h[n_levels], (unsigned)batch);
  if (grid.y > 65535 || grid.z > 65535) return OXM_ERR_ARGUMENT;
  if (L == 26)
    px_f32_kernel<26><<<grid, kPxCols, smem, s>>>(ctx->ops, frames, g, S, ybar, thb, so2, hbo, hb, offset);
  else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(px_f32_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    px_f32_kernel<0><<<grid, kPxCols, smem, s>>>(ctx->ops, frames, g, S, ybar, thb, so2, hbo, hb, offset);
  }
  st = check_launch("hybrid_px_f32");
  mark(ev, 3, s);
  return st;
}

extern "C" int oxm_hybrid_frame_f64(const oxm_ctx* ctx, const double* frames, int64_t batch, int64_t height,
                                    int64_t width, int n_levels, double calibration, void* workspace,
                                    size_t workspace_bytes_, double* cube, double* hbo, double* hb, double* offset,
                                    int32_t* fits, uint32_t* flags, void* stream, void* const* ev) {
  LevelDims d;
  int64_t nll;
  double *S, *ybar;
  int st = hybrid_prologue<double>(ctx, frames, batch, height, width, n_levels, workspace, workspace_bytes_, d, nll,
                                   S, ybar);
  if (st) return st;
  if (batch == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  cudaStream_t s = as_stream(stream);
  mark(ev, 0, s);
  if ((st = launch_ll<double>(frames, batch, d, ybar, nll, flags, s))) return st;
  mark(ev, 1, s);
  if ((st = launch_em_soa(ctx->ops, ybar, nll, S, fits, s))) return st;
  mark(ev, 2, s);
  PxGeom g{height, width, d.h[n_levels], d.w[n_levels], nll, n_levels, calibration};
  const int64_t npx = batch * height * width;
  if (ctx->ops.L == 26)
    px_f64_kernel<26><<<grid_1d(npx, 128), 128, 0, s>>>(ctx->ops, frames, g, batch, S, ybar, cube, hbo, hb, offset);
  else
    px_f64_kernel<0><<<grid_1d(npx, 128), 128, 0, s>>>(ctx->ops, frames, g, batch, S, ybar, cube, hbo, hb, offset);
  st = check_launch("hybrid_px_f64");
  mark(ev, 3, s);
  return st;
}
