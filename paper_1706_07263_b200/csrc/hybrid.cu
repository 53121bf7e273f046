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
// of LL_n / 2^n (bayes.py:185-207).  Launches per batch (fp32 map path):
//   0. zero_counters  fallback / EM work counters
//   1. ll_kernel      one thread per low-pass coefficient: the LL chain in
//                     fp64 with the reference's add order (bit-exact LL),
//                     non-finite / negative checks -> flags, EM fit #1
//   2. em_lead_kernel fp32 fits while rel > K tol (oxm_em.cuh)
//   3. em_persistent_kernel<TAIL>  the remaining fits in fp64 -> S as an
//                     fp32 (hi, lo) pair per band
//   4. px kernel      one thread per (2 columns, R rows of a block): rebuild
//                     the 26-band spectrum in registers, MUFU lg2, 3x26 fit,
//                     THb/SO2; pixels whose smallest band < fallback_below
//                     (cancellation guard, ~0.4 % of textured pixels) are
//                     recomputed in fp64 by their warp right away, except the
//                     "sensitive" ones, which are listed with their blocks for
//   5. em exact pass  all-fp64 EM of those blocks (~1 % of them), then
//   6. px_fallback_kernel  the deferred pixels.
// With the all-fp64 EM schedule (oxm_ctx_set_em_lead ratio <= 1) 2 and 5-6
// go: one all-fp64 persistent EM, every fallback pixel finished in 4.  The fp64 variant
// (drop-in API): everything fp64, optional (H, W, L) cube, no fallback.
// Neither the directional planes nor the 26-channel cube touch HBM on the
// fp32 path: HBM traffic is the frame read twice, the per-block spectra
// (8 B/band/coefficient) once, and the maps written once.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "oxm_em.cuh"
#include "oxm_tma.cuh"

namespace oxm {
namespace {

constexpr int kMaxLevels = 24;
constexpr int kLlThreads = 128;
#ifndef OXM_PX_THREADS
#define OXM_PX_THREADS 64
#endif
constexpr int kPxThreads = OXM_PX_THREADS;  // threads per CTA in the fp32 map kernel (2 pixel columns each)
constexpr int kFbThreads = 128;

struct LevelDims {
  int n;
  int64_t h[kMaxLevels + 1], w[kMaxLevels + 1];  // [0] = frame
};

// Frame sample accessors.  `at(i)` returns sample i (HWC order) as the fp64
// value the reference sees: the float itself, or count * scale for 16-bit PPM
// rasters (io.py:139-162 reads big-endian u16 counts and multiplies by the
// `# scale` comment in fp64).
template <typename T>
struct PlainSrc {
  const T* p;
  static constexpr bool kF32 = sizeof(T) == 4;
  __device__ __forceinline__ double at(int64_t i) const { return (double)ldg(p + i); }
  __device__ __forceinline__ float atf(int64_t i) const { return (float)ldg(p + i); }
};

struct PpmSrc {
  const uint16_t* p;
  double scale;
  int big_endian;
  static constexpr bool kF32 = false;
  __device__ __forceinline__ double at(int64_t i) const {
    unsigned v = ldg(p + i);
    if (big_endian) v = ((v & 0xffu) << 8) | (v >> 8);
    return (double)v * scale;
  }
};

// Low-pass value at level K, position (i, j), channel c, with the per-level
// edge replication of haar.py:80-85 (the odd partner falls back to its twin).
template <typename Src, int K>
struct LowPass {
  __device__ __forceinline__ static double at(const Src& img, int64_t base, const LevelDims& d, int64_t i, int64_t j,
                                              int c, bool& bad) {
    const int64_t i1 = min(2 * i + 1, d.h[K - 1] - 1);
    const int64_t j1 = min(2 * j + 1, d.w[K - 1] - 1);
    const double a = LowPass<Src, K - 1>::at(img, base, d, 2 * i, 2 * j, c, bad);
    const double b = LowPass<Src, K - 1>::at(img, base, d, 2 * i, j1, c, bad);
    const double cc = LowPass<Src, K - 1>::at(img, base, d, i1, 2 * j, c, bad);
    const double dd = LowPass<Src, K - 1>::at(img, base, d, i1, j1, c, bad);
    return 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b), cc), dd);
  }
};

template <typename Src>
struct LowPass<Src, 0> {
  __device__ __forceinline__ static double at(const Src& img, int64_t base, const LevelDims& d, int64_t i, int64_t j,
                                              int c, bool& bad) {
    const double v = img.at(base + (i * d.w[0] + j) * 3 + c);
    bad |= !isfinite(v);
    return v;
  }
};

// Low-pass of NLV more levels for every position of the output plane of
// every frame.  OUT_YBAR: ybar[c][idx] = LL * 2^-scale_exp (SoA, final);
// otherwise an unscaled HWC fp64 plane feeding the next pass (n > 3 is done
// as a chain of <= 3-level passes, no recursion on the device stack).
template <typename Src, int NLV, bool OUT_YBAR>
__global__ void __launch_bounds__(kLlThreads) ll_kernel(const __grid_constant__ DevOps ops, const Src frames,
                                                        int64_t batch, LevelDims d, double* __restrict__ out,
                                                        int64_t nll, int scale_exp, uint32_t* flags,
                                                        double* __restrict__ xinit, uint8_t* __restrict__ blkflag) {
  const int64_t idx = (int64_t)blockIdx.x * kLlThreads + threadIdx.x;
  if (idx >= nll) return;
  const int64_t hL = d.h[NLV], wL = d.w[NLV];
  const int64_t per = hL * wL;
  int64_t f, by, bx;
  if (nll <= 0xffffffffll) {  // 32-bit divisions (64-bit ones are ~70-instruction sequences)
    const uint32_t i32 = (uint32_t)idx, p32 = (uint32_t)per, w32 = (uint32_t)wL;
    const uint32_t f32 = i32 / p32, r32 = i32 - f32 * p32, y32 = r32 / w32;
    f = f32;
    by = y32;
    bx = r32 - y32 * w32;
  } else {
    f = idx / per;
    const int64_t rem = idx - f * per;
    by = rem / wL;
    bx = rem - by * wL;
  }
  const int64_t base = f * d.h[0] * d.w[0] * 3;
  const double inv = ldexp(1.0, -scale_exp);  // exact
  bool bad = false;
  bool neg = false;
  double yv[3];
  double ll[3];
  // fp32 frames, n <= 3 levels, a block whose 2^n x 2^n pixels are all inside
  // the frame (no edge replication at any level) and 16-byte aligned rows: the
  // block's rows as float4 (n >= 2) / float2 (n = 1) loads instead of 3 4^n
  // strided scalars, the same fp64 adds in the same order as LowPass<> (level by
  // level, window by window; n = 3 streams two level-0 rows at a time).  A
  // sample is non-finite iff the fp64 low-pass sum over its block is (fp32
  // inputs cannot overflow fp64): 3 compares instead of one per sample.
  bool fast = false;
  if constexpr (Src::kF32 && std::is_same<Src, PlainSrc<float>>::value && NLV <= 3) {
    constexpr int S = 1 << NLV;
    fast = ((reinterpret_cast<uintptr_t>(frames.p) & 15) == 0) && (d.w[0] & 3) == 0 && S * by + S <= d.h[0] &&
           S * bx + S <= d.w[0];
    if (fast) {
      const float* blk = frames.p + base + ((S * by) * d.w[0] + S * bx) * 3;
      const int64_t rowf = d.w[0] * 3;
      auto win = [](double a, double b2, double cc, double dd) {
        return 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b2), cc), dd);
      };
      if constexpr (NLV == 1) {
        float px[2][6];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float2 v = ldg(reinterpret_cast<const float2*>(blk + r * rowf) + q);
            px[r][2 * q] = v.x;
            px[r][2 * q + 1] = v.y;
          }
#pragma unroll
        for (int c = 0; c < 3; ++c) ll[c] = win(px[0][c], px[0][3 + c], px[1][c], px[1][3 + c]);
      } else if constexpr (NLV == 2) {
        float px[4][12];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float4* rp = reinterpret_cast<const float4*>(blk + r * rowf);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 v = ldg(rp + q);
            px[r][4 * q] = v.x;
            px[r][4 * q + 1] = v.y;
            px[r][4 * q + 2] = v.z;
            px[r][4 * q + 3] = v.w;
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double l1[2][2];
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
              l1[i][j] = win(px[2 * i][6 * j + c], px[2 * i][6 * j + 3 + c], px[2 * i + 1][6 * j + c],
                             px[2 * i + 1][6 * j + 3 + c]);
          ll[c] = win(l1[0][0], l1[0][1], l1[1][0], l1[1][1]);
        }
      } else {
        double l2[2][2][3];
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2) {
          double l1[2][4][3];
#pragma unroll
          for (int i1 = 0; i1 < 2; ++i1) {
            float px[2][24];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const float4* rp = reinterpret_cast<const float4*>(blk + (4 * i2 + 2 * i1 + r) * rowf);
#pragma unroll
              for (int q = 0; q < 6; ++q) {
                const float4 v = ldg(rp + q);
                px[r][4 * q] = v.x;
                px[r][4 * q + 1] = v.y;
                px[r][4 * q + 2] = v.z;
                px[r][4 * q + 3] = v.w;
              }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int c = 0; c < 3; ++c)
                l1[i1][j][c] = win(px[0][6 * j + c], px[0][6 * j + 3 + c], px[1][6 * j + c], px[1][6 * j + 3 + c]);
          }
#pragma unroll
          for (int j2 = 0; j2 < 2; ++j2)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              l2[i2][j2][c] = win(l1[0][2 * j2][c], l1[0][2 * j2 + 1][c], l1[1][2 * j2][c], l1[1][2 * j2 + 1][c]);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) ll[c] = win(l2[0][0][c], l2[0][1][c], l2[1][0][c], l2[1][1][c]);
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) bad |= !isfinite(ll[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v = fast ? ll[c] : LowPass<Src, NLV>::at(frames, base, d, by, bx, c, bad);
    if constexpr (OUT_YBAR) {
      v *= inv;
      neg |= v < 0.0;
      out[c * nll + idx] = v;
    } else {
      out[3 * idx + c] = v;
    }
    yv[c] = v;
  }
  if (flags && (bad || neg)) atomicOr(flags, (bad ? OXM_FLAG_NONFINITE : 0u) | (neg ? OXM_FLAG_NEGATIVE_LL : 0u));
  if constexpr (OUT_YBAR) {
    if (blkflag) blkflag[idx] = 0;  // exact-block marks of this launch (mark_exact_blocks)
    // fit #1 of the EM (bayes.py:241-250) while the frame streams in
    if (xinit) {
      double x0, x1, x2;
      if (ops.L == 26)
        start_fit<26>(ops, log_table_global(), yv[0], yv[1], yv[2], nullptr, x0, x1, x2);
      else
        start_fit<0>(ops, log_table_global(), yv[0], yv[1], yv[2], nullptr, x0, x1, x2);
      xinit[idx] = x0;
      xinit[nll + idx] = x1;
      xinit[2 * nll + idx] = x2;
    }
  }
}

// ---------------------------------------------------------------------------
// TMA-staged low-pass kernel (fp32 frames, one pass of n <= 2 levels): the
// same outputs as ll_kernel<PlainSrc<float>, NLV, true>, bit for bit.
//
// The batch is viewed as one 2D plane of B*H rows x 3W floats.  A CTA owns a
// tile of TY x TX low-pass blocks (TY 2^n rows x TX 2^n pixels), staged into
// shared memory by one cp.async.bulk.tensor per tile.  Each thread owns one
// low-pass coefficient: it reduces its block to the three fp64 low-pass
// values straight out of shared memory -- interior blocks as conflict-free
// vector loads with compile-time offsets, edge blocks (a tile hanging over
// the frame) through clamped coordinates that reproduce the reference's
// per-level edge replication and always stay inside the tile -- and then the
// tile buffer is released: the elected thread issues the TMA for the CTA's
// next tile (persistent grid, tiles strided by gridDim) while the warps run
// the fp64 start fit (26 table logs per coefficient) and the stores.  One
// buffer per CTA keeps 8 CTAs resident per SM for that fp64 phase.  Rows of
// a tile that belong to the next frame (or lie past the batch, zero-filled)
// are never read.  A sample is non-finite iff the fp64 low-pass sum over its
// block is (fp32 inputs cannot overflow fp64): 3 compares per coefficient.
#ifndef OXM_LL_TMA_THREADS
#define OXM_LL_TMA_THREADS 32
#endif
template <int NLV>
struct LlTma {
  static_assert(NLV == 1 || NLV == 2, "3-level passes keep the per-thread-load ll_kernel (64 samples x 3 channels "
                                      "per thread do not fit a TMA tile pipeline's register budget)");
  static constexpr int S = 1 << NLV;
  // one warp per CTA and per tile: the tile hand-off needs only __syncwarp,
  // so warps never wait for each other (32 CTAs = 32 warps per SM)
  static constexpr int kThreads = OXM_LL_TMA_THREADS;  // coefficients (threads) per tile
  static constexpr int TX = NLV == 1 ? 32 : 16;
  static constexpr int TY = kThreads / TX;
  static constexpr int kRowF = TX * S * 3;                // floats per tile row (box inner dim, 192)
  static constexpr int kRows = TY * S;
  static constexpr int kTileF = kRowF * kRows;
  static constexpr uint32_t kTileBytes = kTileF * 4;
  static constexpr size_t kSmem = (size_t)kTileBytes;
  static constexpr int kMinBlocks = (NLV == 1 ? 1536 : 1024) / kThreads > 32 ? 32 : (NLV == 1 ? 1536 : 1024) / kThreads;
};

// level-K low-pass at level-K position (i, j) with the reference's per-level
// edge replication (LowPass<> on a tile whose origin is frame pixel (r0, c0))
template <int K, int ROWF>
struct LpTile {
  __device__ __forceinline__ static double at(const float* t, int r0, int c0, const LevelDims& d, int i, int j, int c) {
    const int i1 = (int)min((int64_t)(2 * i + 1), d.h[K - 1] - 1);
    const int j1 = (int)min((int64_t)(2 * j + 1), d.w[K - 1] - 1);
    const double a = LpTile<K - 1, ROWF>::at(t, r0, c0, d, 2 * i, 2 * j, c);
    const double b = LpTile<K - 1, ROWF>::at(t, r0, c0, d, 2 * i, j1, c);
    const double cc = LpTile<K - 1, ROWF>::at(t, r0, c0, d, i1, 2 * j, c);
    const double dd = LpTile<K - 1, ROWF>::at(t, r0, c0, d, i1, j1, c);
    return 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b), cc), dd);
  }
};
template <int ROWF>
struct LpTile<0, ROWF> {
  __device__ __forceinline__ static double at(const float* t, int r0, int c0, const LevelDims&, int i, int j, int c) {
    return (double)t[(i - r0) * ROWF + (j - c0) * 3 + c];
  }
};

template <int NLV>
__global__ void __launch_bounds__(LlTma<NLV>::kThreads, LlTma<NLV>::kMinBlocks) ll_tma_kernel(
    const __grid_constant__ DevOps ops, const __grid_constant__ CUtensorMap tmap, int64_t batch, LevelDims d,
    double* __restrict__ ybar, int64_t nll, uint32_t* flags, double* __restrict__ xinit,
    uint8_t* __restrict__ blkflag, int tiles_x, int tiles_y) {
  using G = LlTma<NLV>;
  extern __shared__ __align__(128) float tile[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t per_frame = (int64_t)tiles_x * tiles_y;
  const int64_t ntiles = batch * per_frame;
  const int H0 = (int)d.h[0], W0 = (int)d.w[0], hL = (int)d.h[NLV], wL = (int)d.w[NLV];
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int64_t t) {
    if (t >= ntiles) return;
    const int64_t f = t / per_frame;
    const int r = (int)(t - f * per_frame);
    const int ty = r / tiles_x, tx = r - ty * tiles_x;
    mbar_expect_tx(&bar, G::kTileBytes);
    tma_load_2d(tile, &tmap, tx * G::kRowF, (int)(f * H0) + ty * G::kRows, &bar);
  };
  if (tid == 0) issue(blockIdx.x);
  const int ly = tid / G::TX, lx = tid - ly * G::TX;
  const double inv = ldexp(1.0, -NLV);  // exact
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int64_t f = t / per_frame;
    const int r = (int)(t - f * per_frame);
    const int ty = r / tiles_x, tx = r - ty * tiles_x;
    const int by = ty * G::TY + ly, bx = tx * G::TX + lx;
    const bool mine = by < hL && bx < wL;
    mbar_wait(&bar, it & 1);
    double ll[3] = {0.0, 0.0, 0.0};
    if (mine) {
      const int py = by * G::S, px = bx * G::S;
      if (py + G::S <= H0 && px + G::S <= W0) {
        const float* p = tile + ly * G::S * G::kRowF + lx * G::S * 3;
        if constexpr (NLV == 2) {
          float v[4][12];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const float4 w = *reinterpret_cast<const float4*>(p + rr * G::kRowF + 4 * q);
              v[rr][4 * q] = w.x;
              v[rr][4 * q + 1] = w.y;
              v[rr][4 * q + 2] = w.z;
              v[rr][4 * q + 3] = w.w;
            }
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double l1[2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const double a = v[2 * i][6 * j + c], b = v[2 * i][6 * j + 3 + c];
                const double cc = v[2 * i + 1][6 * j + c], dd = v[2 * i + 1][6 * j + 3 + c];
                l1[i][j] = 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(a, b), cc), dd);
              }
            ll[c] = 0.5 * __dadd_rn(__dadd_rn(__dadd_rn(l1[0][0], l1[0][1]), l1[1][0]), l1[1][1]);
          }
        } else if constexpr (NLV == 1) {
          float v[2][6];
#pragma unroll
          for (int rr = 0; rr < 2; ++rr)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const float2 w = *reinterpret_cast<const float2*>(p + rr * G::kRowF + 2 * q);
              v[rr][2 * q] = w.x;
              v[rr][2 * q + 1] = w.y;
            }
#pragma unroll
          for (int c = 0; c < 3; ++c)
            ll[c] = 0.5 * __dadd_rn(__dadd_rn(__dadd_rn((double)v[0][c], (double)v[0][3 + c]), (double)v[1][c]),
                                    (double)v[1][3 + c]);
        }
      } else {
        const int r0 = ty * G::kRows, c0 = tx * G::TX * G::S;
#pragma unroll
        for (int c = 0; c < 3; ++c) ll[c] = LpTile<NLV, G::kRowF>::at(tile, r0, c0, d, by, bx, c);
      }
    }
    if constexpr (G::kThreads == 32) __syncwarp(); else __syncthreads();  // blocks in registers: buffer free
    if (tid == 0) {
      fence_proxy_async();
      issue(t + gridDim.x);
    }
    if (mine) {
      const int64_t idx = (f * hL + by) * wL + bx;
      bool bad = false, neg = false;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        bad |= !isfinite(ll[c]);
        ll[c] *= inv;
        neg |= ll[c] < 0.0;
        ybar[c * nll + idx] = ll[c];
      }
      if (flags && (bad || neg)) atomicOr(flags, (bad ? OXM_FLAG_NONFINITE : 0u) | (neg ? OXM_FLAG_NEGATIVE_LL : 0u));
      if (blkflag) blkflag[idx] = 0;
      if (xinit) {
        double x0, x1, x2;
        if (ops.L == 26)
          start_fit<26>(ops, log_table_global(), ll[0], ll[1], ll[2], nullptr, x0, x1, x2);
        else
          start_fit<0>(ops, log_table_global(), ll[0], ll[1], ll[2], nullptr, x0, x1, x2);
        xinit[idx] = x0;
        xinit[nll + idx] = x1;
        xinit[2 * nll + idx] = x2;
      }
    }
  }
}

// TMA low-pass launch; returns false (nothing launched) when the frames
// cannot be described by a tensor map -- the caller then runs ll_kernel
template <int NLV>
bool launch_ll_tma_n(const DevOps& ops, const float* frames, int64_t batch, const LevelDims& d, double* ybar,
                     int64_t nll, uint32_t* flags, double* xinit, uint8_t* blkflag, cudaStream_t s) {
  using G = LlTma<NLV>;
  const int64_t H0 = d.h[0], W0 = d.w[0];
  if (batch * H0 >= (int64_t(1) << 31) || 3 * W0 >= (int64_t(1) << 31)) return false;
  CUtensorMap map;
  if (!make_tmap_2d(&map, frames, false, (uint64_t)(3 * W0), (uint64_t)(batch * H0), (uint64_t)(12 * W0), G::kRowF,
                    G::kRows))
    return false;
  auto kern = ll_tma_kernel<NLV>;
  // per launch (the attribute is per function and device; a host call of a few us)
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::kSmem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int tiles_x = (int)ceil_div(d.w[NLV], G::TX), tiles_y = (int)ceil_div(d.h[NLV], G::TY);
  const int64_t ntiles = batch * tiles_x * tiles_y;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::kThreads, G::kSmem) != cudaSuccess || per_sm < 1)
    return false;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)device_sms() * per_sm);
  kern<<<(unsigned)grid, G::kThreads, G::kSmem, s>>>(ops, map, batch, d, ybar, nll, flags, xinit, blkflag, tiles_x,
                                                      tiles_y);
  return true;
}

// Default: the per-thread-load ll_kernel, which measured faster on the fused
// path (profiles/r02_ll_tma_ab.txt: 6.12 vs 6.49 us per 1080p frame; the
// pass is bound jointly by HBM and the fp64 start fit, and the per-thread
// kernel keeps more independent warps in flight than the tile pipeline).
// OXM_LL_TMA=1 in the environment selects ll_tma_kernel (read at each launch).
inline bool ll_tma_enabled() {
  const char* e = getenv("OXM_LL_TMA");
  return e && e[0] == '1';
}

bool launch_ll_tma(const DevOps& ops, const float* frames, int64_t batch, const LevelDims& d, double* ybar, int64_t nll,
                   uint32_t* flags, double* xinit, uint8_t* blkflag, cudaStream_t s) {
  if (!ll_tma_enabled() || batch <= 0) return false;
  switch (d.n) {
    case 1: return launch_ll_tma_n<1>(ops, frames, batch, d, ybar, nll, flags, xinit, blkflag, s);
    case 2: return launch_ll_tma_n<2>(ops, frames, batch, d, ybar, nll, flags, xinit, blkflag, s);
    default: return false;
  }
}

// Per-pixel fp64 spectrum + fit (used by the fp64 kernel and as the fp32
// kernel's cancellation fallback).  Returns x = (hbo, hb, offset) unscaled.
template <int KL, typename SpecLoad, typename CubeStore>
__device__ __forceinline__ void pixel_fit_f64(const DevOps& ops, SpecLoad spec, double d0, double d1, double d2,
                                              double& x0, double& x1, double& x2, CubeStore cube_store) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll(KL > 0 ? LM : 1)
  for (int l = 0; l < LM; ++l) {
    if (KL == 0 && l >= L) break;
    const double s = fma(ops.solve[l][2], d2, fma(ops.solve[l][1], d1, fma(ops.solve[l][0], d0, spec(l))));
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

// Where the per-pixel kernel sends the pixels it does not finish itself
// (the fp64 fallback's "sensitive" ones, see px_f32_kernel's tail).
struct FbOut {
  uint32_t* count;      // deferred pixels listed (fb list)
  uint32_t* list;
  uint8_t* blkflag;     // [nll] block marked for the exact pass
  uint32_t* blk_list;   // marked blocks
  uint32_t* blk_count;
  uint32_t* queued;     // every pixel that took the fp64 fallback (statistics)
  int classify;         // 1: EM precision schedule active (hi parts only, defer sensitive pixels)
};

struct PxGeom {
  int64_t H, W, hL, wL, nll;
  int n;
  double cal;
};

// fp32 map kernel.  CTA = kPxThreads threads x R rows of one low-pass block
// row of one frame; each thread owns two adjacent columns (always in the same
// low-pass block: n >= 1 and the first column is even) and R rows, and walks
// the bands once, updating its 2R pixels per band.  The two columns of a row
// form one float2 lane pair, so every FMA issues as a packed FFMA2.
// Per band and pixel: 3 FMA (solve d, started from the block spectrum), one
// 3-input min per band pair (fallback detection), MUFU lg2, 2 FMA (hbo, hb;
// +1 for the offset plane when requested).  No eps clamp: any pixel with a
// band below fallback_below (>= eps) is recomputed in fp64 by the fixup
// kernel, which applies the reference's clamp.  The block spectrum row
// Shi[coef][Lp] is read with 16-byte loads (Lp = L rounded up to 4), shared
// through L1 by the threads of a block.
template <int KL, int R, bool PLANES, typename Src>
#ifndef OXM_PX_MIN_BLOCKS
#define OXM_PX_MIN_BLOCKS 14
#endif
__global__ void __launch_bounds__(kPxThreads, OXM_PX_MIN_BLOCKS) px_f32_kernel(const __grid_constant__ DevOps ops,
                                                            const Src frames, PxGeom g,
                                                            const float* __restrict__ Shi, const float* __restrict__ Slo,
                                                            int Lp, const double* __restrict__ ybar,
                                                            float* __restrict__ thb, float* __restrict__ so2,
                                                            float* __restrict__ hbo, float* __restrict__ hb,
                                                            float* __restrict__ off, FbOut fb) {
  constexpr int LM = BandCount<KL>::kMax;
  const int L = BandCount<KL>::get(ops);
  const int64_t f = blockIdx.z;
  const int bs = 1 << g.n;               // rows per low-pass block
  const int cpb = bs > R ? bs / R : 1;   // row chunks per block row (a power of two)
  const int64_t by = blockIdx.y >> (__ffs(cpb) - 1);
  const int64_t row0 = by * bs + (int64_t)(blockIdx.y & (cpb - 1)) * R;
  // threads past the right edge stay (on the last even column, storing
  // nothing) so that every warp is full for the cooperative fallback below
  const int64_t col_raw = 2 * ((int64_t)blockIdx.x * kPxThreads + threadIdx.x);  // first of the two columns
  const bool live = col_raw < g.W;
  const int64_t col = live ? col_raw : ((g.W - 1) & ~int64_t(1));
  const bool two = col + 1 < g.W;
  const int nrow = (int)min64(min64(R, g.H - row0), (int64_t)bs);
  const int64_t bidx = (f * g.hL + by) * g.wL + (col >> g.n);

  double yb[3];
  float yh[3], yl[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    yb[k] = ybar[(int64_t)k * g.nll + bidx];
    yh[k] = __double2float_rn(yb[k]);
    yl[k] = __double2float_rn(yb[k] - (double)yh[k]);
  }
  float2 d[R][3], a0[R], a1[R], a2[R];
  float vmin[R][2];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t p = (f * g.H + row0 + min(r, nrow - 1)) * g.W + col;
    const int64_t p1 = two ? p + 1 : p;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if constexpr (Src::kF32) {
        d[r][k].x = (frames.atf(3 * p + k) - yh[k]) - yl[k];  // exact-ish: rgb is an fp32 value
        d[r][k].y = (frames.atf(3 * p1 + k) - yh[k]) - yl[k];
      } else {
        d[r][k].x = __double2float_rn(frames.at(3 * p + k) - yb[k]);  // decoded sample in fp64
        d[r][k].y = __double2float_rn(frames.at(3 * p1 + k) - yb[k]);
      }
    }
    a0[r] = a1[r] = a2[r] = make_float2(0.f, 0.f);
    vmin[r][0] = vmin[r][1] = 3.0e38f;
  }
  // the per-band constants are pre-duplicated float2s in DevOps (FFMA2 operands)
  auto spec = [&](int l, float sh, int r) {
    return __ffma2_rn(ops.solve_f2[l][2], d[r][2],
                      __ffma2_rn(ops.solve_f2[l][1], d[r][1], __ffma2_rn(ops.solve_f2[l][0], d[r][0], make_float2(sh, sh))));
  };
  auto fit = [&](int l, float2 s, int r) {
    const float2 lg = make_float2(lg2_approx(s.x), lg2_approx(s.y));
    a0[r] = __ffma2_rn(ops.fitl2_f2[0][l], lg, a0[r]);
    a1[r] = __ffma2_rn(ops.fitl2_f2[1][l], lg, a1[r]);
    if constexpr (PLANES) a2[r] = __ffma2_rn(ops.fitl2_f2[2][l], lg, a2[r]);
  };
  const float* sp = Shi + bidx * Lp;
  if constexpr (KL > 0 && KL % 2 == 0) {
    const float4* sp4 = reinterpret_cast<const float4*>(sp);
#pragma unroll
    for (int qq = 0; qq < (KL + 3) / 4; ++qq) {
      const float4 v = ldg(sp4 + qq);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int h = 0; h < 4; h += 2) {
        const int l = 4 * qq + h;
        if (l < KL) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float2 s0 = spec(l, vv[h], r);
            const float2 s1 = spec(l + 1, vv[h + 1], r);
            vmin[r][0] = fminf(vmin[r][0], fminf(s0.x, s1.x));
            vmin[r][1] = fminf(vmin[r][1], fminf(s0.y, s1.y));
            fit(l, s0, r);
            fit(l + 1, s1, r);
          }
        }
      }
    }
  } else {
#pragma unroll(KL > 0 ? LM : 1)
    for (int l = 0; l < LM; ++l) {
      if (KL == 0 && l >= L) break;
      const float sh = ldg(sp + l);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const float2 s0 = spec(l, sh, r);
        vmin[r][0] = fminf(vmin[r][0], s0.x);
        vmin[r][1] = fminf(vmin[r][1], s0.y);
        fit(l, s0, r);
      }
    }
  }
  const float cal = (float)g.cal;
  const float thr = (float)ops.fallback_below;
  unsigned fbmask = 0;  // bit 2r + c: pixel (row r, column c) takes the fp64 fallback
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t p = (f * g.H + row0 + r) * g.W + col;
    if (live && r < nrow) {
      const float2 xo = make_float2(a0[r].x * cal, a0[r].y * cal), xd = make_float2(a1[r].x * cal, a1[r].y * cal);
      const float2 co = make_float2(fmaxf(xo.x, 0.f), fmaxf(xo.y, 0.f));
      const float2 t = make_float2(co.x + fmaxf(xd.x, 0.f), co.y + fmaxf(xd.y, 0.f));
      const float2 so = make_float2(t.x > 0.f ? __fdividef(co.x, t.x) : qnan_f(), t.y > 0.f ? __fdividef(co.y, t.y) : qnan_f());
      if (two && (p & 1) == 0) {  // 8-byte aligned pair
        *reinterpret_cast<float2*>(thb + p) = t;
        *reinterpret_cast<float2*>(so2 + p) = so;
      } else {
        thb[p] = t.x;
        so2[p] = so.x;
        if (two) {
          thb[p + 1] = t.y;
          so2[p + 1] = so.y;
        }
      }
      if constexpr (PLANES) {
        hbo[p] = xo.x;
        hb[p] = xd.x;
        off[p] = a2[r].x;
        if (two) {
          hbo[p + 1] = xo.y;
          hb[p + 1] = xd.y;
          off[p + 1] = a2[r].y;
        }
      }
      // fminf drops NaN operands, so a NaN band (non-finite input: flagged by the
      // low-pass kernel, and launch() callers must check the flags) is caught
      // through the fit sums it poisons instead
      if (!(vmin[r][0] >= thr) || isnan(a0[r].x + a1[r].x)) fbmask |= 1u << (2 * r);
      if (two && (!(vmin[r][1] >= thr) || isnan(a0[r].y + a1[r].y))) fbmask |= 2u << (2 * r);
    }
  }
  // Cancellation guard: pixels with a band below fallback_below (~0.4% of
  // textured pixels, but spread so that about half of all warps hold one or
  // two) are recomputed in fp64 right here by their warp, one pixel per pass:
  // lane l takes band l (the block spectrum, the reference's eps clamp, a
  // table log) and the three fit sums are reduced with xor shuffles (every
  // lane ends with the same bits).  The pixel's rgb, ybar and spectrum rows
  // were just read by this warp, so they come from L1, not DRAM; the
  // operators' band rows come from a 64-byte-per-band device copy, loaded
  // once per warp.  With the EM precision schedule (fb.classify) a pixel with
  // a band in [eps / 2, exact_below) is "sensitive" to the schedule's ~1e-8
  // spectrum deviation (see px_fallback_kernel): it is listed for the
  // deferred pass and its block for the all-fp64 exact pass instead.  Without
  // the schedule the spectrum is hi + lo (fp64 to 48 bits) and every pixel is
  // finished here.  (Band counts above 32 take each lane's extra bands from
  // the same rows.)
  if (__any_sync(0xffffffffu, fbmask != 0)) {
    const int lane = threadIdx.x & 31;
    unsigned mask = fbmask;
    if (fb.queued) {
      const unsigned nq = __reduce_add_sync(0xffffffffu, __popc(mask));
      if (lane == 0) atomicAdd(fb.queued, nq);
    }
    __syncwarp();  // every lane's fp32 map stores land before the fp64 rewrites below
    const double2* rows = reinterpret_cast<const double2*>(ops.band_rows);  // 4 double2 per band
    double2 r01 = make_double2(0.0, 0.0), r23 = r01, r45 = r01;
    if (lane < L) {
      r01 = ldg(rows + 4 * lane);
      r23 = ldg(rows + 4 * lane + 1);
      r45 = ldg(rows + 4 * lane + 2);
    }
    const double lo_b = 0.5 * ops.eps, hi_b = ops.exact_below, eps = ops.eps;
    const double2* logt = log_table_global();
    const uint32_t W32 = (uint32_t)g.W, prow = (uint32_t)(f * g.H + row0), col32 = (uint32_t)col;
    const uint32_t frow = (uint32_t)((f * g.hL + by) * g.wL);
    for (;;) {
      const unsigned m = __ballot_sync(0xffffffffu, mask != 0);
      if (!m) break;
      const int owner = __ffs(m) - 1;
      const int bit = __shfl_sync(0xffffffffu, mask ? __ffs(mask) - 1 : 0, owner);
      if (lane == owner) mask &= mask - 1;
      const uint32_t ocol = __shfl_sync(0xffffffffu, col32, owner) + (uint32_t)(bit & 1);
      const uint32_t p = (prow + (uint32_t)(bit >> 1)) * W32 + ocol;
      const uint32_t ob = frow + (ocol >> g.n);
      const double D0 = frames.at(3 * (int64_t)p) - ybar[ob];
      const double D1 = frames.at(3 * (int64_t)p + 1) - ybar[g.nll + ob];
      const double D2 = frames.at(3 * (int64_t)p + 2) - ybar[2 * g.nll + ob];
      double a0s = 0.0, a1s = 0.0, a2s = 0.0;
      bool sens = false;
      for (int l = lane; l < L; l += 32) {
        double2 q01 = r01, q23 = r23, q45 = r45;
        if (l >= 32) {
          q01 = ldg(rows + 4 * l);
          q23 = ldg(rows + 4 * l + 1);
          q45 = ldg(rows + 4 * l + 2);
        }
        double S = (double)ldg(Shi + (int64_t)ob * Lp + l);
        if (!fb.classify) S += (double)ldg(Slo + (int64_t)ob * Lp + l);
        const double sp = fma(q23.x, D2, fma(q01.y, D1, fma(q01.x, D0, S)));
        sens |= fb.classify && sp >= lo_b && sp < hi_b;
        const double lg = log_tab(fmax(sp, eps), logt);
        a0s = fma(q23.y, lg, a0s);
        a1s = fma(q45.x, lg, a1s);
        a2s = fma(q45.y, lg, a2s);
      }
      if (__any_sync(0xffffffffu, sens)) {  // defer: the exact pass re-estimates its block all-fp64
        if (lane == owner) {
          fb.list[atomicAdd(fb.count, 1u)] = p;
          unsigned* word = reinterpret_cast<unsigned*>(fb.blkflag + (ob & ~3u));
          const unsigned bitm = 1u << (8 * (ob & 3u));
          if (!(atomicOr(word, bitm) & bitm)) fb.blk_list[atomicAdd(fb.blk_count, 1u)] = ob;
        }
        continue;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        a0s += __shfl_xor_sync(0xffffffffu, a0s, o);
        a1s += __shfl_xor_sync(0xffffffffu, a1s, o);
        a2s += __shfl_xor_sync(0xffffffffu, a2s, o);
      }
      if (lane == owner) {
        const float xo = (float)(-a0s * g.cal), xd = (float)(-a1s * g.cal);
        const float co = fmaxf(xo, 0.f);
        const float t = co + fmaxf(xd, 0.f);
        thb[p] = t;
        so2[p] = t > 0.f ? __fdividef(co, t) : qnan_f();
        if constexpr (PLANES) {
          hbo[p] = xo;
          hb[p] = xd;
          off[p] = (float)(-a2s);
        }
      }
    }
  }
}

// fp64 recompute of the deferred pixels -- the "sensitive" fallback pixels
// px_f32_kernel listed -- after the exact pass has re-estimated their blocks
// all-fp64 (hi + lo spectrum parts).  With the EM's fp32 lead-in the block
// spectra differ from the all-fp64 ones by ~1e-8 relative, and a fallback
// pixel amplifies that by |S| / s_l through log s_l for every band
// s_l = S_l + solve (rgb - ybar) that is small but not clamped; bands below
// eps / 2 are clamped to eps either way, so only pixels with a band in
// [eps / 2, exact_below) wait for the exact pass (~15% of textured fallback
// pixels).  kFbLanes (2) threads per pixel, each taking every kFbLanes-th
// band, partial fit sums reduced with shuffles; grid-stride over the
// device-side count; table log (~1 ulp) after the reference's eps clamp.
// Operators are staged in shared memory by CTAs that have work (the per-lane
// band index would serialise constant-bank reads).  Every pixel is written
// exactly once after the exact pass, from spectra no kernel modifies any
// more: the output does not depend on scheduling.
#ifndef OXM_FB_LANES
#define OXM_FB_LANES 2
#endif
constexpr int kFbLanes = OXM_FB_LANES;  // threads per deferred pixel (1, 2 or 4)
#ifndef OXM_FB_CTAS_PER_SM
#define OXM_FB_CTAS_PER_SM 32
#endif
template <int KL, typename Src>
__global__ void __launch_bounds__(kFbThreads) px_fallback_kernel(const __grid_constant__ DevOps ops,
                                                                 const Src frames, PxGeom g,
                                                                 const float* __restrict__ Shi,
                                                                 const float* __restrict__ Slo, int Lp,
                                                                 const double* __restrict__ ybar,
                                                                 const uint32_t* __restrict__ fb_count,
                                                                 const uint32_t* __restrict__ fb_list,
                                                                 float* __restrict__ thb, float* __restrict__ so2,
                                                                 float* __restrict__ hbo, float* __restrict__ hb,
                                                                 float* __restrict__ off) {
  __shared__ double T[kMaxBands][3], F[3][kMaxBands];
  constexpr int kPerCta = kFbThreads / kFbLanes;
  const uint32_t cnt = *fb_count;
  if ((int64_t)blockIdx.x * kPerCta >= cnt) return;  // whole CTA idle: skip the staging
  const int64_t stride = (int64_t)gridDim.x * kPerCta;
  const int L = ops.L;
  for (int q = threadIdx.x; q < 3 * L; q += kFbThreads) {
    T[q / 3][q % 3] = ops.solve[q / 3][q % 3];
    F[q / L][q % L] = ops.fitm[q / L][q % L];
  }
  __syncthreads();
  const int sub = threadIdx.x & (kFbLanes - 1);
  // pixel indices are < 2^32 (checked at launch): 32-bit index arithmetic
  const uint32_t plane = (uint32_t)(g.H * g.W), W = (uint32_t)g.W;
  const double2* logt = log_table_global();
  // group collectives use the group's own lanes: other groups of the warp may
  // have left the loop
  const unsigned grp = ((1u << kFbLanes) - 1u) << ((threadIdx.x & 31) & ~(kFbLanes - 1));
  for (int64_t i = (int64_t)blockIdx.x * kPerCta + threadIdx.x / kFbLanes; i < cnt; i += stride) {
    const uint32_t p = fb_list[i];
    const uint32_t f = p / plane;
    const uint32_t rem = p - f * plane;
    const uint32_t row = rem / W, col = rem - row * W;
    const int64_t bidx = ((int64_t)f * g.hL + (row >> g.n)) * g.wL + (col >> g.n);
    const double D0 = frames.at(3 * (int64_t)p) - ybar[bidx];
    const double D1 = frames.at(3 * (int64_t)p + 1) - ybar[g.nll + bidx];
    const double D2 = frames.at(3 * (int64_t)p + 2) - ybar[2 * g.nll + bidx];
    const float* hi = Shi + bidx * Lp;
    const float* lo = Slo + bidx * Lp;
    constexpr int kPer = (BandCount<KL>::kMax + kFbLanes - 1) / kFbLanes;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int l = sub + kFbLanes * k;
      if (l < L) {
        const double S = (double)ldg(hi + l) + (double)ldg(lo + l);
        const double sp = fma(T[l][2], D2, fma(T[l][1], D1, fma(T[l][0], D0, S)));
        const double lg = log_tab(fmax(sp, ops.eps), logt);
        a0 = fma(F[0][l], lg, a0);
        a1 = fma(F[1][l], lg, a1);
        a2 = fma(F[2][l], lg, a2);
      }
    }
#pragma unroll
    for (int o = 1; o < kFbLanes; o <<= 1) {
      a0 += __shfl_xor_sync(grp, a0, o);
      a1 += __shfl_xor_sync(grp, a1, o);
      a2 += __shfl_xor_sync(grp, a2, o);
    }
    if (sub == 0) {
      const float xo = (float)(-a0 * g.cal), xd = (float)(-a1 * g.cal);
      const float co = fmaxf(xo, 0.f);
      const float t = co + fmaxf(xd, 0.f);
      thb[p] = t;
      so2[p] = t > 0.f ? __fdividef(co, t) : qnan_f();
      if (hbo) {
        hbo[p] = xo;
        hb[p] = xd;
        off[p] = (float)(-a2);
      }
    }
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
  pixel_fit_f64<KL>(
      ops, [&](int l) { return S[(int64_t)l * g.nll + bidx]; }, D0, D1, D2, x0, x1, x2,
      [&](int l, double s) {
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

// Workspace (256-B aligned sections):
//   ybar  3 x nll  double
//   spectra  fp64 SoA S[l][i] (fp64 path), or fp32 Shi[i][Lp] then Slo[i][Lp]
//            (fp32 path; Lp = L rounded up to 4 for 16-byte row loads)
//   x_init   3 x nll double (fit #1),  fit counts  nll int32   (EM bookkeeping)
//   fallback counter + EM chunk counter (256 B), fallback list (batch*H*W uint32)   [fp32 path]
struct Workspace {
  double* ybar;
  double* S;
  float* Shi;
  float* Slo;
  int Lp;
  double* xinit;
  int32_t* fits;
  int32_t* fits_out;              // the fit counts the EM writes: the caller's array, or `fits`
  float* xh;                      // EM hand-over state of the fp32 lead-in, [3][nll]
  uint32_t* fb_count;
  unsigned long long* em_work;    // EM chunk counter (same 256-byte block as fb_count)
  unsigned long long* lead_work;  // lead-in chunk counter (same block)
  unsigned long long* em_stats;   // [3] EM work counters (same block, EmIO::stats)
  unsigned long long* sel_work;   // chunk counter of the exact-block EM pass (same block)
  uint32_t* blk_count;            // number of exact blocks (same block)
  uint32_t* queued;               // pixels that took the fp64 fallback (same block)
  uint8_t* blk_flag;              // [nll] block marked for the exact pass (zeroed by ll_kernel)
  uint32_t* blk_list;             // [nll] marked blocks
  uint32_t* fb_list;
};

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

inline int padded_bands(int L) { return (L + 3) & ~3; }

size_t workspace_bytes(int L, int64_t nll, int64_t npx) {
  return 256 + align256(sizeof(double) * 3 * (size_t)nll) +
         align256(sizeof(double) * (size_t)padded_bands(L) * (size_t)nll) +
         align256(sizeof(double) * 3 * (size_t)nll) + align256(sizeof(int32_t) * (size_t)nll) +
         align256(sizeof(float) * 3 * (size_t)nll) + align256((size_t)nll) + align256(sizeof(uint32_t) * (size_t)nll) +
         256 + align256(sizeof(uint32_t) * (size_t)npx);
}

Workspace carve(void* ws, int L, int64_t nll) {
  uintptr_t p = (reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255);
  Workspace w;
  w.ybar = reinterpret_cast<double*>(p);
  p += align256(sizeof(double) * 3 * (size_t)nll);
  w.S = reinterpret_cast<double*>(p);
  w.Lp = padded_bands(L);
  w.Shi = reinterpret_cast<float*>(p);
  w.Slo = w.Shi + (size_t)w.Lp * (size_t)nll;
  p += align256(sizeof(double) * (size_t)w.Lp * (size_t)nll);
  w.xinit = reinterpret_cast<double*>(p);
  p += align256(sizeof(double) * 3 * (size_t)nll);
  w.fits = reinterpret_cast<int32_t*>(p);
  w.fits_out = w.fits;
  p += align256(sizeof(int32_t) * (size_t)nll);
  w.xh = reinterpret_cast<float*>(p);
  p += align256(sizeof(float) * 3 * (size_t)nll);
  w.blk_flag = reinterpret_cast<uint8_t*>(p);
  p += align256((size_t)nll);
  w.blk_list = reinterpret_cast<uint32_t*>(p);
  p += align256(sizeof(uint32_t) * (size_t)nll);
  w.fb_count = reinterpret_cast<uint32_t*>(p);
  w.em_work = reinterpret_cast<unsigned long long*>(p + 128);
  w.lead_work = reinterpret_cast<unsigned long long*>(p + 192);
  w.em_stats = reinterpret_cast<unsigned long long*>(p + 8);
  w.blk_count = reinterpret_cast<uint32_t*>(p + 4);
  w.queued = reinterpret_cast<uint32_t*>(p + 32);
  w.sel_work = reinterpret_cast<unsigned long long*>(p + 200);
  w.fb_list = reinterpret_cast<uint32_t*>(p + 256);
  return w;
}

// zeroes the fallback counter as part of the low-pass launch (no memset node)
template <typename Src, bool OUT_YBAR>
void launch_ll_pass(const DevOps& ops, const Src& src, int64_t batch, const LevelDims& d, int nlv, double* out,
                    int64_t count, int scale_exp, uint32_t* flags, double* xinit, uint8_t* blkflag, cudaStream_t s) {
  const unsigned grid = grid_1d(count, kLlThreads);
  switch (nlv) {
    case 1: ll_kernel<Src, 1, OUT_YBAR><<<grid, kLlThreads, 0, s>>>(ops, src, batch, d, out, count, scale_exp, flags, xinit, blkflag); break;
    case 2: ll_kernel<Src, 2, OUT_YBAR><<<grid, kLlThreads, 0, s>>>(ops, src, batch, d, out, count, scale_exp, flags, xinit, blkflag); break;
    default: ll_kernel<Src, 3, OUT_YBAR><<<grid, kLlThreads, 0, s>>>(ops, src, batch, d, out, count, scale_exp, flags, xinit, blkflag); break;
  }
}

// LL chain: one launch for n <= 3; for deeper pyramids, 3-level passes through
// fp64 HWC intermediate planes (stream-ordered scratch), the last one writing
// ybar.  The add order per level is the reference's in every pass.
template <typename Src>
int launch_ll(const DevOps& ops, const Src& frames, int64_t batch, const LevelDims& d, double* ybar, int64_t nll,
              uint32_t* flags, double* xinit, uint8_t* blkflag, cudaStream_t s) {
  const int n = d.n;
  if constexpr (std::is_same<Src, PlainSrc<float>>::value) {
    if (n <= 3 && launch_ll_tma(ops, frames.p, batch, d, ybar, nll, flags, xinit, blkflag, s))
      return check_launch("hybrid_ll_tma");
  }
  if (n <= 3) {
    launch_ll_pass<Src, true>(ops, frames, batch, d, n, ybar, nll, n, flags, xinit, blkflag, s);
    return check_launch("hybrid_ll");
  }
  double* prev = nullptr;
  int done = 0;
  int st = OXM_OK;
  while (done < n) {
    const int nl = n - done > 3 ? 3 : n - done;
    LevelDims dp{};
    dp.n = nl;
    for (int k = 0; k <= nl; ++k) {
      dp.h[k] = d.h[done + k];
      dp.w[k] = d.w[done + k];
    }
    const bool last = done + nl == n;
    const int64_t count = batch * dp.h[nl] * dp.w[nl];
    double* next = nullptr;
    if (!last) {
      cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&next), sizeof(double) * 3 * (size_t)count, s);
      if (err != cudaSuccess) {
        set_last_error("hybrid_ll scratch", err);
        st = OXM_ERR_CUDA;
        break;
      }
    }
    if (done == 0)
      launch_ll_pass<Src, false>(ops, frames, batch, dp, nl, next, count, 0, flags, nullptr, nullptr, s);
    else if (last)
      launch_ll_pass<PlainSrc<double>, true>(ops, PlainSrc<double>{prev}, batch, dp, nl, ybar, count, n, flags, xinit, blkflag, s);
    else
      launch_ll_pass<PlainSrc<double>, false>(ops, PlainSrc<double>{prev}, batch, dp, nl, next, count, 0, flags, nullptr, nullptr, s);
    st = check_launch("hybrid_ll");
    if (prev) cudaFreeAsync(prev, s);
    prev = next;
    if (st) break;
    done += nl;
  }
  if (prev) cudaFreeAsync(prev, s);
  return st;
}

inline bool em_lead_active(const DevOps& ops) { return ops.L == 26 && ops.lead_thr_f > 0.0f && ops.max_iters > 2; }
inline bool exact_blocks_active(const DevOps& ops) { return em_lead_active(ops) && ops.exact_below > 0.0; }

template <bool F32OUT>
int launch_em_soa(const DevOps& ops, const double* ybar, int64_t nll, const Workspace& w, int32_t* fits,
                  cudaStream_t s, int reserve = 0, cudaEvent_t split = nullptr) {
  EmIO io{};
  io.em_reserve = reserve;
  io.y = ybar;
  io.y_soa = 1;
  io.n = nll;
  if (F32OUT) {
    io.Shi = w.Shi;
    io.Slo = w.Slo;
    io.Lp = w.Lp;
  } else {
    io.S = w.S;
  }
  io.xinit = w.xinit;
  io.xinit_ready = 1;  // computed by the low-pass kernel
  io.fits = fits ? fits : w.fits;
  io.work = w.em_work;  // zeroed by zero_counters
  if (F32OUT) {  // fp32 lead-in + fp64 tail (the fp64 API path stays all-fp64)
    io.xh = w.xh;
    io.lead_work = w.lead_work;
    io.stats = w.em_stats;
    // with the exact-block pass, only its blocks' lo parts are ever read
    if (exact_blocks_active(ops)) io.Slo = nullptr;
  }
  constexpr SpecOut out = F32OUT ? SpecOut::kAosF32HiLo : SpecOut::kSoaF64;
  if (ops.L == 26) return launch_em<26, out>(ops, io, s, split);
  return launch_em<0, out>(ops, io, s, split);
}

template <int KL, bool PLANES, typename Src>
void launch_px_rows(const DevOps& ops, const Src& frames, const PxGeom& g, dim3 grid, int R, const Workspace& w,
                    float* thb, float* so2, float* hbo, float* hb, float* off, const FbOut& fb, cudaStream_t s) {
  if (R == 2)
    px_f32_kernel<KL, 2, PLANES, Src><<<grid, kPxThreads, 0, s>>>(ops, frames, g, w.Shi, w.Slo, w.Lp, w.ybar, thb, so2, hbo, hb, off, fb);
  else
    px_f32_kernel<KL, 4, PLANES, Src><<<grid, kPxThreads, 0, s>>>(ops, frames, g, w.Shi, w.Slo, w.Lp, w.ybar, thb, so2, hbo, hb, off, fb);
}

template <int KL, typename Src>
int launch_px_f32(const DevOps& ops, const Src& frames, const PxGeom& g, int64_t batch, const Workspace& w,
                  float* thb, float* so2, float* hbo, float* hb, float* off, cudaStream_t s,
                  cudaEvent_t fixup_ev = nullptr) {
  if (!thb || !so2) return OXM_ERR_ARGUMENT;
  // the planes are written all three or none
  const bool planes = hbo || hb || off;
  if (planes && !(hbo && hb && off)) return OXM_ERR_ARGUMENT;
  const int bs = 1 << g.n;
#ifndef OXM_PX_ROWS
#define OXM_PX_ROWS 4
#endif
  const int R = bs >= OXM_PX_ROWS ? OXM_PX_ROWS : bs;
  const int64_t cpb = bs > R ? bs / R : 1;
  dim3 grid((unsigned)ceil_div(g.W, 2 * kPxThreads), (unsigned)(g.hL * cpb), (unsigned)batch);
  if (g.hL * cpb > 65535 || batch > 65535) return OXM_ERR_ARGUMENT;
  const bool classify = exact_blocks_active(ops);
  const FbOut fb{w.fb_count, w.fb_list, w.blk_flag, w.blk_list, w.blk_count, w.queued, classify ? 1 : 0};
  if (planes)
    launch_px_rows<KL, true>(ops, frames, g, grid, R, w, thb, so2, hbo, hb, off, fb, s);
  else
    launch_px_rows<KL, false>(ops, frames, g, grid, R, w, thb, so2, hbo, hb, off, fb, s);
  int st = check_launch("hybrid_px_f32");
  if (st) return st;
  if (fixup_ev) cudaEventRecord(fixup_ev, s);
  if (!classify) return OXM_OK;  // every fallback pixel was finished by px_f32_kernel
  EmIO io{};
  io.y = w.ybar;
  io.y_soa = 1;
  io.n = g.nll;
  io.Shi = w.Shi;
  io.Slo = w.Slo;
  io.Lp = w.Lp;
  io.xinit = w.xinit;
  io.xinit_ready = 1;
  io.fits = w.fits_out;
  io.work = w.sel_work;
  io.sel = w.blk_list;
  io.sel_count = w.blk_count;
  if ((st = launch_em_selected<26, SpecOut::kAosF32HiLo>(ops, io, s))) return st;
  const unsigned fb_grid = (unsigned)device_sms() * OXM_FB_CTAS_PER_SM;
  px_fallback_kernel<KL, Src><<<fb_grid, kFbThreads, 0, s>>>(ops, frames, g, w.Shi, w.Slo, w.Lp, w.ybar, w.fb_count,
                                                             w.fb_list, thb, so2, hbo, hb, off);
  return check_launch("hybrid_fallback");
}

inline cudaEvent_t as_event(void* e) { return reinterpret_cast<cudaEvent_t>(e); }

inline void mark(void* const* ev, int i, cudaStream_t s) {
  if (ev && ev[i]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[i]), s);
}

int hybrid_prologue(const oxm_ctx* ctx, const void* frames, int64_t batch, int64_t H, int64_t W, int n,
                    void* ws, size_t ws_bytes, LevelDims& d, int64_t& nll, Workspace& w) {
  if (!ctx || batch < 0 || (batch > 0 && !frames)) return OXM_ERR_ARGUMENT;
  if (n < 1 || n > kMaxLevels) return OXM_ERR_ARGUMENT;
  // pipeline.py:177-181: frame must be at least 2^n in both dimensions
  if (H < ((int64_t)1 << n) || W < ((int64_t)1 << n)) return OXM_ERR_ARGUMENT;
  int st = level_dims(H, W, n, d);
  if (st) return st;
  nll = batch * d.h[n] * d.w[n];
  const int L = ctx->ops.L;
  if (batch == 0) return OXM_OK;
  if (!ws || ws_bytes < workspace_bytes(L, nll, batch * H * W)) return OXM_ERR_WORKSPACE;
  w = carve(ws, L, nll);
  return OXM_OK;
}

// fallback + EM chunk counter reset, ordered before the low-pass kernel
__global__ void zero_counters(uint32_t* fb, unsigned long long* em, unsigned long long* lead,
                              unsigned long long* stats, unsigned long long* sel, uint32_t* blk, uint32_t* queued) {
  *fb = 0u;
  *em = 0ull;
  *lead = 0ull;
  stats[0] = stats[1] = stats[2] = 0ull;
  *sel = 0ull;
  *blk = 0u;
  *queued = 0u;
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_hybrid_em_counters(const oxm_ctx* ctx, void* workspace, int64_t batch, int64_t height,
                                      int64_t width, int n_levels, uint64_t* out, void* stream) {
  LevelDims d;
  if (!ctx || !workspace || !out || level_dims(height, width, n_levels, d) != OXM_OK || batch < 0)
    return OXM_ERR_ARGUMENT;
  const Workspace w = carve(workspace, ctx->ops.L, batch * d.h[n_levels] * d.w[n_levels]);
  DeviceGuard dg(ctx->device);
  cudaStream_t s = as_stream(stream);
  uint32_t blk = 0, queued = 0, deferred = 0;
  cudaError_t err = cudaMemcpyAsync(out, w.em_stats, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (err == cudaSuccess) err = cudaMemcpyAsync(&blk, w.blk_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (err == cudaSuccess) err = cudaMemcpyAsync(&queued, w.queued, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (err == cudaSuccess) err = cudaMemcpyAsync(&deferred, w.fb_count, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (err == cudaSuccess) err = cudaStreamSynchronize(s);
  out[3] = blk;
  out[4] = queued;
  out[5] = deferred;
  if (err != cudaSuccess) {
    set_last_error("oxm_hybrid_em_counters", err);
    return OXM_ERR_CUDA;
  }
  return OXM_OK;
}

extern "C" size_t oxm_hybrid_workspace_bytes(const oxm_ctx* ctx, int64_t batch, int64_t height, int64_t width,
                                             int n_levels) {
  LevelDims d;
  if (!ctx || level_dims(height, width, n_levels, d) != OXM_OK || batch < 0) return 0;
  return workspace_bytes(ctx->ops.L, batch * d.h[n_levels] * d.w[n_levels], batch * height * width);
}

namespace oxm {
namespace {
template <typename Src>
int hybrid_maps(const oxm_ctx* ctx, const void* raw, const Src& src, int64_t batch, int64_t height, int64_t width,
                int n_levels, double calibration, void* workspace, size_t workspace_bytes_, float* thb, float* so2,
                float* hbo, float* hb, float* offset, int32_t* fits, uint32_t* flags, void* stream,
                void* const* ev, void* stream_px = nullptr, int reserve = 0) {
  LevelDims d;
  int64_t nll;
  Workspace w;
  int st = hybrid_prologue(ctx, raw, batch, height, width, n_levels, workspace, workspace_bytes_, d, nll, w);
  if (st) return st;
  if (batch == 0) return OXM_OK;
  // the fallback list and its kernel use 32-bit pixel indices
  if (batch * height * width >= ((int64_t)1 << 32)) return OXM_ERR_ARGUMENT;
  DeviceGuard dg(ctx->device);
  cudaStream_t s = as_stream(stream);
  mark(ev, 0, s);
  zero_counters<<<1, 1, 0, s>>>(w.fb_count, w.em_work, w.lead_work, w.em_stats, w.sel_work, w.blk_count, w.queued);
  if ((st = launch_ll(ctx->ops, src, batch, d, w.ybar, nll, flags, w.xinit, w.blk_flag, s))) return st;
  mark(ev, 1, s);
  if (fits) w.fits_out = fits;
  if ((st = launch_em_soa<true>(ctx->ops, w.ybar, nll, w, fits, s, reserve,
                                ev ? as_event(ev[2]) : nullptr)))
    return st;
  mark(ev, 3, s);
  if (stream_px) {  // split launch: the per-pixel stage runs on its own stream after the EM
    cudaEvent_t em_done = nullptr;
    cudaError_t err = cudaEventCreateWithFlags(&em_done, cudaEventDisableTiming);
    if (err == cudaSuccess) err = cudaEventRecord(em_done, s);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(as_stream(stream_px), em_done, 0);
    if (em_done) cudaEventDestroy(em_done);  // released once it has completed
    if (err != cudaSuccess) {
      set_last_error("split launch event", err);
      return OXM_ERR_CUDA;
    }
    s = as_stream(stream_px);
  }
  PxGeom g{height, width, d.h[n_levels], d.w[n_levels], nll, n_levels, calibration};
  if (ctx->ops.L == 26)
    st = launch_px_f32<26>(ctx->ops, src, g, batch, w, thb, so2, hbo, hb, offset, s, ev ? as_event(ev[4]) : nullptr);
  else
    st = launch_px_f32<0>(ctx->ops, src, g, batch, w, thb, so2, hbo, hb, offset, s, ev ? as_event(ev[4]) : nullptr);
  mark(ev, 5, s);
  return st;
}
}  // namespace
}  // namespace oxm

extern "C" int oxm_hybrid_maps_f32(const oxm_ctx* ctx, const float* frames, int64_t batch, int64_t height,
                                   int64_t width, int n_levels, double calibration, void* workspace,
                                   size_t workspace_bytes_, float* thb, float* so2, float* hbo, float* hb,
                                   float* offset, int32_t* fits, uint32_t* flags, void* stream,
                                   void* const* ev) {
  return hybrid_maps(ctx, frames, PlainSrc<float>{frames}, batch, height, width, n_levels, calibration, workspace,
                     workspace_bytes_, thb, so2, hbo, hb, offset, fits, flags, stream, ev);
}

extern "C" int oxm_hybrid_maps_f32_split(const oxm_ctx* ctx, const float* frames, int64_t batch, int64_t height,
                                         int64_t width, int n_levels, double calibration, void* workspace,
                                         size_t workspace_bytes_, float* thb, float* so2, float* hbo, float* hb,
                                         float* offset, int32_t* fits, uint32_t* flags, void* stream_em,
                                         void* stream_px, int em_reserve) {
  if (!stream_px) return OXM_ERR_ARGUMENT;
  return hybrid_maps(ctx, frames, PlainSrc<float>{frames}, batch, height, width, n_levels, calibration, workspace,
                     workspace_bytes_, thb, so2, hbo, hb, offset, fits, flags, stream_em, nullptr, stream_px,
                     em_reserve);
}

extern "C" int oxm_hybrid_maps_u16(const oxm_ctx* ctx, const uint16_t* frames, int big_endian, double scale,
                                   int64_t batch, int64_t height, int64_t width, int n_levels, double calibration,
                                   void* workspace, size_t workspace_bytes_, float* thb, float* so2, float* hbo,
                                   float* hb, float* offset, int32_t* fits, uint32_t* flags, void* stream,
                                   void* const* ev) {
  if (!(scale > 0.0)) return OXM_ERR_DATA;  // io.py:101-102
  return hybrid_maps(ctx, frames, PpmSrc{frames, scale, big_endian}, batch, height, width, n_levels, calibration,
                     workspace, workspace_bytes_, thb, so2, hbo, hb, offset, fits, flags, stream, ev);
}

extern "C" int oxm_hybrid_frame_f64(const oxm_ctx* ctx, const double* frames, int64_t batch, int64_t height,
                                    int64_t width, int n_levels, double calibration, void* workspace,
                                    size_t workspace_bytes_, double* cube, double* hbo, double* hb, double* offset,
                                    int32_t* fits, uint32_t* flags, void* stream, void* const* ev) {
  LevelDims d;
  int64_t nll;
  Workspace w;
  int st = hybrid_prologue(ctx, frames, batch, height, width, n_levels, workspace, workspace_bytes_, d, nll, w);
  if (st) return st;
  if (batch == 0) return OXM_OK;
  DeviceGuard dg(ctx->device);
  cudaStream_t s = as_stream(stream);
  mark(ev, 0, s);
  zero_counters<<<1, 1, 0, s>>>(w.fb_count, w.em_work, w.lead_work, w.em_stats, w.sel_work, w.blk_count, w.queued);
  if ((st = launch_ll(ctx->ops, PlainSrc<double>{frames}, batch, d, w.ybar, nll, flags, w.xinit, nullptr, s))) return st;
  mark(ev, 1, s);
  mark(ev, 2, s);  // no fp32 lead-in on the fp64 path
  if ((st = launch_em_soa<false>(ctx->ops, w.ybar, nll, w, fits, s))) return st;
  mark(ev, 3, s);
  PxGeom g{height, width, d.h[n_levels], d.w[n_levels], nll, n_levels, calibration};
  const int64_t npx = batch * height * width;
  const double* S = w.S;
  if (ctx->ops.L == 26)
    px_f64_kernel<26><<<grid_1d(npx, 128), 128, 0, s>>>(ctx->ops, frames, g, batch, S, w.ybar, cube, hbo, hb, offset);
  else
    px_f64_kernel<0><<<grid_1d(npx, 128), 128, 0, s>>>(ctx->ops, frames, g, batch, S, w.ybar, cube, hbo, hb, offset);
  st = check_launch("hybrid_px_f64");
  mark(ev, 4, s);  // no separate fixup stage on the fp64 path
  mark(ev, 5, s);
  return st;
}
