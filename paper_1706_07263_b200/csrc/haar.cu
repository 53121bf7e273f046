// K1 / K2: fused multi-level 2D Haar forward and inverse (fp32 and fp64).
//
// Reference semantics: haar.py:24-33 (orthonormal 4x4 window matrix, window
// order TL,TR,BL,BR = a,b,c,d), haar.py:80-85 (per-level right/bottom edge
// replication of odd planes), haar.py:88-101 (lp,dh,dv,dd), haar.py:104-117
// (inverse butterflies + crop to orig_shape), haar.py:120-150 (recursion).
//
// Design: one thread owns one (coarsest-position, channel) column of the
// pyramid for a pass of up to 3 levels, i.e. a 2^NL x 2^NL pixel block of one
// channel, held entirely in registers.  The frame is read exactly once per
// pass and every coefficient written once; adjacent threads own adjacent
// channels / blocks so HWC loads and stores stay sector-contiguous per warp.
// Deeper pyramids chain passes through the coarsest low-pass plane (which
// the reference returns anyway).  The add order matches NumPy's left-to-right
// evaluation of `0.5 * (a + b - c - d)` so fp64 results are bit-identical.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "oxm_common.cuh"
#include "oxm_tma.cuh"

namespace oxm {
namespace {

constexpr int kMaxPass = 3;  // levels fused per pass

struct FwdGeom {
  int64_t C;
  int64_t h[kMaxPass + 1], w[kMaxPass + 1];  // [0] = source plane dims
  int64_t off[kMaxPass + 1][4];              // element offsets of lp,dh,dv,dd per level (1..NL)
};

// t -> (channel c, column J, row I) of the coarsest plane; 32-bit divisions
// whenever the index space fits (64-bit division is a ~70-instruction
// sequence, which made these streaming kernels issue-bound)
__device__ __forceinline__ void split_index(int64_t t, int64_t total, int64_t C, int64_t w, int64_t& c, int64_t& J,
                                            int64_t& I) {
  if (total <= 0xffffffffll) {
    const uint32_t tt = (uint32_t)t, CC = (uint32_t)C, ww = (uint32_t)w;
    const uint32_t rest = tt / CC;
    c = tt - rest * CC;
    const uint32_t Ii = rest / ww;
    J = rest - Ii * ww;
    I = Ii;
  } else {
    c = t % C;
    const int64_t rest = t / C;
    J = rest % w;
    I = rest / w;
  }
}


// IT: index type -- int32_t whenever the source plane and every output plane
// fit (the launcher checks), so the per-thread address math is 32-bit.
template <typename T, int NL, typename IT>
__global__ void __launch_bounds__(256) haar_fwd_kernel(const T* __restrict__ src, FwdGeom g,
                                                       T* __restrict__ out, uint32_t* flags) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t total = g.h[NL] * g.w[NL] * g.C;
  if (t >= total) return;
  int64_t c64, J64, I64;
  split_index(t, total, g.C, g.w[NL], c64, J64, I64);
  const IT C = (IT)g.C, c = (IT)c64, J = (IT)J64, I = (IT)I64;
  const IT H0 = (IT)g.h[0], W0 = (IT)g.w[0];
  constexpr int S0 = 1 << NL;

  T p[S0][S0];
  bool bad = false;
#pragma unroll
  for (int r = 0; r < S0; ++r) {
    const IT row = min(I * S0 + r, H0 - 1);
#pragma unroll
    for (int s = 0; s < S0; ++s) {
      const IT col = min(J * S0 + s, W0 - 1);
      const T v = ldg(src + (row * W0 + col) * C + c);
      bad |= !isfinite(v);
      p[r][s] = v;
    }
  }
  if (bad && flags) atomicOr(flags, OXM_FLAG_NONFINITE);

#pragma unroll
  for (int k = 0; k < NL; ++k) {
    const int Sk = S0 >> k;
    const int Sn = Sk >> 1;
    const IT br = I * Sk, bc = J * Sk;  // global position of p[0][0] at level k
    const IT hk = (IT)g.h[k], wk = (IT)g.w[k];
    const IT hn = (IT)g.h[k + 1], wn = (IT)g.w[k + 1];
    T* const o0 = out + g.off[k + 1][0];
    T* const o1 = out + g.off[k + 1][1];
    T* const o2 = out + g.off[k + 1][2];
    T* const o3 = out + g.off[k + 1][3];
#pragma unroll
    for (int i = 0; i < Sn; ++i) {
#pragma unroll
      for (int j = 0; j < Sn; ++j) {
        // edge replication: the odd partner row/col falls back to its twin
        const bool rowok = br + 2 * i + 1 < hk;
        const bool colok = bc + 2 * j + 1 < wk;
        const T a = p[2 * i][2 * j];
        const T b = colok ? p[2 * i][2 * j + 1] : a;
        const T cc = rowok ? p[2 * i + 1][2 * j] : a;
        const T d = rowok ? (colok ? p[2 * i + 1][2 * j + 1] : cc) : b;
        const T lp = T(0.5) * (((a + b) + cc) + d);
        const T dh = T(0.5) * (((a + b) - cc) - d);
        const T dv = T(0.5) * (((a - b) - cc) + d);
        const T dd = T(0.5) * (((a - b) + cc) - d);
        const IT gi = (br >> 1) + i, gj = (bc >> 1) + j;
        if (gi < hn && gj < wn) {
          const IT e = (gi * wn + gj) * C + c;
          o0[e] = lp;
          o1[e] = dh;
          o2[e] = dv;
          o3[e] = dd;
        }
        p[i][j] = lp;  // (i,j) <= (2i,2j): only already-consumed windows are overwritten
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 with TMA-staged 2D tiles in and out (3-channel HWC planes: RGB frames).
// Same per-thread work and the same arithmetic as haar_fwd_kernel
// (bit-identical outputs); only the data movement differs:
//   in:  the plane is a 2D tensor of h0 rows x 3 w0 elements; a CTA's tile of
//        TY x TX coarsest blocks (TY 2^NL rows x TX 2^NL pixels x 3 channels,
//        768-byte rows) arrives by one cp.async.bulk.tensor load;
//   out: every thread writes its coefficients into per-(level, plane) tiles
//        in shared memory and one elected thread stores them with 4 NL
//        cp.async.bulk.tensor stores (one tensor map per output plane; the
//        hardware clips the parts of edge tiles outside a plane).
// A persistent CTA walks tiles strided by gridDim; each thread copies its
// block's samples to registers first, so the input buffer is released (and
// the next tile's load issued) before the butterflies run.  Thread
// t = (ly TX + lx) 3 + c owns channel c of block (ly, lx).  Interior blocks
// read their samples at compile-time offsets, blocks at the right / bottom
// edge through clamped ones (the reference's replication, inside the tile).
#ifndef OXM_K1_STAGES
#define OXM_K1_STAGES 2
#endif
#ifndef OXM_K1_TY_DIV
#define OXM_K1_TY_DIV 2
#endif
template <typename T, int NL>
struct FwdTma {
  static constexpr int S = 1 << NL;
  static constexpr int TX = (sizeof(T) == 4 ? 64 : 32) / S;  // 768-byte input tile rows
  static constexpr int TY = NL == 3 ? 8 : 128 / OXM_K1_TY_DIV / TX;
  static constexpr int kStages = OXM_K1_STAGES;  // input tiles in flight per CTA
  static constexpr int kThreads = 3 * TX * TY;
  static constexpr int kRowE = TX * S * 3;
  static constexpr int kRows = TY * S;
  static constexpr int kTileE = kRowE * kRows;
  static constexpr uint32_t kTileBytes = kTileE * sizeof(T);
  // output tile of level k (1..NL): (kRows >> k) rows x (kRowE >> k) elements, 4 planes each
  __host__ __device__ static constexpr int out_elems(int k) { return (kRows >> k) * (kRowE >> k); }
  __host__ __device__ static constexpr int out_offset(int k, int q) {  // elements from the staging base
    int o = 0;
    for (int l = 1; l < k; ++l) o += 4 * out_elems(l);
    return o + q * out_elems(k);
  }
  static constexpr int kOutE = out_offset(NL + 1, 0);
  static constexpr size_t kSmem = sizeof(T) * (size_t)(kStages * kTileE + kOutE);
};

struct FwdMaps {
  CUtensorMap in;
  CUtensorMap out[kMaxPass][4];  // level k+1, plane q (lp, dh, dv, dd)
};

template <typename T, int NL>
__global__ void __launch_bounds__(FwdTma<T, NL>::kThreads) haar_fwd_tma_kernel(const __grid_constant__ FwdMaps maps,
                                                                             FwdGeom g, uint32_t* flags,
                                                                             int tiles_x, int tiles_y) {
  using G = FwdTma<T, NL>;
  constexpr int S0 = G::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* const tiles = reinterpret_cast<T*>(smem_raw);  // kStages input tiles
  T* const stage = tiles + G::kStages * G::kTileE;   // output staging
  __shared__ __align__(8) uint64_t bar[G::kStages];
  const int tid = threadIdx.x;
  const int ntiles = tiles_x * tiles_y;
  const int H0 = (int)g.h[0], W0 = (int)g.w[0];
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < G::kStages; ++b) mbar_init(&bar[b], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int t, int b) {
    if (t >= ntiles) return;
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    mbar_expect_tx(&bar[b], G::kTileBytes);
    tma_load_2d(tiles + b * G::kTileE, &maps.in, tx * G::kRowE, ty * G::kRows, &bar[b]);
  };
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < G::kStages; ++b) issue(blockIdx.x + b * gridDim.x, b);
  }
  const int c = tid % 3, blk = tid / 3;
  const int ly = blk / G::TX, lx = blk - ly * G::TX;
  bool bad = false;
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int ty = t / tiles_x, tx = t - ty * tiles_x;
    const int I = ty * G::TY + ly, J = tx * G::TX + lx;
    const int buf = it % G::kStages;
    mbar_wait(&bar[buf], (it / G::kStages) & 1);
    const T* tile = tiles + buf * G::kTileE;
    T p[S0][S0];
    if (I * S0 + S0 <= H0 && J * S0 + S0 <= W0) {
      const T* q = tile + (ly * S0) * G::kRowE + lx * S0 * 3 + c;
#pragma unroll
      for (int r = 0; r < S0; ++r)
#pragma unroll
        for (int u = 0; u < S0; ++u) p[r][u] = q[r * G::kRowE + 3 * u];
    } else {
      // clamped (edge) samples; blocks entirely past the plane read in-tile
      // garbage that only lands in clipped parts of the output boxes
      const int r0 = ty * G::kRows, c0 = tx * G::TX * S0;
#pragma unroll
      for (int r = 0; r < S0; ++r) {
        const int row = max(min(I * S0 + r, H0 - 1) - r0, 0);
#pragma unroll
        for (int u = 0; u < S0; ++u) p[r][u] = tile[row * G::kRowE + max(min(J * S0 + u, W0 - 1) - c0, 0) * 3 + c];
      }
    }
    if (tid == 0) tma_store_wait_read0();  // the previous tile's stores have read the staging tiles
    __syncthreads();                        // input buffer consumed, staging buffer free
    if (tid == 0) {
      fence_proxy_async();
      issue(t + G::kStages * gridDim.x, buf);
    }
    const bool valid = I < (int)g.h[NL] && J < (int)g.w[NL];
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const int Sk = S0 >> k;
      const int Sn = Sk >> 1;
      const int br = I * Sk, bc = J * Sk;  // global position of p[0][0] at level k
      const int hk = (int)g.h[k], wk = (int)g.w[k];
      const int orow = G::kRowE >> (k + 1);  // elements per staging row at level k+1
      T* const s0 = stage + G::out_offset(k + 1, 0) + (ly * Sn) * orow + lx * Sn * 3 + c;
      const int pl = G::out_elems(k + 1);
#pragma unroll
      for (int i = 0; i < Sn; ++i) {
#pragma unroll
        for (int j = 0; j < Sn; ++j) {
          const bool rowok = br + 2 * i + 1 < hk;
          const bool colok = bc + 2 * j + 1 < wk;
          const T a = p[2 * i][2 * j];
          const T b = colok ? p[2 * i][2 * j + 1] : a;
          const T cc = rowok ? p[2 * i + 1][2 * j] : a;
          const T d = rowok ? (colok ? p[2 * i + 1][2 * j + 1] : cc) : b;
          const T lp = T(0.5) * (((a + b) + cc) + d);
          const T dh = T(0.5) * (((a + b) - cc) - d);
          const T dv = T(0.5) * (((a - b) - cc) + d);
          const T dd = T(0.5) * (((a - b) + cc) - d);
          // level 1 sees every sample: its low-pass is finite iff its four inputs
          // are (an overflowing sum is re-checked sample by sample)
          if (k == 0 && valid && !isfinite(lp)) bad |= !(isfinite(a) && isfinite(b) && isfinite(cc) && isfinite(d));
          T* o = s0 + i * orow + 3 * j;
          o[0] = lp;
          o[pl] = dh;
          o[2 * pl] = dv;
          o[3 * pl] = dd;
          p[i][j] = lp;
        }
      }
    }
    fence_proxy_async();  // staging writes -> visible to the TMA stores
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int k = 1; k <= NL; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tma_store_2d(&maps.out[k - 1][q], stage + G::out_offset(k, q), (tx * G::kRowE) >> k, (ty * G::kRows) >> k);
      tma_store_commit();
    }
  }
  if (tid == 0) tma_store_wait_all();
  if (flags && __syncthreads_or(bad) && tid == 0) atomicOr(flags, OXM_FLAG_NONFINITE);
}

// OXM_HAAR_TMA=0 in the environment selects haar_fwd_kernel (A/B switch)
inline bool haar_tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("OXM_HAAR_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

// launches the TMA pass when the planes allow it (3 channels, 16-byte aligned
// rows and plane bases, 32-bit in-plane indices); false = not launched
// Host cost of a launch: encoding the 4 NL + 1 tensor maps and the launch
// configuration queries take longer than the 1080p kernel itself, so
// back-to-back calls would leave the GPU idle between frames.  Both are
// cached: the maps for the last kFwdMapCache (source, output, geometry) sets
// (a video loop reuses its buffers), the shared-memory attribute and the
// occupancy once per kernel instantiation and device.
constexpr int kFwdMapCache = 16;
struct FwdMapEntry {
  const void* src = nullptr;
  const void* out = nullptr;
  FwdGeom g{};
  int nl = 0, esz = 0;
  FwdMaps maps;
};

template <typename T, int NL>
bool fwd_maps(const T* src, const FwdGeom& g, T* out, FwdMaps& maps) {
  using G = FwdTma<T, NL>;
  static std::mutex mu;
  static FwdMapEntry cache[kFwdMapCache];
  static int victim = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (const FwdMapEntry& e : cache)
    if (e.src == src && e.out == out && e.nl == NL && e.esz == (int)sizeof(T) && !std::memcmp(&e.g, &g, sizeof(g))) {
      maps = e.maps;
      return true;
    }
  const bool f64 = sizeof(T) == 8;
  if (!make_tmap_2d(&maps.in, src, f64, (uint64_t)(3 * g.w[0]), (uint64_t)g.h[0], (uint64_t)(3 * g.w[0] * sizeof(T)),
                    G::kRowE, G::kRows))
    return false;
  for (int k = 1; k <= NL; ++k)
    for (int q = 0; q < 4; ++q)
      if (!make_tmap_2d(&maps.out[k - 1][q], out + g.off[k][q], f64, (uint64_t)(3 * g.w[k]), (uint64_t)g.h[k],
                        (uint64_t)(3 * g.w[k] * sizeof(T)), G::kRowE >> k, G::kRows >> k))
        return false;
  FwdMapEntry& e = cache[victim];
  victim = (victim + 1) % kFwdMapCache;
  e.src = src;
  e.out = out;
  e.g = g;
  e.nl = NL;
  e.esz = (int)sizeof(T);
  e.maps = maps;
  return true;
}

// resident CTAs per SM of haar_fwd_tma_kernel<T, NL>, setting its
// shared-memory attribute on first use per device; 0 = unusable.  (Templated
// on the instantiation, not on the kernel's pointer type, which every
// instantiation shares.)
template <typename T, int NL>
int fwd_tma_ctas_per_sm() {
  using G = FwdTma<T, NL>;
  auto kern = haar_fwd_tma_kernel<T, NL>;
  const int threads = G::kThreads;
  const size_t smem = G::kSmem;
  constexpr int kDevs = 64;
  static std::mutex mu;
  static int per_sm[kDevs] = {};  // 0 = not configured yet, -1 = failed
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) {
    cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (per_sm[dev] == 0) {
    int n = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = -1;
    }
    per_sm[dev] = n;
  }
  return per_sm[dev] > 0 ? per_sm[dev] : 0;
}

// launches the TMA pass when the planes allow it (3 channels, 16-byte aligned
// rows and plane bases, 32-bit in-plane indices); false = not launched
template <typename T, int NL>
bool launch_fwd_tma(const T* src, const FwdGeom& g, T* out, uint32_t* flags, cudaStream_t stream) {
  using G = FwdTma<T, NL>;
  if (!haar_tma_enabled() || g.C != 3) return false;
  if (g.h[0] * g.w[0] * 3 >= ((int64_t)1 << 31)) return false;
  auto kern = haar_fwd_tma_kernel<T, NL>;
  const int per_sm = fwd_tma_ctas_per_sm<T, NL>();
  if (per_sm < 1) return false;
  FwdMaps maps;
  if (!fwd_maps<T, NL>(src, g, out, maps)) return false;
  const int tiles_x = (int)ceil_div(g.w[NL], G::TX), tiles_y = (int)ceil_div(g.h[NL], G::TY);
  const int64_t grid = std::min<int64_t>((int64_t)tiles_x * tiles_y, (int64_t)device_sms() * per_sm);
  kern<<<(unsigned)grid, G::kThreads, G::kSmem, stream>>>(maps, g, flags, tiles_x, tiles_y);
  return true;
}

struct InvGeom {
  int64_t C;
  int64_t h[kMaxPass + 1], w[kMaxPass + 1];  // [l] = dims of the level-l low-pass / dir planes; [0] = output
  int64_t off[kMaxPass + 1][3];              // dh,dv,dd element offsets at level l (1..NL)
};

template <typename T, int NL, typename IT>
__global__ void __launch_bounds__(256) haar_inv_kernel(const T* __restrict__ top, const T* __restrict__ dirs,
                                                       InvGeom g, T* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const IT C = (IT)g.C;
  const int64_t total = g.h[NL] * g.w[NL] * g.C;
  if (t >= total) return;
  int64_t c64, J64, I64;
  split_index(t, total, g.C, g.w[NL], c64, J64, I64);
  const IT c = (IT)c64, J = (IT)J64, I = (IT)I64;
  constexpr int S0 = 1 << NL;

  T p[S0][S0];
  p[0][0] = ldg(top + (I * (IT)g.w[NL] + J) * C + c);
#pragma unroll
  for (int l = NL; l >= 1; --l) {
    const int Sl = 1 << (NL - l);  // positions per side owned at level l
    const IT br = I * Sl, bc = J * Sl;
    const IT hl = (IT)g.h[l], wl = (IT)g.w[l];
    const IT ho = (IT)g.h[l - 1], wo = (IT)g.w[l - 1];
    const T* const d0 = dirs + g.off[l][0];
    const T* const d1 = dirs + g.off[l][1];
    const T* const d2 = dirs + g.off[l][2];
    // walk backwards so in-place expansion never overwrites an unread parent
#pragma unroll
    for (int i = Sl - 1; i >= 0; --i) {
#pragma unroll
      for (int j = Sl - 1; j >= 0; --j) {
        const IT gi = br + i, gj = bc + j;
        T lp = p[i][j], dh = T(0), dv = T(0), dd = T(0);
        if (gi < hl && gj < wl) {
          const IT e = (gi * wl + gj) * C + c;
          dh = ldg(d0 + e);
          dv = ldg(d1 + e);
          dd = ldg(d2 + e);
        }
        const T o00 = T(0.5) * (((lp + dh) + dv) + dd);
        const T o01 = T(0.5) * (((lp + dh) - dv) - dd);
        const T o10 = T(0.5) * (((lp - dh) - dv) + dd);
        const T o11 = T(0.5) * (((lp - dh) + dv) - dd);
        if (l == 1) {
          const IT r0 = 2 * gi, c0 = 2 * gj;
          if (r0 < ho) {
            if (c0 < wo) out[(r0 * wo + c0) * C + c] = o00;
            if (c0 + 1 < wo) out[(r0 * wo + c0 + 1) * C + c] = o01;
          }
          if (r0 + 1 < ho) {
            if (c0 < wo) out[((r0 + 1) * wo + c0) * C + c] = o10;
            if (c0 + 1 < wo) out[((r0 + 1) * wo + c0 + 1) * C + c] = o11;
          }
        } else {
          p[2 * i][2 * j] = o00;
          p[2 * i][2 * j + 1] = o01;
          p[2 * i + 1][2 * j] = o10;
          p[2 * i + 1][2 * j + 1] = o11;
        }
      }
    }
  }
}

template <typename T>
int haar_forward_impl(const T* image, int64_t H, int64_t W, int64_t C, int n, T* planes, uint32_t* flags,
                      cudaStream_t stream) {
  if (n < 1 || H < 1 || W < 1 || C < 1) return OXM_ERR_ARGUMENT;
  if (!image || !planes) return OXM_ERR_ARGUMENT;
  // dims and plane offsets of every level
  int64_t hh = H, ww = W, off = 0;
  const T* src = image;
  int64_t level = 0;  // levels done
  while (level < n) {
    const int NL = static_cast<int>(min64(kMaxPass, n - level));
    FwdGeom g{};
    g.C = C;
    g.h[0] = hh;
    g.w[0] = ww;
    for (int k = 1; k <= NL; ++k) {
      g.h[k] = (g.h[k - 1] + 1) / 2;
      g.w[k] = (g.w[k - 1] + 1) / 2;
      const int64_t sz = g.h[k] * g.w[k] * C;
      for (int q = 0; q < 4; ++q) g.off[k][q] = off + q * sz;
      off += 4 * sz;
    }
    const int64_t total = g.h[NL] * g.w[NL] * C;
    const int threads = 128;
    const unsigned grid = grid_1d(total, threads);
    // 32-bit in-plane indices when the source plane and the largest output plane fit
    const bool i32 = g.h[0] * g.w[0] * C < ((int64_t)1 << 31);
    const bool tma = NL == 1   ? launch_fwd_tma<T, 1>(src, g, planes, flags, stream)
                     : NL == 2 ? launch_fwd_tma<T, 2>(src, g, planes, flags, stream)
                               : launch_fwd_tma<T, 3>(src, g, planes, flags, stream);
    if (tma) {
    } else if (i32) {
      switch (NL) {
        case 1: haar_fwd_kernel<T, 1, int32_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
        case 2: haar_fwd_kernel<T, 2, int32_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
        default: haar_fwd_kernel<T, 3, int32_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
      }
    } else {
      switch (NL) {
        case 1: haar_fwd_kernel<T, 1, int64_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
        case 2: haar_fwd_kernel<T, 2, int64_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
        default: haar_fwd_kernel<T, 3, int64_t><<<grid, threads, 0, stream>>>(src, g, planes, flags); break;
      }
    }
    int st = check_launch("haar_forward");
    if (st) return st;
    // next pass starts from this pass's coarsest low-pass plane
    src = planes + g.off[NL][0];
    hh = g.h[NL];
    ww = g.w[NL];
    level += NL;
  }
  return OXM_OK;
}

template <typename T>
int haar_inverse_impl(const T* coarse_lp, const T* dirs, const int64_t* shp, int n, int64_t C, T* out,
                      cudaStream_t stream) {
  if (n < 1 || C < 1 || !coarse_lp || !dirs || !out || !shp) return OXM_ERR_ARGUMENT;
  // validate the chain: level k planes (h_k, w_k); crop (oh_k, ow_k) <= 2*(h_k, w_k) effectively;
  // level k-1's planes must equal level k's crop (haar.py:105-109).
  int64_t eff_h[64], eff_w[64];
  if (n > 60) return OXM_ERR_ARGUMENT;
  for (int k = 0; k < n; ++k) {
    const int64_t h = shp[4 * k + 0], w = shp[4 * k + 1], oh = shp[4 * k + 2], ow = shp[4 * k + 3];
    if (h < 1 || w < 1 || oh < 0 || ow < 0) return OXM_ERR_DATA;
    eff_h[k] = std::min(oh, 2 * h);  // numpy slicing clamps out[:oh, :ow]
    eff_w[k] = std::min(ow, 2 * w);
    if (k > 0 && (shp[4 * (k - 1) + 0] != eff_h[k] || shp[4 * (k - 1) + 1] != eff_w[k])) return OXM_ERR_DATA;
  }
  if (eff_h[0] < 1 || eff_w[0] < 1) return OXM_ERR_DATA;
  // element offsets of each level's dh,dv,dd in the packed dirs buffer
  int64_t doff[64];
  int64_t acc = 0;
  for (int k = 0; k < n; ++k) {
    doff[k] = acc;
    acc += 3 * shp[4 * k] * shp[4 * k + 1] * C;
  }
  // passes from the coarsest level down; intermediate low-pass planes live in
  // stream-ordered scratch that is released right after its consumer launch
  const T* top = coarse_lp;
  T* prev_scratch = nullptr;
  int hi = n;  // levels hi .. lo+1 handled by this pass (1-based)
  int st = OXM_OK;
  while (hi > 0) {
    const int NLc = std::min(kMaxPass, hi);
    const int lo = hi - NLc;
    InvGeom g{};
    g.C = C;
    for (int l = 1; l <= NLc; ++l) {
      const int k = lo + l - 1;  // 0-based pyramid level index
      g.h[l] = shp[4 * k];
      g.w[l] = shp[4 * k + 1];
      for (int q = 0; q < 3; ++q) g.off[l][q] = doff[k] + q * g.h[l] * g.w[l] * C;
    }
    g.h[0] = eff_h[lo];
    g.w[0] = eff_w[lo];
    T* dst = out;
    T* new_scratch = nullptr;
    if (lo > 0) {
      const size_t bytes = sizeof(T) * (size_t)(g.h[0] * g.w[0] * C);
      cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&new_scratch), bytes, stream);
      if (err != cudaSuccess) {
        set_last_error("haar_inverse scratch", err);
        st = OXM_ERR_CUDA;
        break;
      }
      dst = new_scratch;
    }
    const int64_t total = g.h[NLc] * g.w[NLc] * C;
    const int threads = 128;
    const unsigned grid = grid_1d(total, threads);
    // 32-bit in-plane indices when the output plane (the largest) fits
    if (g.h[0] * g.w[0] * C < ((int64_t)1 << 31)) {
      switch (NLc) {
        case 1: haar_inv_kernel<T, 1, int32_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
        case 2: haar_inv_kernel<T, 2, int32_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
        default: haar_inv_kernel<T, 3, int32_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
      }
    } else {
      switch (NLc) {
        case 1: haar_inv_kernel<T, 1, int64_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
        case 2: haar_inv_kernel<T, 2, int64_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
        default: haar_inv_kernel<T, 3, int64_t><<<grid, threads, 0, stream>>>(top, dirs, g, dst); break;
      }
    }
    st = check_launch("haar_inverse");
    if (prev_scratch) cudaFreeAsync(prev_scratch, stream);
    prev_scratch = new_scratch;
    if (st) break;
    top = dst;
    hi = lo;
  }
  if (prev_scratch) cudaFreeAsync(prev_scratch, stream);
  return st;
}

}  // namespace
}  // namespace oxm

using namespace oxm;

extern "C" int oxm_haar_layout(int64_t height, int64_t width, int n_levels, int64_t* level_hw,
                               int64_t* total_elems_per_channel) {
  if (n_levels < 1 || height < 1 || width < 1) return OXM_ERR_ARGUMENT;
  int64_t h = height, w = width, tot = 0;
  for (int k = 0; k < n_levels; ++k) {
    h = (h + 1) / 2;
    w = (w + 1) / 2;
    if (level_hw) {
      level_hw[2 * k] = h;
      level_hw[2 * k + 1] = w;
    }
    tot += 4 * h * w;
  }
  if (total_elems_per_channel) *total_elems_per_channel = tot;
  return OXM_OK;
}

extern "C" int oxm_haar_forward_f32(const float* image, int64_t height, int64_t width, int64_t channels,
                                    int n_levels, float* planes, uint32_t* flags, void* stream) {
  return haar_forward_impl<float>(image, height, width, channels, n_levels, planes, flags, as_stream(stream));
}

extern "C" int oxm_haar_forward_f64(const double* image, int64_t height, int64_t width, int64_t channels,
                                    int n_levels, double* planes, uint32_t* flags, void* stream) {
  return haar_forward_impl<double>(image, height, width, channels, n_levels, planes, flags, as_stream(stream));
}

extern "C" int oxm_haar_inverse_f32(const float* coarse_lp, const float* dirs, const int64_t* level_shapes,
                                    int n_levels, int64_t channels, float* out, void* stream) {
  return haar_inverse_impl<float>(coarse_lp, dirs, level_shapes, n_levels, channels, out, as_stream(stream));
}

extern "C" int oxm_haar_inverse_f64(const double* coarse_lp, const double* dirs, const int64_t* level_shapes,
                                    int n_levels, int64_t channels, double* out, void* stream) {
  return haar_inverse_impl<double>(coarse_lp, dirs, level_shapes, n_levels, channels, out, as_stream(stream));
}
