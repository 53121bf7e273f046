/*
 * oximap_b200.h -- C ABI of the B200-native haemoglobin-map path.
 *
 * The reference (`oximap`, /root/reference/pkg/src/oximap) is pure Python and
 * has no FFI layer: its boundary is the public Python API re-exported by
 * pkg/src/oximap/__init__.py:10-80.  Every entry point below replaces the body
 * of one of those Python functions (cited per function); a ctypes binding of
 * this header is what `oximap` would call.
 *
 * Conventions
 *  - Plain C types only: device pointers, element counts, a cudaStream_t passed
 *    as `void*` (NULL = legacy default stream).  No torch types.
 *  - All arrays are C-order.  Images/planes are HWC interleaved (H, W, C) like
 *    the reference's NumPy arrays; per-coefficient vectors are (n, 3) / (n, L).
 *  - Every function returns an `int` status (OXM_OK or a negative OXM_ERR_*).
 *    Shape/config errors are returned before any launch.  Data-dependent
 *    errors (non-finite input, negative low-pass) are detected on the device and
 *    reported as bits in a caller-owned `uint32_t* flags` word that the caller
 *    reads after synchronising the stream (the reference raises them eagerly,
 *    haar.py:133-134, bayes.py:77-78).
 *  - Launches are asynchronous on `stream`; the library holds no global
 *    mutable state besides immutable operator contexts.
 */
#ifndef OXIMAP_B200_H
#define OXIMAP_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define OXM_API __attribute__((visibility("default")))
#else
#define OXM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define OXM_ABI_VERSION 2
#define OXM_MAX_BANDS 64 /* spectral bands L supported by the kernels */

/* Status codes; the Python host maps them onto the reference exception
 * classes of errors.py:1-30. */
enum {
  OXM_OK = 0,
  OXM_ERR_ARGUMENT = -1,        /* ArgumentError                         */
  OXM_ERR_DATA = -2,            /* DataError                             */
  OXM_ERR_NUMERICAL = -3,       /* NumericalError                        */
  OXM_ERR_SINGULAR = -4,        /* SingularOperatorError                 */
  OXM_ERR_ILL_CONDITIONED = -5, /* IllConditionedPriorError              */
  OXM_ERR_CUDA = -10,           /* CUDA runtime error (launch / device)  */
  OXM_ERR_WORKSPACE = -11       /* workspace too small                   */
};

/* Device-side flag bits (OR-ed into *flags by the kernels). */
#define OXM_FLAG_NONFINITE 1u   /* input sample not finite: haar.py:133-134, core.py:18-22 */
#define OXM_FLAG_NEGATIVE_LL 2u /* low-pass coefficient < 0: bayes.py:77-78               */

/* Host-side operator set (all float64, C-order).  Built by the Python host
 * exactly as the reference builds them:
 *   solve     L x 3  Tikhonov ridge inverse (C^T C + g I)^-1 C^T   unmix.py:53-74
 *   fit_mat   3 x L  (xi^T xi)^-1 xi^T                             bayes.py:99-104
 *   xi        L x 3  chromophore basis (hbo, hb, 1); xi[:, 2] must be 1  core.py:134-158
 *   sens      3 x L  camera sensitivity C                          core.py:112-131
 *   gain      L x 3  N^-1 C^T, N = C^T C + beta D2^T D2            bayes.py:117-129
 * The shape-prior update N^-1 (C^T y + P e) of bayes.py:131-135 is evaluated
 * as e + gain (y - C e), an exact identity because N^-1 P = I - N^-1 C^T C. */
typedef struct oxm_operators {
  int32_t n_bands;   /* L, 3 <= L <= OXM_MAX_BANDS   */
  int32_t max_iters; /* BayesConfig.max_iters >= 1   */
  double epsilon;    /* BayesConfig.epsilon in (0,1) */
  double rel_tol;    /* BayesConfig.rel_tol > 0      */
  double fallback_below; /* fp32 map path: recompute a pixel in fp64 when its
                            smallest reconstructed band is below this       */
  const double* solve;
  const double* fit_mat;
  const double* xi;
  const double* sens;
  const double* gain;
} oxm_operators;

typedef struct oxm_ctx oxm_ctx;

/* ---- library ------------------------------------------------------------ */
OXM_API int oxm_abi_version(void);
OXM_API const char* oxm_status_string(int status);
/* Last CUDA error string recorded by this thread (for OXM_ERR_CUDA). */
OXM_API const char* oxm_last_error(void);

/* Immutable per-device operator context.
 * Replaces the per-call operator construction of pipeline.py:182 /
 * bayes.py:239-240 (done once per (sensitivity, basis, config)). */
OXM_API int oxm_ctx_create(int device, const oxm_operators* ops, oxm_ctx** out);
OXM_API int oxm_ctx_destroy(oxm_ctx* ctx);
/* EM precision schedule of the fp32 map path (oxm_hybrid_maps_f32/_u16/_split).
 * ratio > 1: fits run in fp32 while rel > ratio * rel_tol, then in fp64; a
 * fp64 step with |rel/rel_tol - 1| < guard (or reaching max_iters) redoes
 * its coefficient in fp64 from fit #1.  ratio <= 1: all fits in fp64.
 * exact_below > 0: low-pass blocks holding a fallback pixel with a band in
 * [epsilon / 2, exact_below) are re-estimated all-fp64 before the fp64 pixel
 * fallback (such small unclamped bands would amplify the schedule's ~1e-8
 * spectrum deviation through log s); 0 = never.  Default (16, 0.01, ops.fallback_below).  The drop-in fp64 entry
 * points are always all-fp64.  Not thread-safe against concurrent launches on
 * the same context. */
OXM_API int oxm_ctx_set_em_lead(oxm_ctx* ctx, double ratio, double guard, double exact_below);
/* Guard band of the fp64 tail's first steps: tail step j (j = 1 is the redo of
 * the lead-in's uncommitted fit, whose input carries the fp32 hand-over noise
 * undamped) with |rel/rel_tol - 1| < max(guard, guard1 * 2^(-(j-1) h)),
 * h = halvings_per_step (>= 1; 64 = only the first step is widened; from the
 * third step on the band is max(guard, guard1 * 2^(-2h))), or any
 * stop at j = 1, redoes the coefficient in fp64 from fit #1.  Default
 * (max(0.10, guard), 2); oxm_ctx_set_em_lead resets it. */
OXM_API int oxm_ctx_set_em_first_guard(oxm_ctx* ctx, double guard1, int halvings_per_step);
/* Diagnostics for tools/em_margin_study.py: device buffers of (n_coefficients x 24)
 * entries; the fp64 EM kernels of later launches on this context record, for fit m
 * of low-pass coefficient i, rel at rel[i * 24 + m] and the tail step index (0 =
 * exact fp64 trajectory, j = 1, 2 = j-th step after the fp32 hand-over, 3 = a
 * later one) at
 * step[i * 24 + m].  NULL, NULL (default) turns it off. */
OXM_API int oxm_ctx_set_em_debug_log(oxm_ctx* ctx, float* rel, uint8_t* step);

/* ---- K1: multi-level Haar forward ---------------------------------------
 * Replaces haar.forward (haar.py:120-142) incl. per-level edge replication
 * (haar.py:80-85).  `planes` receives, for level k = 1..n (finest first), the
 * four planes lp, dh, dv, dd of shape (h_k, w_k, C) back to back, where
 * h_k = ceil(h_{k-1} / 2).  oxm_haar_layout gives h_k, w_k and the total
 * element count.  Non-finite input sets OXM_FLAG_NONFINITE. */
OXM_API int oxm_haar_layout(int64_t height, int64_t width, int n_levels,
                    int64_t* level_hw /* n_levels x 2, may be NULL */,
                    int64_t* total_elems_per_channel);
OXM_API int oxm_haar_forward_f32(const float* image, int64_t height, int64_t width, int64_t channels,
                         int n_levels, float* planes, uint32_t* flags, void* stream);
OXM_API int oxm_haar_forward_f64(const double* image, int64_t height, int64_t width, int64_t channels,
                         int n_levels, double* planes, uint32_t* flags, void* stream);

/* ---- K2: multi-level Haar inverse ---------------------------------------
 * Replaces haar.inverse (haar.py:104-117, 145-150).  `level_shapes` holds for
 * each level k = 1..n (finest first) four int64: plane rows h_k, plane cols
 * w_k, and the crop (orig rows, orig cols) of that level.  `dirs` packs dh, dv,
 * dd of every level (finest first), each (h_k, w_k, C); `coarse_lp` is the
 * residual low-pass (h_n, w_n, C).  Output (orig rows_1, orig cols_1, C).
 * Inconsistent shapes return OXM_ERR_DATA (haar.py:105-109). */
OXM_API int oxm_haar_inverse_f32(const float* coarse_lp, const float* dirs, const int64_t* level_shapes,
                         int n_levels, int64_t channels, float* out, void* stream);
OXM_API int oxm_haar_inverse_f64(const double* coarse_lp, const double* dirs, const int64_t* level_shapes,
                         int n_levels, int64_t channels, double* out, void* stream);

/* ---- K3: per-coefficient 3 -> L linear unmix ----------------------------
 * Replaces tikhonov_unmix (unmix.py:77-82) and, with the min-norm matrix,
 * lsq_unmix (unmix.py:21-37): out[i, :] = matrix (L x 3, host) @ rgb[i, :]. */
OXM_API int oxm_unmix_f32(int n_bands, const double* matrix, const float* rgb, int64_t n, float* out,
                  void* stream);
OXM_API int oxm_unmix_f64(int n_bands, const double* matrix, const double* rgb, int64_t n, double* out,
                  void* stream);

/* ---- K4: iterative low-pass (shape-prior EM) estimator ------------------
 * Replaces estimate_lowpass / _iterate_block (bayes.py:185-272).  `y` is the
 * unit-scale low-pass data (n, 3) (rgb_lp / scale, bayes.py:237).  `init`
 * (n, L) replaces the Tikhonov start when non-NULL (bayes.py:243-249).
 * Outputs: spectra (n, L), x (n, 3) = (hbo, hb, offset) fit of spectra, and
 * fits (n) = number of Beer-Lambert fits run for that coefficient (the
 * discrete stopping decision of bayes.py:199-205), each may be NULL. */
OXM_API int oxm_em_lowpass(const oxm_ctx* ctx, const double* y, const double* init, int64_t n,
                   double* spectra, double* x, int32_t* fits, void* stream);

/* Shape-prior update for arbitrary (y, e) pairs: expectation_step
 * (bayes.py:162-182), out (n, L) = N^-1 (C^T y + P e) (no clamp). */
OXM_API int oxm_expectation_step(const oxm_ctx* ctx, const double* y, const double* e, int64_t n,
                         double* out, void* stream);

/* ---- K5: per-pixel Beer-Lambert fit -------------------------------------
 * Replaces fit_cube (pipeline.py:66-94) / fit_concentration (bayes.py:138-151):
 * x = -fit_mat log(max(s, eps)) then x * (cal, cal, 1).  Outputs planar
 * hbo, hb, offset (n each); any may be NULL. */
OXM_API int oxm_fit_f32(const oxm_ctx* ctx, const float* cube, int64_t n, double calibration,
                float* hbo, float* hb, float* offset, void* stream);
OXM_API int oxm_fit_f64(const oxm_ctx* ctx, const double* cube, int64_t n, double calibration,
                double* hbo, double* hb, double* offset, void* stream);
/* Beer-Lambert forward model exp(-xi x): expected_spectrum (bayes.py:154-159). */
OXM_API int oxm_expected_spectrum_f64(const oxm_ctx* ctx, const double* x, int64_t n, double* out,
                              void* stream);

/* ---- K6: fused hybrid estimator (estimate_frame mode="hybrid") ----------
 * Replaces pipeline.py:176-217 + fit_cube + ConcentrationMap.thb/sat_o2
 * (core.py:197-209) for a batch of `batch` frames (batch, H, W, 3).
 * Uses the exact collapse of the hybrid path: for pixel p in low-pass block
 * b = (py >> n, px >> n),  cube(p) = S[b] + solve (rgb(p) - LL_n[b] / 2^n),
 * with LL_n the recursively edge-replicated low-pass (haar.py:80-101) and
 * S = the EM spectra of LL_n / 2^n (bayes.py:185-207).
 * Workspace: oxm_hybrid_workspace_bytes(); any output pointer may be NULL.
 * f32 variant: fp64 low-pass chain, EM with an fp32 lead-in and an fp64
 * tail (fit counts bit-exact, spectra ~1e-8 relative of all-fp64; see
 * oxm_ctx_set_em_lead), fp32 per-pixel stage with an fp64 recompute of
 * pixels whose smallest band < ops.fallback_below.
 * Outputs are planar (batch, H, W); fits is (batch, ceil(H/2^n), ceil(W/2^n)).
 * stage_events: NULL, or 6 cudaEvent_t recorded on `stream` before the
 * low-pass kernel, before the EM's fp32 lead-in, before its fp64 kernel,
 * before the per-pixel kernel (which also finishes most fp64-fallback pixels
 * in place), before the fixup (exact-block EM, deferred pixels) and after it (live
 * per-kernel timing for the roofline report; with no lead-in, events 1 and 2
 * coincide). */
OXM_API size_t oxm_hybrid_workspace_bytes(const oxm_ctx* ctx, int64_t batch, int64_t height,
                                  int64_t width, int n_levels);
/* EM work counters of the last fp32-map launch that used `workspace` (same
 * geometry): out[0] fp32 fits of the lead-in, out[1] fp64 fits of the tail,
 * out[2] tail restarts in exact mode, out[3] low-pass blocks re-estimated
 * all-fp64 for the fp64 pixel fallback, out[4] pixels that took the fp64
 * fallback, out[5] of those, the ones deferred to after the exact pass
 * (`out` holds 6 values).  Synchronises `stream`. */
OXM_API int oxm_hybrid_em_counters(const oxm_ctx* ctx, void* workspace, int64_t batch, int64_t height,
                                   int64_t width, int n_levels, uint64_t* out, void* stream);
OXM_API int oxm_hybrid_maps_f32(const oxm_ctx* ctx, const float* frames, int64_t batch, int64_t height,
                        int64_t width, int n_levels, double calibration, void* workspace,
                        size_t workspace_bytes, float* thb, float* so2, float* hbo, float* hb,
                        float* offset, int32_t* fits, uint32_t* flags, void* stream,
                        void* const* stage_events);
/* Split launch for sub-batch pipelining: low-pass chain + EM on stream_em,
 * then (after an event) the per-pixel stage on stream_px, so the caller can
 * overlap the per-pixel stage of sub-batch k (MUFU/FMA pipes) with the EM of
 * sub-batch k+1 (fp64 pipe).  em_reserve leaves that many CTA slots per SM
 * free during the persistent EM for the concurrent kernel. */
OXM_API int oxm_hybrid_maps_f32_split(const oxm_ctx* ctx, const float* frames, int64_t batch, int64_t height,
                              int64_t width, int n_levels, double calibration, void* workspace,
                              size_t workspace_bytes, float* thb, float* so2, float* hbo, float* hb,
                              float* offset, int32_t* fits, uint32_t* flags, void* stream_em, void* stream_px,
                              int em_reserve);
/* 16-bit PPM rasters (the CLI's input format, io.py:88-162): `frames` holds
 * (batch, H, W, 3) u16 counts, big-endian as stored in the file when
 * big_endian != 0; sample value = count * scale computed in fp64 exactly as
 * read_ppm does.  Halves host->device bytes versus fp32 frames. */
OXM_API int oxm_hybrid_maps_u16(const oxm_ctx* ctx, const uint16_t* frames, int big_endian, double scale,
                        int64_t batch, int64_t height, int64_t width, int n_levels, double calibration,
                        void* workspace, size_t workspace_bytes, float* thb, float* so2, float* hbo, float* hb,
                        float* offset, int32_t* fits, uint32_t* flags, void* stream, void* const* stage_events);
/* f64 variant used by the drop-in estimate_frame: everything in fp64, and the
 * (H, W, L) spectral cube (pipeline.py:207-208) is produced when cube != NULL. */
OXM_API int oxm_hybrid_frame_f64(const oxm_ctx* ctx, const double* frames, int64_t batch, int64_t height,
                         int64_t width, int n_levels, double calibration, void* workspace,
                         size_t workspace_bytes, double* cube, double* hbo, double* hb,
                         double* offset, int32_t* fits, uint32_t* flags, void* stream,
                         void* const* stage_events);

/* ---- off-path helpers ------------------------------------
 * Synthetic frames on the device: synth.py:150-184 (forward model exp(-xi x),
 * Gaussian reflectance noise floored at 1e-6, camera projection x exposure)
 * for `count` frames of one (H, W, 3) truth map (hbo, hb, offset), fp32.
 * Noise: Philox4x32-10 keyed by `seed`, indexed by (frame0 + f, pixel, band). */
OXM_API int oxm_synth_frames_f32(const oxm_ctx* ctx, const float* truth, int64_t height, int64_t width,
                         int64_t count, double noise_sigma, double exposure, uint64_t seed,
                         uint64_t frame0, float* out, void* stream);
/* Pulse sequence on the device: synth.py:187-231 (pulse_sequence) -- frame
 * frame0 + f scales both haemoglobin truth planes by
 * 1 + amplitude * sin(2 pi pulse_hz (frame0 + f) / fps) (offset unchanged), then
 * the forward model / noise / projection of oxm_synth_frames_f32.  Requires
 * amplitude >= 0 and, when amplitude > 0, 0 < pulse_hz < fps / 2 (synth.py:209-216). */
OXM_API int oxm_synth_pulse_frames_f32(const oxm_ctx* ctx, const float* truth, int64_t height, int64_t width,
                         int64_t count, double noise_sigma, double exposure, uint64_t seed,
                         uint64_t frame0, double fps, double pulse_hz, double amplitude, float* out,
                         void* stream);
/* Patch-mean THb trace: timeseries.py:44-73 -- per frame, the sum and count
 * of finite THb values in rect (x, y, w, h) of (batch, H, W) maps. */
OXM_API int oxm_patch_mean_f32(const float* thb, int64_t batch, int64_t height, int64_t width, int x, int y,
                       int w, int h, double* sums, unsigned long long* counts, void* stream);

/* SPC1 map payload (io.py:34-39, 79-80): interleave hbo, hb, offset planes
 * (n each) into the file's (H, W, 3) little-endian fp32 layout. */
OXM_API int oxm_pack_hwc3_f32(const float* a, const float* b, const float* c, int64_t n, float* out, void* stream);

/* ---- roofline probes ------------------------------------------------------
 * Measure the pipe peaks the non-GEMM kernels are bound by, on this device:
 * fp64 FMA throughput (EM) and fp32 MUFU lg2 throughput (per-pixel fit).
 * Each launches `blocks` x 256 threads doing `iters` rounds of 8 independent
 * chains; *ops_per_launch receives the operation count (FMA or lg2). */
OXM_API int oxm_probe_fp64_fma(int blocks, int iters, double* sink, double* ops_per_launch, void* stream);
OXM_API int oxm_probe_mufu_lg2(int blocks, int iters, float* sink, double* ops_per_launch, void* stream);

/* Self-test of the EM's table-driven fp64 transcendentals (oxm_math.cuh):
 * out[i] = exp(in[i] * ln2/256) (which == 0: the EM's pre-scaled argument,
 * |in| < 2.5e5) or log(in[i]) (which == 1, in > 0 normal), evaluated exactly
 * as the EM kernels do.  For accuracy tests against a high-precision
 * reference; not on the hot path. */
OXM_API int oxm_selftest_math(const double* in, int64_t n, int which, double* out, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* OXIMAP_B200_H */
