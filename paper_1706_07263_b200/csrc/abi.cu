// C-ABI plumbing: status strings, per-thread CUDA error text and the
// immutable per-device operator context (include/oximap_b200.h).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>

#include "oxm_common.cuh"
#include "oxm_tables.h"

namespace oxm {

static thread_local char g_last_error[256] = "";

void set_last_error(const char* where, cudaError_t err) {
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s (%s)", where, cudaGetErrorString(err),
                cudaGetErrorName(err));
}

namespace {
// fp32 lead-in defaults (tools/em_lead_sweep.py): hand over to
// fp64 once rel <= 16 tol; redo in fp64 when a tail step has |rel/tol - 1| < 1%
constexpr double kDefaultLeadRatio = 16.0;
constexpr double kDefaultLeadGuard = 0.01;
// The tail's first step redoes the lead-in's uncommitted fit from the fp32 state
// itself, so its rel carries the hand-over noise undamped (~2.5e-6 |x| / (tol |x|)
// = ~2.5% of tol; tools/em_flip_study.py found the K = 4 flips exactly there, at
// rel/tol = 0.998 with the tail continuing): its guard band is 10x wider, and the
// band halves with every further tail step (the iteration contracts by <= 1/2 per
// fit, so the hand-over noise in rel does too) down to the plain guard.
constexpr double kDefaultFirstGuard = 0.10;
constexpr int kDefaultGuardShift = 2;  // the band quarters per tail step (the measured contraction)

void set_first_guard(DevOps& d, double g1, int shift) {
  d.guard1 = g1;
  d.guard_shift = shift;
  for (int k = 0; k < 3; ++k) {
    // step j = k + 1; the last entry serves every later step, so it uses the
    // larger of step 3's band and the floor (exact for shift >= 2 or g1 <= 4 guard)
    const double gj = std::fmax(d.guard, g1 * std::ldexp(1.0, -k * shift));
    d.band_lo[k] = (1.0 - gj) * (1.0 - gj) * d.rel_tol * d.rel_tol;
    d.band_hi[k] = (1.0 + gj) * (1.0 + gj) * d.rel_tol * d.rel_tol;
  }
}

void set_em_lead(DevOps& d, double ratio, double guard, double exact_below) {
  d.exact_below = exact_below;
  const double kt = ratio * d.rel_tol;
  d.lead_thr_f = ratio > 1.0 ? static_cast<float>(kt * kt) : 0.0f;
  d.guard = guard;
  set_first_guard(d, kDefaultFirstGuard > guard ? kDefaultFirstGuard : guard, kDefaultGuardShift);
}
}  // namespace

}  // namespace oxm

using namespace oxm;

extern "C" int oxm_abi_version(void) { return OXM_ABI_VERSION; }

extern "C" const char* oxm_last_error(void) { return g_last_error; }

extern "C" const char* oxm_status_string(int status) {
  switch (status) {
    case OXM_OK: return "ok";
    case OXM_ERR_ARGUMENT: return "argument error";
    case OXM_ERR_DATA: return "data error";
    case OXM_ERR_NUMERICAL: return "numerical error";
    case OXM_ERR_SINGULAR: return "singular operator";
    case OXM_ERR_ILL_CONDITIONED: return "ill-conditioned prior";
    case OXM_ERR_CUDA: return "cuda error";
    case OXM_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

extern "C" int oxm_ctx_create(int device, const oxm_operators* o, oxm_ctx** out) {
  if (!o || !out) return OXM_ERR_ARGUMENT;
  *out = nullptr;
  const int L = o->n_bands;
  // BayesConfig.__post_init__ domain (bayes.py:50-58)
  if (L < 3 || L > kMaxBands) return OXM_ERR_ARGUMENT;
  if (o->max_iters < 1) return OXM_ERR_ARGUMENT;
  if (!(o->epsilon > 0.0 && o->epsilon < 1.0)) return OXM_ERR_ARGUMENT;
  if (!(o->rel_tol > 0.0)) return OXM_ERR_ARGUMENT;
  if (!o->solve || !o->fit_mat || !o->xi || !o->sens || !o->gain) return OXM_ERR_ARGUMENT;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    set_last_error("oxm_ctx_create", cudaErrorInvalidDevice);
    cudaGetLastError();
    return OXM_ERR_CUDA;
  }
  oxm_ctx* c = new (std::nothrow) oxm_ctx();
  if (!c) return OXM_ERR_CUDA;
  std::memset(static_cast<void*>(&c->ops), 0, sizeof(c->ops));
  c->device = device;
  DevOps& d = c->ops;
  d.L = L;
  d.max_iters = o->max_iters;
  d.eps = o->epsilon;
  d.rel_tol = o->rel_tol;
  d.rel_tol2 = o->rel_tol * o->rel_tol;
  // the fp32 map path skips the eps clamp, which is only sound when every
  // band below the fallback threshold is recomputed in fp64
  d.fallback_below = o->fallback_below > o->epsilon ? o->fallback_below : o->epsilon;
  d.eps_f = static_cast<float>(o->epsilon);
  const double ln2 = 0.69314718055994530942;
  for (int l = 0; l < L; ++l) {
    for (int k = 0; k < 3; ++k) {
      d.solve[l][k] = o->solve[3 * l + k];
      d.xi[l][k] = o->xi[3 * l + k];
      d.gain[l][k] = o->gain[3 * l + k];
      d.fitm[k][l] = o->fit_mat[k * L + l];
      d.sens[k][l] = o->sens[k * L + l];
      d.solve_f[l][k] = static_cast<float>(d.solve[l][k]);
      d.fitl2_f[k][l] = static_cast<float>(-ln2 * d.fitm[k][l]);
      d.solve_f2[l][k] = make_float2(d.solve_f[l][k], d.solve_f[l][k]);
      d.fitl2_f2[k][l] = make_float2(d.fitl2_f[k][l], d.fitl2_f[k][l]);
    }
  }
  const double log2e = 1.44269504088896340736;
  for (int l = 0; l < L; ++l) {
    d.xl2_t[0][l] = static_cast<float>(-log2e * d.xi[l][0]);
    d.xl2_t[1][l] = static_cast<float>(-log2e * d.xi[l][1]);
    for (int k = 0; k < 3; ++k) {
      d.sens_f[k][l] = static_cast<float>(d.sens[k][l]);
      d.gain_t[k][l] = static_cast<float>(d.gain[l][k]);
    }
  }
  set_em_lead(d, kDefaultLeadRatio, kDefaultLeadGuard, d.fallback_below);
  for (int l = 0; l < L; ++l) {
    d.xis[l][0] = d.xi[l][0] * kExpScale;
    d.xis[l][1] = d.xi[l][1] * kExpScale;
  }
  // the EM kernels use xi[:, 2] == 1 (ChromophoreBasis contract, core.py:152-153)
  for (int l = 0; l < L; ++l)
    if (d.xi[l][2] != 1.0) {
      delete c;
      return OXM_ERR_ARGUMENT;
    }
  for (int l = 0; l < L; ++l)
    for (int k = 0; k < 3; ++k)
      if (!std::isfinite(d.solve[l][k]) || !std::isfinite(d.xi[l][k]) || !std::isfinite(d.gain[l][k]) ||
          !std::isfinite(d.fitm[k][l]) || !std::isfinite(d.sens[k][l])) {
        delete c;
        return OXM_ERR_NUMERICAL;
      }
  {
    double rows[kMaxBands * 8] = {};
    for (int l = 0; l < L; ++l)
      for (int k = 0; k < 3; ++k) {
        rows[8 * l + k] = d.solve[l][k];
        rows[8 * l + 3 + k] = d.fitm[k][l];
      }
    DeviceGuard dg(device);
    void* dev = nullptr;
    cudaError_t err = cudaMalloc(&dev, sizeof(double) * 8 * (size_t)L);
    if (err == cudaSuccess) err = cudaMemcpy(dev, rows, sizeof(double) * 8 * (size_t)L, cudaMemcpyHostToDevice);
    if (err != cudaSuccess) {
      set_last_error("oxm_ctx_create band rows", err);
      if (dev) cudaFree(dev);
      delete c;
      return OXM_ERR_CUDA;
    }
    d.band_rows = static_cast<const double*>(dev);
  }
  *out = c;
  return OXM_OK;
}

extern "C" int oxm_ctx_set_em_lead(oxm_ctx* ctx, double ratio, double guard, double exact_below) {
  if (!ctx || !(ratio >= 0.0) || !(guard >= 0.0 && guard < 1.0) || !(exact_below >= 0.0)) return OXM_ERR_ARGUMENT;
  if (ratio > 1.0 && (ratio * ctx->ops.rel_tol >= 1.0 || guard <= 0.0)) return OXM_ERR_ARGUMENT;
  set_em_lead(ctx->ops, ratio, guard, exact_below);
  return OXM_OK;
}

extern "C" int oxm_ctx_set_em_first_guard(oxm_ctx* ctx, double guard1, int halvings_per_step) {
  if (!ctx || !(guard1 >= 0.0 && guard1 < 1.0) || halvings_per_step < 1) return OXM_ERR_ARGUMENT;
  set_first_guard(ctx->ops, guard1, halvings_per_step > 64 ? 64 : halvings_per_step);
  return OXM_OK;
}

extern "C" int oxm_ctx_set_em_debug_log(oxm_ctx* ctx, float* rel, uint8_t* step) {
  if (!ctx || (!rel) != (!step)) return OXM_ERR_ARGUMENT;
  ctx->ops.dbg_rel = rel;
  ctx->ops.dbg_step = step;
  return OXM_OK;
}

extern "C" int oxm_ctx_destroy(oxm_ctx* ctx) {
  if (ctx && ctx->ops.band_rows) {
    DeviceGuard dg(ctx->device);
    cudaFree(const_cast<double*>(ctx->ops.band_rows));
  }
  delete ctx;
  return OXM_OK;
}
