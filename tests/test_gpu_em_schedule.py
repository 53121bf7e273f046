"""GPU tests of the EM precision schedule of the fp32 map path (oxm_em.cuh:
fp32 lead-in -> fp64 tail with guard-band restarts -> all-fp64 re-estimate of
the blocks holding "sensitive" fallback pixels).

The schedule must not change any discrete decision: per-coefficient fit
counts equal the all-fp64 schedule's (which equal the oracle's,
test_gpu_pipeline.py), and maps stay within a small multiple of fp32
rounding of the all-fp64 schedule, far inside the north-star tolerances."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import paper_1706_07263_b200 as ox
from oracle import oximap_oracle as O
from paper_1706_07263_b200 import _native, synth

pytestmark = pytest.mark.gpu


def _run(cuda, sensitivity, basis, frames, n, em_lead):
    eng = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=n), em_lead=em_lead)
    x = torch.from_numpy(frames.astype(np.float32)).to(cuda)
    out = eng.run(x, fits=True)
    torch.cuda.synchronize()
    B, H, W = frames.shape[:3]
    return eng, out, eng.em_counters(B, H, W)


def _maps(out):
    return out.thb.double().cpu().numpy(), out.so2.double().cpu().numpy(), out.fits.cpu().numpy()


@pytest.fixture(scope="module")
def textured(sensitivity, basis):
    # 2 textured 1080p frames: thousands of fallback pixels, some sensitive
    return np.stack([synth.phantom_rgb_f32(1080, 1920, s, sensitivity, basis) for s in (11, 12)])


def test_schedule_matches_all_fp64(cuda, sensitivity, basis, textured):
    _, ref, c0 = _run(cuda, sensitivity, basis, textured, 2, None)
    assert c0["lead_fits"] == 0 and c0["exact_blocks"] == 0
    rt, rs, rf = _maps(ref)
    for lead in ((16.0, 0.01), (8.0, 0.01), (64.0, 0.01)):
        _, out, c = _run(cuda, sensitivity, basis, textured, 2, lead)
        t, s, f = _maps(out)
        assert np.array_equal(f, rf), f"{lead}: {np.sum(f != rf)} fit-count differences"
        assert np.array_equal(np.isnan(s), np.isnan(rs))
        ok = ~np.isnan(rs)
        assert np.max(np.abs(t - rt) / np.abs(rt)) < 1e-5, lead
        assert np.max(np.abs(s[ok] - rs[ok])) < 5e-6, lead
        assert c["lead_fits"] > 0 and c["tail_fits"] > 0
        # the counters account for every fit past fit #1 (restarted work on top)
        assert c["lead_fits"] + c["tail_fits"] >= int(f.sum()) - f.size
        assert c["exact_blocks"] > 0  # textured 1080p frames always hold sensitive fallback pixels


def test_schedule_vs_oracle_textured(cuda, sensitivity, basis, textured):
    _, out, _ = _run(cuda, sensitivity, basis, textured[:1], 2, (16.0, 0.01))
    ref = O.estimate_frame(textured[0], sensitivity.c, basis.xi, n_levels=2, want_cube=False,
                           threads=O.default_threads())
    t, s, f = _maps(out)
    assert np.array_equal(f[0], ref["fits"])
    assert np.array_equal(np.isnan(s[0]), np.isnan(ref["so2"]))
    assert np.all(np.abs(t[0] - ref["thb"]) <= 1e-4 * np.abs(ref["thb"]))
    ok = ~np.isnan(ref["so2"])
    assert np.max(np.abs(s[0][ok] - ref["so2"][ok])) <= 1e-5


def test_exact_blocks_needed(cuda, sensitivity, basis, textured):
    """Without the exact re-estimate the sensitive fallback pixels carry the
    schedule's spectrum deviation amplified by cancellation (the reason the
    pass exists); fit counts are still exact."""
    _, ref, _ = _run(cuda, sensitivity, basis, textured, 2, None)
    _, out, c = _run(cuda, sensitivity, basis, textured, 2, (16.0, 0.01, 0.0))
    assert c["exact_blocks"] == 0
    rt, rs, rf = _maps(ref)
    t, s, f = _maps(out)
    assert np.array_equal(f, rf)
    with_exact = _maps(_run(cuda, sensitivity, basis, textured, 2, (16.0, 0.01))[1])
    dev_without = np.max(np.abs(t - rt) / np.abs(rt))
    dev_with = np.max(np.abs(with_exact[0] - rt) / np.abs(rt))
    assert dev_with < dev_without


def test_schedule_deterministic(cuda, sensitivity, basis, textured):
    eng, a, _ = _run(cuda, sensitivity, basis, textured, 2, (16.0, 0.01))
    b = eng.run(torch.from_numpy(textured.astype(np.float32)).to(cuda), fits=True)
    assert torch.equal(a.thb, b.thb)
    assert torch.equal(a.so2.nan_to_num(-1.0), b.so2.nan_to_num(-1.0))
    assert torch.equal(a.fits, b.fits)


def test_max_iters_small_with_lead(cuda, sensitivity, basis):
    """max_iters 2 and 3: the lead-in may commit no fit / one fit; counts and
    maps must still equal the oracle's (capped coefficients restart exactly)."""
    rgb = synth.phantom_rgb_f32(64, 96, 3, sensitivity, basis)
    for it in (2, 3):
        cfg = ox.PipelineConfig(n_levels=2, bayes=ox.BayesConfig(max_iters=it))
        eng = ox.HybridMapEngine(sensitivity, basis, cfg)
        out = eng.run(torch.from_numpy(rgb[None].astype(np.float32)).to(cuda), fits=True)
        ref = O.estimate_frame(rgb, sensitivity.c, basis.xi, n_levels=2, max_iters=it, want_cube=False)
        assert np.array_equal(out.fits[0].cpu().numpy(), ref["fits"]), it
        assert np.all(np.abs(out.thb[0].cpu().numpy() - ref["thb"]) <= 1e-4 * np.abs(ref["thb"]))


def test_set_em_lead_validation(cuda, sensitivity, basis):
    eng = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=2), em_lead=None)
    lib, h = _native.load(), eng.ctx.handle
    ok, bad = _native.OXM_OK, _native.OXM_ERR_ARGUMENT
    assert lib.oxm_ctx_set_em_lead(h, 16.0, 0.01, 2e-3) == ok
    assert lib.oxm_ctx_set_em_lead(h, 0.0, 0.01, 0.0) == ok   # all-fp64
    assert lib.oxm_ctx_set_em_lead(h, 1e4, 0.01, 0.0) == bad  # ratio * tol >= 1
    assert lib.oxm_ctx_set_em_lead(h, 16.0, 1.0, 0.0) == bad  # guard >= 1
    assert lib.oxm_ctx_set_em_lead(h, 16.0, 0.0, 0.0) == bad  # lead-in without a guard band
    assert lib.oxm_ctx_set_em_lead(h, -1.0, 0.01, 0.0) == bad
    assert lib.oxm_ctx_set_em_lead(h, 16.0, 0.01, -1.0) == bad
    assert lib.oxm_ctx_set_em_lead(None, 16.0, 0.01, 0.0) == bad
    out = (ctypes.c_uint64 * 6)()
    assert lib.oxm_hybrid_em_counters(None, None, 1, 8, 8, 1, out, None) == bad


def test_large_batch_exact_pass_matches_small(cuda, sensitivity, basis):
    """Batches of >= 2^21 low-pass coefficients run the exact-block pass on the
    one-lane persistent kernel, smaller ones on 4-lane groups: same fit counts,
    maps equal to within fp32 rounding (the two differ only in the summation
    order of the 26-term sums)."""
    import bench

    frames = bench.make_frames(17, 1080, 1920, 0.3, 0, cuda)  # 17 x 129600 > 2^21 coefficients
    eng = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=2))
    big = eng.run(frames, fits=True)
    c = eng.em_counters(17, 1080, 1920)
    assert c["exact_blocks"] > 0
    for b0 in range(0, 17, 4):
        small = eng.run(frames[b0:b0 + 4].contiguous(), fits=True)
        nb = small.thb.shape[0]
        assert torch.equal(small.fits, big.fits[b0:b0 + nb])
        rt = big.thb[b0:b0 + nb].double()
        assert float(((small.thb.double() - rt).abs() / rt.abs()).max()) < 1e-6
        rs, ss = big.so2[b0:b0 + nb], small.so2
        assert torch.equal(torch.isnan(rs), torch.isnan(ss))
        ok = ~torch.isnan(rs)
        assert float((rs[ok] - ss[ok]).abs().max()) < 1e-6


@pytest.mark.parametrize("gain", [1e-4, 3e-2, 30.0])
def test_schedule_extreme_exposure(cuda, sensitivity, basis, gain):
    """Very dark / very bright frames push the fp32 lead-in toward underflow,
    clamping and overflow (non-finite fp32 steps hand over the last finite
    state): fit counts must still equal the all-fp64 schedule's."""
    rgb = (synth.phantom_rgb_f32(96, 128, 21, sensitivity, basis) * gain).astype(np.float32).astype(np.float64)
    frames = rgb[None]
    _, ref, _ = _run(cuda, sensitivity, basis, frames, 2, None)
    _, out, _ = _run(cuda, sensitivity, basis, frames, 2, (16.0, 0.01))
    rt, rs, rf = _maps(ref)
    t, s, f = _maps(out)
    assert np.array_equal(f, rf)
    assert np.array_equal(np.isnan(s), np.isnan(rs))
    ok = np.isfinite(rt) & (np.abs(rt) > 0)
    assert np.max(np.abs(t[ok] - rt[ok]) / np.abs(rt[ok]), initial=0.0) < 1e-5
    oks = ~np.isnan(rs)
    assert np.max(np.abs(s[oks] - rs[oks]), initial=0.0) < 5e-6


def test_bench_configuration_vs_oracle(cuda, sensitivity, basis):
    """The bench's own workload (bench.py: DEFAULT_BATCH = 128 device-synthesised
    textured 1080p frames, n = 2) through the engine exactly as timed: 16.6 M low-pass
    coefficients, so the exact-block pass runs the one-lane persistent kernel
    over the selection list (kExactSeqMinN = 2^21).  One frame of each of the
    four truth maps, plus the last frame, against the pinned oracle: fit counts
    bit-exact, THb <= 1e-4 relative, SO2 <= 1e-5 absolute, NaN pattern
    identical; and every coefficient of the batch against the all-fp64 EM
    schedule (em_lead=None): 0 fit-count differences."""
    import bench

    B, H, W = bench.DEFAULT_BATCH, 1080, 1920
    frames = bench.make_frames(B, H, W, 0.3, 0, cuda)
    eng = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=2))
    out = eng.run(frames, fits=True)
    torch.cuda.synchronize()
    c = eng.em_counters(B, H, W)
    nll = out.fits.numel()
    assert nll >= 2**21 and c["exact_blocks"] > 0 and c["restarts"] > 0
    ref64 = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=2), em_lead=None).run(frames, fits=True)
    flips = int((ref64.fits != out.fits).sum())
    assert flips == 0, f"{flips} fit-count differences vs the all-fp64 schedule over {nll} coefficients"
    thb, so2, fits = out.thb.cpu().numpy(), out.so2.cpu().numpy(), out.fits.cpu().numpy()
    host = frames.cpu().numpy().astype(np.float64)
    for b in (0, 16, 32, 48, B - 1):
        ref = O.estimate_frame(host[b], sensitivity.c, basis.xi, n_levels=2, want_cube=False,
                               threads=O.default_threads())
        assert np.array_equal(fits[b], ref["fits"]), f"frame {b}: {np.sum(fits[b] != ref['fits'])} fit-count flips"
        assert np.array_equal(np.isnan(so2[b]), np.isnan(ref["so2"])), b
        assert np.all(np.abs(thb[b] - ref["thb"]) <= 1e-4 * np.abs(ref["thb"])), b
        ok = ~np.isnan(ref["so2"])
        assert np.max(np.abs(so2[b][ok] - ref["so2"][ok])) <= 1e-5, b


def test_schedule_knobs_and_debug_log(cuda, sensitivity, basis):
    """oxm_ctx_set_em_first_guard validates its arguments; the
    per-fit rel log of oxm_ctx_set_em_debug_log reproduces the stopping rule
    (bayes.py:199-205): for every coefficient of the all-fp64 schedule, rel of
    its last fit is < tol and every earlier logged rel is >= tol."""
    from paper_1706_07263_b200.device import ptr

    lib = _native.load()
    ok, bad = _native.OXM_OK, _native.OXM_ERR_ARGUMENT
    eng = ox.HybridMapEngine(sensitivity, basis, ox.PipelineConfig(n_levels=2), em_lead=None)
    h = eng.ctx.handle
    assert lib.oxm_ctx_set_em_first_guard(h, 0.1, 2) == ok
    assert lib.oxm_ctx_set_em_first_guard(h, 1.5, 2) == bad
    assert lib.oxm_ctx_set_em_first_guard(h, 0.1, 0) == bad
    rgb = synth.phantom_rgb_f32(96, 128, 17, sensitivity, basis)
    x = torch.from_numpy(rgb[None].astype(np.float32)).to(cuda)
    nll = 24 * 32
    rel = torch.zeros(nll * 24, dtype=torch.float32, device=cuda)
    step = torch.zeros(nll * 24, dtype=torch.uint8, device=cuda)
    assert lib.oxm_ctx_set_em_debug_log(h, ptr(rel), None) == bad
    assert lib.oxm_ctx_set_em_debug_log(h, ptr(rel), ptr(step)) == ok
    out = eng.run(x, fits=True)
    torch.cuda.synchronize()
    assert lib.oxm_ctx_set_em_debug_log(h, None, None) == ok
    fits = out.fits.reshape(-1).cpu().numpy()
    r = rel.reshape(nll, 24).cpu().numpy()
    assert np.all(step.cpu().numpy() == 0)  # all-fp64: every fit is on the exact trajectory
    for i in range(nll):
        m = fits[i]
        assert r[i, m] < 1e-4 * (1 + 1e-5), (i, m, r[i, m])
        assert np.all(r[i, 2:m] >= 1e-4 * (1 - 1e-5)), (i, r[i, :m + 1])
    ref = O.estimate_frame(rgb, sensitivity.c, basis.xi, n_levels=2, want_cube=False)
    assert np.array_equal(out.fits[0].cpu().numpy(), ref["fits"])


def test_engine_audit(cuda, sensitivity, basis, textured):
    """HybridMapEngine.audit: the runtime flip detector the bench line reports
    (parity.schedule) as a product API."""
    eng, out, _ = _run(cuda, sensitivity, basis, textured, 2, ox.engine.DEFAULT_EM_LEAD)
    x = torch.from_numpy(textured.astype(np.float32)).to(cuda)
    rep = eng.audit(x, out)
    assert rep["coefficients"] == out.fits.numel()
    assert rep["fit_count_flips"] == 0
    assert rep["so2_nan_pattern_equal"]
    assert rep["max_thb_rel"] < 1e-5 and rep["max_so2_abs"] < 5e-6
    # a flip is reported as one
    out.fits.view(-1)[7] += 1
    assert eng.audit(x, out)["fit_count_flips"] == 1
    with pytest.raises(ox.ArgumentError):
        eng.audit(x, eng.allocate(*textured.shape[:3]))
