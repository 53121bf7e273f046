"""The drop-in name set and the reference's off-path host API (metrics,
pulse analysis, pulse_sequence), pinned against tests/golden/api.npz made by
running the reference (tools/make_golden_api.py).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1706_07263_b200 as ox
from paper_1706_07263_b200 import synth, timeseries


def test_reference_names_importable(golden):
    ref_names = set(str(n) for n in golden("api")["all_names"])
    assert ref_names <= set(ox.__all__), sorted(ref_names - set(ox.__all__))
    for name in ref_names:
        assert hasattr(ox, name), name


def test_concentration_mse_matches_reference(golden):
    g = golden("api")
    a, b = ox.ConcentrationMap.from_stacked(g["mse_a"]), ox.ConcentrationMap.from_stacked(g["mse_b"])
    for tag, m in (("full", None), ("masked", g["mse_mask"])):
        r = ox.concentration_mse(a, b, m)
        assert np.array_equal(np.array([r.mse, r.rmse, r.mse_hbo, r.mse_hb, r.n_pixels], dtype=np.float64),
                              g[f"mse_{tag}"])
    with pytest.raises(ox.ArgumentError, match="no pixels"):
        ox.concentration_mse(a, b, np.zeros((20, 30), dtype=bool))
    with pytest.raises(ox.ArgumentError, match="boolean"):
        ox.concentration_mse(a, b, np.ones((20, 30)))
    small = ox.ConcentrationMap.from_stacked(g["mse_a"][:5])
    with pytest.raises(ox.ArgumentError, match="dimensions differ"):
        ox.concentration_mse(a, small)


def test_pulse_analysis_matches_reference(golden):
    g = golden("api")
    tr = ox.Trace(fps=30.0, values=g["trace"])
    der = timeseries.smooth_derivative(tr, 0.4)
    assert np.array_equal(der.values, g["deriv"])
    assert np.array_equal(np.array(ox.dominant_frequency(der)), g["dom_mean"])
    assert np.array_equal(np.array(ox.dominant_frequency(tr, (0.6, 3.0), "linear")), g["dom_linear"])
    with pytest.raises(ox.ArgumentError, match="Nyquist"):
        ox.dominant_frequency(tr, (0.6, 15.0))
    with pytest.raises(ox.ArgumentError, match="detrend"):
        ox.dominant_frequency(tr, detrend="cubic")
    with pytest.raises(ox.ArgumentError):
        ox.Trace(fps=0.0, values=[1.0])
    rep = ox.PulseReport(trace=tr, derivative=der, peak_hz=1.25, power_fraction=0.5)
    assert rep.bpm == 75.0


def test_pulse_sequence_matches_reference(golden, sensitivity, basis):
    g = golden("api")
    for tag, sigma in (("noisy", 0.01), ("clean", 0.0)):
        spec = ox.tissue_phantom_spec(24, 32, seed=5, noise_sigma=sigma, texture_density=0.3)
        frames = np.stack([f.data for f in ox.pulse_sequence(spec, 30.0, 0.2, 1.2, 0.1, sensitivity, basis)])
        assert np.array_equal(frames, g[f"pulse_{tag}"]), tag
    spec = ox.tissue_phantom_spec(8, 8, seed=1)
    for kw in (dict(fps=0.0), dict(pulse_hz=20.0), dict(amplitude=-0.1), dict(duration_s=0.0)):
        args = dict(fps=30.0, duration_s=1.0, pulse_hz=1.0, amplitude=0.1)
        args.update(kw)
        with pytest.raises(ox.ArgumentError):
            next(ox.pulse_sequence(spec, args["fps"], args["duration_s"], args["pulse_hz"], args["amplitude"],
                                   sensitivity, basis))
    assert synth.pulse_modulation(0, 30.0, 1.0, 0.2) == 1.0
