#!/usr/bin/env python3
"""Generate tests/golden/api.npz by running the REFERENCE's off-path public
API (metrics, timeseries pulse analysis, pulse_sequence) and recording its
__all__, so the drop-in name set and these host functions are pinned on a box
without /root/reference.  Build container only:  python tools/make_golden_api.py
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parents[1] / "tests" / "golden" / "api.npz"


def main() -> None:
    sys.path.insert(0, str(REF))
    import oximap
    from oximap import fixtures, synth, timeseries
    from oximap.core import ConcentrationMap
    from oximap.metrics import concentration_mse

    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    rng = np.random.default_rng(7)
    g = {"all_names": np.array(sorted(oximap.__all__))}

    # metrics.concentration_mse (metrics.py:29-58), with and without a mask
    a = ConcentrationMap(hbo=rng.normal(40, 5, (20, 30)), hb=rng.normal(30, 5, (20, 30)), offset=rng.normal(0, 1, (20, 30)))
    b = ConcentrationMap(hbo=rng.normal(40, 5, (20, 30)), hb=rng.normal(30, 5, (20, 30)), offset=rng.normal(0, 1, (20, 30)))
    mask = rng.random((20, 30)) < 0.4
    g["mse_a"], g["mse_b"], g["mse_mask"] = a.stacked(), b.stacked(), mask
    for tag, m in (("full", None), ("masked", mask)):
        r = concentration_mse(a, b, m)
        g[f"mse_{tag}"] = np.array([r.mse, r.rmse, r.mse_hbo, r.mse_hb, r.n_pixels], dtype=np.float64)

    # timeseries: smooth_derivative / dominant_frequency on a noisy pulse trace
    fps = 30.0
    t = np.arange(300) / fps
    vals = 60 + 2.0 * np.sin(2 * np.pi * 1.3 * t) + 0.3 * rng.normal(size=t.size) + 0.5 * t
    tr = timeseries.Trace(fps=fps, values=vals)
    der = timeseries.smooth_derivative(tr, 0.4)
    g["trace"], g["deriv"] = vals, der.values
    g["dom_mean"] = np.array(timeseries.dominant_frequency(der))
    g["dom_linear"] = np.array(timeseries.dominant_frequency(tr, (0.6, 3.0), "linear"))

    # pulse_sequence (synth.py:187-231): noisy (seeded draws) and noise-free
    for tag, sigma in (("noisy", 0.01), ("clean", 0.0)):
        spec = synth.tissue_phantom_spec(24, 32, seed=5, noise_sigma=sigma, texture_density=0.3)
        frames = list(synth.pulse_sequence(spec, 30.0, 0.2, 1.2, 0.1, sens, basis))
        g[f"pulse_{tag}"] = np.stack([f.data for f in frames])

    # analyze_pulse on a map sequence (the GPU test runs its patch mean on the device)
    spec = synth.tissue_phantom_spec(32, 40, seed=9, noise_sigma=0.0, texture_density=0.0)
    truth = synth.truth_map(spec) if hasattr(synth, "truth_map") else synth.generate_phantom(spec, sens, basis)[0]
    maps = []
    for k in range(90):
        m = 1.0 + 0.05 * np.sin(2 * np.pi * 1.1 * k / 30.0)
        maps.append(ConcentrationMap(hbo=truth.hbo * m, hb=truth.hb * m, offset=truth.offset))
    rep = timeseries.analyze_pulse(maps, (4, 4, 16, 16), 30.0)
    g["ap_hbo"], g["ap_hb"], g["ap_off"] = truth.hbo, truth.hb, truth.offset  # maps rebuilt as above in the test
    g["ap_trace"], g["ap_deriv"] = rep.trace.values, rep.derivative.values
    g["ap_peak"] = np.array([rep.peak_hz, rep.power_fraction, rep.bpm])
    np.savez_compressed(OUT, **g)
    print(f"{OUT.name}: {OUT.stat().st_size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
