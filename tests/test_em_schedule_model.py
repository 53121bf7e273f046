"""CPU model of the EM precision schedule (tools/mixed_em_study.py, NumPy):
fp32 lead-in with injected MUFU-sized noise while rel > K tol, fp64 tail with
the 1% guard band.  Checks the schedule's premise on the oracle's arithmetic
without a GPU: no unguarded fit-count difference, spectra within ~1e-6 of the
all-fp64 ones, and a guard band that catches only a few percent of
coefficients.  The GPU kernels are checked against the all-fp64 schedule and
the oracle in tests/test_gpu_em_schedule.py."""

from __future__ import annotations

import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))


def test_schedule_model_small_frame():
    import mixed_em_study as M

    from paper_1706_07263_b200 import fixtures, synth

    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    rgb = synth.phantom_rgb_f32(96, 128, 5, sens, basis)
    r = M.run(rgb, 1, 16.0, 0.01, 2.4e-7, np.random.default_rng(0))
    assert r["flips"] == 0
    assert r["guard_frac"] < 0.06
    assert r["S_rel_max"] < 1e-6
    assert r["fp32_steps"] > r["fp64_steps"]  # most fits run in the lead-in
