"""§8f helpers on the GPU: device synth frames and the patch-mean trace."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1706_07263_b200 as ox
from paper_1706_07263_b200 import synth
from paper_1706_07263_b200.timeseries import patch_mean, patch_means_device

pytestmark = pytest.mark.gpu


def test_device_synth_noise_free_matches_forward_model(cuda, sensitivity, basis):
    spec = synth.tissue_phantom_spec(64, 80, seed=3, noise_sigma=0.0)
    truth = synth.truth_map(spec)
    got = synth.device_frames(truth, sensitivity, basis, 2, noise_sigma=0.0).cpu().numpy()
    want = synth.synthesize_rgb(synth.forward_msi(truth, basis), sensitivity).data
    assert np.max(np.abs(got[0] - want) / want) <= 2e-5
    assert np.array_equal(got[0], got[1])


def test_device_synth_noise_statistics_and_streams(cuda, sensitivity, basis):
    H, W = 256, 256
    flat = ox.ConcentrationMap(hbo=np.full((H, W), 30.0), hb=np.full((H, W), 20.0), offset=np.zeros((H, W)))
    sigma = 0.01
    a = synth.device_frames(flat, sensitivity, basis, 4, noise_sigma=sigma, seed=7)
    b = synth.device_frames(flat, sensitivity, basis, 2, noise_sigma=sigma, seed=7, frame0=2)
    assert torch.equal(a[2:], b)                      # counter-based: frame k is frame0 + k
    assert not torch.equal(a[0], a[1])
    clean = synth.device_frames(flat, sensitivity, basis, 1, noise_sigma=0.0)[0]
    resid = (a - clean).double().cpu().numpy().reshape(-1, 3)
    expect = sigma * np.sqrt((sensitivity.c ** 2).sum(axis=1))
    assert np.allclose(resid.std(axis=0), expect, rtol=0.02)
    assert np.all(np.abs(resid.mean(axis=0)) < 0.01 * expect)


def test_patch_mean(cuda, rng):
    thb = rng.uniform(5, 80, size=(5, 40, 60)).astype(np.float32)
    thb[1, 10:20, 5:9] = np.nan
    thb[3] = np.nan  # frame without a valid pixel -> interpolated
    rect = (3, 7, 20, 15)
    x, y, w, h = rect
    got = patch_means_device(torch.from_numpy(thb).to(cuda), rect)
    for f in range(5):
        p = thb[f, y:y + h, x:x + w].astype(np.float64)
        v = p[np.isfinite(p)]
        if v.size:
            assert got[f] == pytest.approx(v.mean(), rel=1e-12)
        else:
            assert np.isnan(got[f])
    tr = patch_mean(torch.from_numpy(thb).to(cuda), rect, fps=25.0)
    assert tr.values[3] == pytest.approx(0.5 * (tr.values[2] + tr.values[4]))
    maps = [ox.ConcentrationMap(hbo=np.nan_to_num(t, nan=-1.0), hb=np.zeros_like(t), offset=np.zeros_like(t))
            for t in thb[:3]]
    tr2 = patch_mean(maps, rect, fps=25.0)
    assert len(tr2) == 3
    with pytest.raises(ox.ArgumentError):
        patch_means_device(torch.from_numpy(thb).to(cuda), (50, 0, 20, 5))
