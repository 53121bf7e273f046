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


def test_ppm_to_spc1_files(cuda, tmp_path, sensitivity, basis):
    """GPU-native `oximap estimate`: PPM written in the reference format ->
    SPC1 maps, compared with the oracle on the decoded frame."""
    from oracle import oximap_oracle as O
    from paper_1706_07263_b200.io import estimate_files, read_ppm_raw

    rgb = synth.phantom_rgb_f32(72, 100, 5, sensitivity, basis)
    scale = float(rgb.max()) / 65535.0
    counts = np.clip(np.round(rgb / scale), 0, 65535).astype(">u2")
    src = tmp_path / "f.ppm"
    src.write_bytes(f"P6\n# scale {scale!r}\n100 72\n65535\n".encode("ascii") + counts.tobytes())
    raw, sc = read_ppm_raw(src)
    assert sc == scale and raw.shape == (72, 100, 3)
    dst = tmp_path / "m.spc"
    assert estimate_files([src], [dst], sensitivity, basis, ox.PipelineConfig(n_levels=2)) == 1
    buf = dst.read_bytes()
    header, payload = buf.split(b"\n", 1)
    assert header.split() == [b"SPC1", b"72", b"100", b"3", b"0.0", b"1.0"]
    maps = np.frombuffer(payload, dtype="<f4").reshape(72, 100, 3).astype(np.float64)
    ref = O.estimate_frame(counts.astype(np.float64) * scale, sensitivity.c, basis.xi, n_levels=2)
    assert np.max(np.abs(maps[..., :2] - ref["x"][..., :2])) <= 1e-4 * np.max(np.abs(ref["x"][..., :2]))
    with pytest.raises(ox.DataError):
        bad = tmp_path / "b.ppm"
        bad.write_bytes(b"P6\n100 72\n255\n" + b"\0" * 10)
        read_ppm_raw(bad)


def test_device_pulse_frames_match_pulse_sequence(cuda, golden, sensitivity, basis):
    """Device pulse_sequence (oxm_synth_pulse_frames_f32) without noise equals
    the reference's noise-free pulse_sequence frames (golden) to fp32 rounding
    of the forward model; frame0 offsets the pulse phase like frame index t."""
    g = golden("api")
    ref = g["pulse_clean"]
    spec = ox.tissue_phantom_spec(24, 32, seed=5, noise_sigma=0.0, texture_density=0.3)
    truth = synth.truth_map(spec)
    dev = synth.device_pulse_frames(truth, sensitivity, basis, ref.shape[0], fps=30.0, pulse_hz=1.2, amplitude=0.1,
                                    noise_sigma=0.0, device=cuda).double().cpu().numpy()
    assert np.max(np.abs(dev - ref) / np.abs(ref)) < 2e-5
    tail = synth.device_pulse_frames(truth, sensitivity, basis, 2, fps=30.0, pulse_hz=1.2, amplitude=0.1,
                                     noise_sigma=0.0, frame0=3, device=cuda).double().cpu().numpy()
    assert np.max(np.abs(tail - ref[3:5]) / np.abs(ref[3:5])) < 2e-5
    # the modulation is what moves THb: frames differ from the static phantom
    static = synth.device_frames(truth, sensitivity, basis, 1, noise_sigma=0.0, device=cuda).double().cpu().numpy()
    assert np.max(np.abs(dev[1] - static[0])) > 1e-3
    with pytest.raises(ox.ArgumentError):
        synth.device_pulse_frames(truth, sensitivity, basis, 1, fps=30.0, pulse_hz=16.0, amplitude=0.1, device=cuda)


def test_analyze_pulse_matches_reference(cuda, golden):
    """analyze_pulse with the patch mean on the device (fp32 THb) against the
    reference's all-host report: trace to fp32 rounding, same peak."""
    g = golden("api")
    maps = []
    for k in range(90):
        m = 1.0 + 0.05 * np.sin(2 * np.pi * 1.1 * k / 30.0)
        maps.append(ox.ConcentrationMap(hbo=g["ap_hbo"] * m, hb=g["ap_hb"] * m, offset=g["ap_off"]))
    rep = ox.analyze_pulse(maps, (4, 4, 16, 16), 30.0)
    assert np.max(np.abs(rep.trace.values - g["ap_trace"]) / g["ap_trace"]) < 1e-6
    assert abs(rep.peak_hz - g["ap_peak"][0]) < 1e-3 and abs(rep.bpm - g["ap_peak"][2]) < 0.06
