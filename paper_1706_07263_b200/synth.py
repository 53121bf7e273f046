"""Synthetic inputs: tissue phantoms -> reflectance cube -> RGB frames.

Input generation only (SURVEY §2 marks synth out of the hot-path scope); it
restates the reference generator (synth.py:28-184) with the same seeded draw
order, but renders the thousands of capillary-scale blobs in one vectorised
scatter-add instead of a Python loop per blob, so 1080p phantoms take about a
second.  ``device_frames`` runs the forward model, Philox noise and camera
projection in the oxm_synth_frames_f32 kernel to build large
benchmark batches on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from .core import CameraSensitivity, ChromophoreBasis, ConcentrationMap, RgbImage, SpectralCube, check_grids
from .errors import ArgumentError

REFLECTANCE_FLOOR = 1e-6  # synth.py:25


@dataclass(frozen=True)
class GaussianBlob:
    cx: float
    cy: float
    radius: float
    hbo: float
    hb: float

    def __post_init__(self):
        if self.radius <= 0:
            raise ArgumentError(f"blob radius must be > 0, got {self.radius}")


@dataclass(frozen=True)
class PhantomSpec:
    height: int
    width: int
    background: tuple[float, float] = (30.0, 30.0)
    blobs: tuple[GaussianBlob, ...] = ()
    illumination_offset: float = 0.0
    noise_sigma: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.height < 1 or self.width < 1:
            raise ArgumentError("phantom must be at least 1x1")
        if min(self.background) < 0:
            raise ArgumentError("background concentrations must be >= 0")
        if self.noise_sigma < 0:
            raise ArgumentError(f"noise_sigma must be >= 0, got {self.noise_sigma}")
        object.__setattr__(self, "blobs", tuple(self.blobs))


def tissue_phantom_spec(
    height: int,
    width: int,
    seed: int = 0,
    noise_sigma: float = 0.01,
    background: tuple[float, float] = (32.0, 28.0),
    n_features: int = 6,
    feature_amp: float = 10.0,
    texture_density: float = 0.3,
    texture_amp: float = 20.0,
) -> PhantomSpec:
    """Smooth perfusion features + balanced 2x2 capillary spike pairs
    (synth.py:97-147); identical seeded draws."""
    rng = np.random.default_rng(seed)
    blobs = []
    short = min(height, width)
    for _ in range(n_features):
        cx = rng.uniform(0.15, 0.85) * width
        cy = rng.uniform(0.15, 0.85) * height
        radius = rng.uniform(0.08, 0.2) * short
        a = rng.uniform(-feature_amp, feature_amp)
        b = rng.uniform(-feature_amp, feature_amp)
        blobs.append(GaussianBlob(cx, cy, radius, a, b))
    pairs = int(texture_density * (height // 2) * (width // 2))
    half_w, half_h = max(width // 2, 1), max(height // 2, 1)
    for _ in range(pairs):
        wx = int(rng.integers(0, half_w)) * 2
        wy = int(rng.integers(0, half_h)) * 2
        a = rng.uniform(-texture_amp, texture_amp)
        b = rng.uniform(-texture_amp, texture_amp)
        horizontal = rng.random() < 0.5
        x2, y2 = (wx + 1, wy) if horizontal else (wx, wy + 1)
        blobs.append(GaussianBlob(float(wx), float(wy), 0.45, a, b))
        blobs.append(GaussianBlob(float(x2), float(y2), 0.45, -a, -b))
    return PhantomSpec(height, width, background, tuple(blobs), noise_sigma=noise_sigma, seed=seed)


def _window(c: float, r: float, size: int) -> tuple[int, int]:
    lo = max(int(np.floor(c - 4 * r)), 0)
    hi = min(int(np.ceil(c + 4 * r)) + 1, size)
    return lo, hi


def truth_map(spec: PhantomSpec) -> ConcentrationMap:
    """Render the truth planes; each blob only inside its +-4 sigma window
    (synth.py:67-94).  Blobs are accumulated in list order."""
    H, W = spec.height, spec.width
    hbo = np.full((H, W), float(spec.background[0]))
    hb = np.full((H, W), float(spec.background[1]))
    blobs = spec.blobs
    i = 0
    while i < len(blobs):
        # maximal run of equal-radius blobs -> one vectorised scatter-add
        j = i
        while j < len(blobs) and blobs[j].radius == blobs[i].radius:
            j += 1
        run = blobs[i:j]
        if len(run) < 8:
            for blob in run:
                x0, x1 = _window(blob.cx, blob.radius, W)
                y0, y1 = _window(blob.cy, blob.radius, H)
                if x0 >= x1 or y0 >= y1:
                    continue
                yy, xx = np.mgrid[y0:y1, x0:x1]
                bump = np.exp(-0.5 * ((xx - blob.cx) ** 2 + (yy - blob.cy) ** 2) / blob.radius**2)
                hbo[y0:y1, x0:x1] += blob.hbo * bump
                hb[y0:y1, x0:x1] += blob.hb * bump
        else:
            r = run[0].radius
            cx = np.array([b.cx for b in run])
            cy = np.array([b.cy for b in run])
            ah = np.array([b.hbo for b in run])
            ab = np.array([b.hb for b in run])
            k = int(np.ceil(4 * r)) + 2
            off = np.arange(-k, k + 1)
            xs = np.floor(cx - 4 * r).astype(np.int64)[:, None] + (off + k)[None, :]
            ys = np.floor(cy - 4 * r).astype(np.int64)[:, None] + (off + k)[None, :]
            x_lo = np.maximum(np.floor(cx - 4 * r), 0)[:, None]
            x_hi = np.minimum(np.ceil(cx + 4 * r) + 1, W)[:, None]
            y_lo = np.maximum(np.floor(cy - 4 * r), 0)[:, None]
            y_hi = np.minimum(np.ceil(cy + 4 * r) + 1, H)[:, None]
            okx = (xs >= x_lo) & (xs < x_hi)
            oky = (ys >= y_lo) & (ys < y_hi)
            YY = np.broadcast_to(ys[:, :, None], (len(run), xs.shape[1], xs.shape[1]))
            XX = np.broadcast_to(xs[:, None, :], YY.shape)
            ok = oky[:, :, None] & okx[:, None, :]
            bump = np.exp(-0.5 * ((XX - cx[:, None, None]) ** 2 + (YY - cy[:, None, None]) ** 2) / r**2)
            flat = (YY * W + XX)[ok]
            np.add.at(hbo.reshape(-1), flat, (ah[:, None, None] * bump)[ok])
            np.add.at(hb.reshape(-1), flat, (ab[:, None, None] * bump)[ok])
        i = j
    offset = np.full((H, W), float(spec.illumination_offset))
    return ConcentrationMap(hbo=np.clip(hbo, 0.0, None), hb=np.clip(hb, 0.0, None), offset=offset)


def forward_msi(truth: ConcentrationMap, basis: ChromophoreBasis) -> SpectralCube:
    """I = exp(-xi x) per pixel (synth.py:150-153)."""
    return SpectralCube(grid=basis.grid, data=np.exp(-(truth.stacked() @ basis.xi.T)))


def synthesize_rgb(cube: SpectralCube, sensitivity: CameraSensitivity, exposure: float = 1.0) -> RgbImage:
    """y = exposure * C i (synth.py:156-163)."""
    if exposure <= 0:
        raise ArgumentError(f"exposure must be > 0, got {exposure}")
    check_grids(cube.grid, sensitivity.grid)
    return RgbImage(data=exposure * (cube.data @ sensitivity.c.T))


def generate_phantom(
    spec: PhantomSpec, sensitivity: CameraSensitivity, basis: ChromophoreBasis, exposure: float = 1.0
) -> tuple[ConcentrationMap, SpectralCube, RgbImage]:
    """Truth, noisy cube (floored) and its RGB view (synth.py:166-184)."""
    truth = truth_map(spec)
    cube = forward_msi(truth, basis)
    if spec.noise_sigma > 0:
        rng = np.random.default_rng(spec.seed)
        noisy = cube.data + rng.normal(0.0, spec.noise_sigma, size=cube.data.shape)
        cube = SpectralCube(grid=cube.grid, data=np.clip(noisy, REFLECTANCE_FLOOR, None))
    return truth, cube, synthesize_rgb(cube, sensitivity, exposure)


def _check_pulse(fps: float, pulse_hz: float, amplitude: float) -> None:
    """synth.py:209-216 argument checks (duration checked by the caller)."""
    if fps <= 0:
        raise ArgumentError(f"fps must be > 0, got {fps}")
    if not 0 < pulse_hz < fps / 2:
        raise ArgumentError(f"pulse_hz must satisfy 0 < pulse_hz < fps/2 = {fps / 2:g}, got {pulse_hz}")
    if amplitude < 0:
        raise ArgumentError(f"amplitude must be >= 0, got {amplitude}")


def pulse_modulation(t: int, fps: float, pulse_hz: float, amplitude: float) -> float:
    """Frame t's haemoglobin scale 1 + a sin(2 pi f t / fps) (synth.py:218)."""
    return 1.0 + amplitude * math.sin(2.0 * math.pi * pulse_hz * t / fps)


def pulse_sequence(
    spec: PhantomSpec,
    fps: float,
    duration_s: float,
    pulse_hz: float,
    amplitude: float,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    exposure: float = 1.0,
) -> Iterator[RgbImage]:
    """Frames whose THb truth is modulated by a sinusoidal pulse
    (synth.py:187-231): frame t scales hbo and hb by 1 + a sin(2 pi f t/fps),
    then forward model, per-frame reflectance noise (the reference's seeded
    draw order, so frames are bit-identical to it) and RGB synthesis.  Host
    input generator, like generate_phantom; ``device_pulse_frames`` renders
    the same sequence on the GPU for long videos."""
    if fps <= 0:
        raise ArgumentError(f"fps must be > 0, got {fps}")
    if duration_s <= 0:
        raise ArgumentError(f"duration_s must be > 0, got {duration_s}")
    _check_pulse(fps, pulse_hz, amplitude)
    truth = truth_map(spec)
    n_frames = int(round(duration_s * fps))
    rng = np.random.default_rng(spec.seed)
    for t in range(n_frames):
        m = pulse_modulation(t, fps, pulse_hz, amplitude)
        cube = forward_msi(ConcentrationMap(hbo=truth.hbo * m, hb=truth.hb * m, offset=truth.offset), basis)
        data = cube.data
        if spec.noise_sigma > 0:
            data = np.clip(data + rng.normal(0.0, spec.noise_sigma, size=data.shape), REFLECTANCE_FLOOR, None)
        yield synthesize_rgb(SpectralCube(grid=cube.grid, data=data), sensitivity, exposure)


def phantom_rgb_f32(
    height: int,
    width: int,
    seed: int,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    *,
    texture_density: float = 0.3,
    noise_sigma: float = 0.01,
) -> np.ndarray:
    """An fp32-exact (H, W, 3) float64 phantom frame: the values both the GPU
    (as float32) and the oracle (as float64) see, so parity compares like
    with like (SURVEY §8c tolerance protocol)."""
    spec = tissue_phantom_spec(height, width, seed=seed, noise_sigma=noise_sigma, texture_density=texture_density)
    _, _, rgb = generate_phantom(spec, sensitivity, basis)
    return rgb.data.astype(np.float32).astype(np.float64)


def device_frames(
    truth: ConcentrationMap,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    count: int,
    *,
    noise_sigma: float = 0.01,
    seed: int = 0,
    frame0: int = 0,
    exposure: float = 1.0,
    device=None,
):
    """(count, H, W, 3) float32 CUDA frames of one truth map, generated by the
    oxm_synth_frames_f32 kernel: forward model, Philox reflectance noise floored
    at REFLECTANCE_FLOOR, camera projection (synth.py:150-184).  Frame k uses
    noise stream index frame0 + k, so long videos can be generated in chunks."""
    import torch

    from . import _native
    from .device import ptr, stream_handle
    from .operators import context, make_operator_set

    return device_pulse_frames(truth, sensitivity, basis, count, noise_sigma=noise_sigma, seed=seed, frame0=frame0,
                               exposure=exposure, device=device)


def device_pulse_frames(
    truth: ConcentrationMap,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    count: int,
    *,
    fps: float = 1.0,
    pulse_hz: float = 0.0,
    amplitude: float = 0.0,
    noise_sigma: float = 0.01,
    seed: int = 0,
    frame0: int = 0,
    exposure: float = 1.0,
    device=None,
):
    """pulse_sequence on the device (synth.py:187-231, oxm_synth_pulse_frames_f32):
    frames frame0 .. frame0 + count - 1 of the pulse-modulated sequence of
    ``truth`` as a (count, H, W, 3) float32 CUDA tensor.  The per-frame scale
    1 + a sin(2 pi f t / fps) is the reference's; the noise is the kernel's
    counter-based Philox stream (statistically, not bitwise, the reference's).
    amplitude 0 gives static phantom frames (device_frames)."""
    import torch

    from . import _native
    from .device import ptr, stream_handle
    from .operators import context, make_operator_set

    check_grids(sensitivity.grid, basis.grid)
    if amplitude != 0.0:
        _check_pulse(fps, pulse_hz, amplitude)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    ops = make_operator_set(n_bands=basis.grid.count, xi=basis.xi, sens=sensitivity.c)
    ctx = context(ops, dev.index)
    x = torch.from_numpy(np.ascontiguousarray(truth.stacked(), dtype=np.float32)).to(dev)
    H, W = truth.hbo.shape
    out = torch.empty((count, H, W, 3), dtype=torch.float32, device=dev)
    st = _native.load().oxm_synth_pulse_frames_f32(ctx.handle, ptr(x), H, W, count, float(noise_sigma),
                                                   float(exposure), int(seed) & (2**64 - 1), int(frame0), float(fps),
                                                   float(pulse_hz), float(amplitude), ptr(out), stream_handle())
    _native.check(st, "synth_pulse_frames")
    return out
