"""End-to-end frame estimators -- drop-in for oximap.pipeline (pipeline.py:1-245).

``estimate_frame(mode="hybrid")`` is the north-star hot path.  Here it runs
the fused K6 kernels (``oxm_hybrid_frame_f64``): fp64 low-pass chain, fp64
EM, and an fp64 per-pixel reconstruction + fit that also materialises the
(H, W, L) SpectralCube the API returns.  The throughput path for video
batches (fp32 maps, no cube) is ``engine.HybridMapEngine``.

The other modes reuse the same kernels: ``tikhonov_only`` = K3 + K5,
``bayes_only`` = K4 at full resolution + K5, ``direct_msi`` = K5.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import Iterable, Iterator

import numpy as np
import torch

from . import _native
from .bayes import BayesConfig, LowPassBlock, em_device, em_operator_set, fit_device
from .core import (
    CameraSensitivity,
    ChromophoreBasis,
    ConcentrationMap,
    RgbImage,
    SpectralCube,
    check_grids,
    trusted_cube,
    trusted_map,
)
from .device import download, ptr, require_cuda, stream_handle, upload
from .errors import ArgumentError, DataError
from .haar import level_dims
from .operators import OperatorSet, context, make_operator_set
from .unmix import TikhonovOperator, apply_matrix_device

MODES = ("hybrid", "tikhonov_only", "bayes_only", "direct_msi")


@dataclass(frozen=True)
class PipelineConfig:
    """Pipeline knobs (pipeline.py:44-63); ``threads`` is accepted and ignored
    by the GPU path."""

    mode: str = "hybrid"
    n_levels: int = 1
    tikhonov_gamma: float = 1e-3  # relative: scaled by trace(C^T C) / L
    bayes: BayesConfig = field(default_factory=BayesConfig)
    threads: int = 1
    calibration_scale: float = 1.0

    def __post_init__(self):
        if self.mode not in MODES:
            raise ArgumentError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.n_levels < 1:
            raise ArgumentError(f"n_levels must be >= 1, got {self.n_levels}")
        if not self.tikhonov_gamma > 0:
            raise ArgumentError(f"tikhonov_gamma must be > 0, got {self.tikhonov_gamma}")
        if self.threads < 1:
            raise ArgumentError(f"threads must be >= 1, got {self.threads}")
        if not self.calibration_scale > 0:
            raise ArgumentError(f"calibration_scale must be > 0, got {self.calibration_scale}")


def _map_from_planes(x: np.ndarray, h: int, w: int) -> ConcentrationMap:
    return ConcentrationMap(hbo=x[:, 0].reshape(h, w), hb=x[:, 1].reshape(h, w), offset=x[:, 2].reshape(h, w))


def fit_cube(
    cube: SpectralCube,
    basis: ChromophoreBasis,
    *,
    epsilon: float = 1e-6,
    calibration_scale: float = 1.0,
    threads: int = 1,
) -> ConcentrationMap:
    """Per-pixel Beer-Lambert fit (pipeline.py:66-94) on the GPU (K5, fp64)."""
    del threads
    check_grids(cube.grid, basis.grid)
    h, w, L = cube.data.shape
    if h * w == 0:
        z = np.zeros((h, w))
        return ConcentrationMap(hbo=z, hb=z, offset=z)
    ops = make_operator_set(n_bands=L, xi=basis.xi, epsilon=epsilon)
    x = fit_device(upload(cube.data.reshape(-1, L), torch.float64, require_cuda()), ops, calibration_scale)
    return _map_from_planes(download(x), h, w)


def hybrid_device(
    frames: torch.Tensor,
    ops: OperatorSet,
    n_levels: int,
    calibration: float,
    *,
    want_cube: bool = True,
    stream=None,
) -> dict:
    """K6 (fp64) on a device batch (B, H, W, 3) float64.  Returns device
    tensors cube (B, H, W, L) | None, x (3, B, H, W), fits (B, hL, wL).
    Raises ArgumentError on size / negative low-pass like pipeline.py:177-193."""
    lib = _native.load()
    frames = frames.contiguous()
    B, H, W, _ = frames.shape
    if H < 2**n_levels or W < 2**n_levels:
        raise ArgumentError(f"frame {H}x{W} is smaller than 2^{n_levels} in one dimension")
    hL, wL = level_dims(H, W, n_levels)[-1]
    L = ops.n_bands
    dev = frames.device
    ctx = context(ops, dev.index)
    ws_bytes = int(lib.oxm_hybrid_workspace_bytes(ctx.handle, B, H, W, n_levels))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    cube = torch.empty((B, H, W, L), dtype=torch.float64, device=dev) if want_cube else None
    x = torch.empty((3, B, H, W), dtype=torch.float64, device=dev)
    fits = torch.empty((B, hL, wL), dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = lib.oxm_hybrid_frame_f64(
        ctx.handle, ptr(frames), B, H, W, n_levels, float(calibration), ptr(ws), ws_bytes,
        ptr(cube), ptr(x[0]), ptr(x[1]), ptr(x[2]), ptr(fits), ptr(flags), stream_handle(stream), None,
    )
    _native.check(st, "hybrid_frame_f64")
    f = int(flags.item())
    if f & _native.FLAG_NONFINITE:
        raise ArgumentError("image contains non-finite values")
    if f & _native.FLAG_NEGATIVE_LL:
        raise ArgumentError("low-pass coefficients must be finite and non-negative")
    return {"cube": cube, "x": x, "fits": fits}


def _hybrid_operators(sensitivity, basis, cfg: PipelineConfig) -> OperatorSet:
    op = TikhonovOperator.from_relative(sensitivity, cfg.tikhonov_gamma)
    return em_operator_set(sensitivity, basis, cfg.bayes, op)


def estimate_frame(
    frame: RgbImage | SpectralCube,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: PipelineConfig,
    stats: dict | None = None,
) -> tuple[SpectralCube, ConcentrationMap]:
    """Surrogate spectral cube + concentration map of one frame
    (pipeline.py:117-217)."""
    check_grids(sensitivity.grid, basis.grid)
    if stats is not None:
        stats.clear()
    grid = sensitivity.grid
    L = grid.count
    eps, cal = cfg.bayes.epsilon, cfg.calibration_scale

    if cfg.mode == "direct_msi":
        if not isinstance(frame, SpectralCube):
            raise ArgumentError("direct_msi mode takes a SpectralCube frame")
        check_grids(frame.grid, basis.grid)
        cmap = fit_cube(frame, basis, epsilon=eps, calibration_scale=cal)
        if stats is not None:
            stats.update(bayes_coefficients=0, tikhonov_coefficients=0)
        return frame, cmap

    if not isinstance(frame, RgbImage):
        raise ArgumentError(f"{cfg.mode} mode takes an RgbImage frame")
    H, W = frame.height, frame.width
    dev = require_cuda()

    if cfg.mode == "bayes_only":
        LowPassBlock(rgb_lp=frame.data, scale=1.0)  # same non-negativity contract (bayes.py:77-78)
        ops = _hybrid_operators(sensitivity, basis, cfg)
        spectra, _, _ = em_device(upload(frame.data.reshape(-1, 3), torch.float64, dev), ops)
        x = fit_device(spectra, ops, cal)
        cube = SpectralCube(grid=grid, data=download(spectra).reshape(H, W, L))
        if stats is not None:
            stats.update(bayes_coefficients=H * W, tikhonov_coefficients=0)
        return cube, _map_from_planes(download(x), H, W)

    if H < 2**cfg.n_levels or W < 2**cfg.n_levels:
        raise ArgumentError(f"frame {H}x{W} is smaller than 2^{cfg.n_levels} in one dimension")
    dims = level_dims(H, W, cfg.n_levels)
    n_lp = dims[-1][0] * dims[-1][1]
    n_dir = 3 * sum(h * w for h, w in dims)

    if cfg.mode == "tikhonov_only":
        # linear end to end: transform -> unmix -> inverse == per-pixel unmix
        op = TikhonovOperator.from_relative(sensitivity, cfg.tikhonov_gamma)
        ops = make_operator_set(n_bands=L, xi=basis.xi, epsilon=eps)
        spec = apply_matrix_device(upload(frame.data.reshape(-1, 3), torch.float64, dev), op.solve)
        x = fit_device(spec, ops, cal)
        cube = SpectralCube(grid=grid, data=download(spec).reshape(H, W, L))
        if stats is not None:
            stats.update(bayes_coefficients=0, tikhonov_coefficients=n_lp + n_dir)
        return cube, _map_from_planes(download(x), H, W)

    # hybrid (outputs come straight from the kernels: no host-side re-validation)
    ops = _hybrid_operators(sensitivity, basis, cfg)
    out = hybrid_device(upload(frame.data[None], torch.float64, dev), ops, cfg.n_levels, cal)
    cube = trusted_cube(grid, _download_large(out["cube"][0]))
    xs = _download_large(out["x"][:, 0])
    cmap = trusted_map(xs[0], xs[1], xs[2])
    if stats is not None:
        stats.update(bayes_coefficients=n_lp, tikhonov_coefficients=n_dir)
    return cube, cmap


def estimate_sequence(
    frames: Iterable[RgbImage],
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: PipelineConfig,
    timings: list | None = None,
) -> Iterator[ConcentrationMap]:
    """Stream maps for a frame sequence (pipeline.py:220-245).

    Hybrid RgbImage sequences are pipelined over two slots: while map i is
    copied back and handed out, frame i+1 is already uploaded and running
    (K6 fp64, workspaces reused, one stream per slot), so the sequence is
    bound by host copies and PCIe, not by the kernels.  Frame i+1 is read from
    the iterator before map i is yielded; errors keep the reference's order
    (a dimension change or bad frame raises after every earlier map has been
    yielded).  ``timings`` gets, per frame, the wall-clock seconds the
    pipeline spent on it (from its submission, or from the previous map being
    ready if later, until its map is ready)."""
    if cfg.mode != "hybrid":
        yield from _sequence_plain(frames, sensitivity, basis, cfg, timings)
        return
    runner = None
    pending: list = []
    last_ready = None
    shape = None

    def finish(job):
        nonlocal last_ready
        cmap, t_sub = runner.collect(job)
        t = time.perf_counter()
        if timings is not None:
            timings.append(t - max(t_sub, last_ready if last_ready is not None else t_sub))
        last_ready = t
        return cmap

    for frame in frames:
        dims = (frame.height, frame.width)
        if shape is None:
            shape = dims
        if dims != shape or not isinstance(frame, RgbImage):
            while pending:
                yield finish(pending.pop(0))
            if dims != shape:
                raise DataError(f"frame dimensions changed mid-stream: {shape} -> {dims}")
            yield estimate_frame(frame, sensitivity, basis, cfg)[1]  # raises the reference's error
            continue
        if runner is None:
            runner = _SequenceRunner(sensitivity, basis, cfg, dims)
        if len(pending) == 2:
            yield finish(pending.pop(0))
        pending.append(runner.submit(frame))
    while pending:
        yield finish(pending.pop(0))


def _sequence_plain(frames, sensitivity, basis, cfg, timings):
    shape = None
    for frame in frames:
        dims = (frame.height, frame.width)
        if shape is None:
            shape = dims
        elif dims != shape:
            raise DataError(f"frame dimensions changed mid-stream: {shape} -> {dims}")
        t0 = time.perf_counter()
        cmap = estimate_frame(frame, sensitivity, basis, cfg)[1]
        if timings is not None:
            timings.append(time.perf_counter() - t0)
        yield cmap


_COPY_POOL = None


def _copy_threads() -> int:
    """Host copy threads: OXM_COPY_THREADS, default min(8, cores / 2) (on a
    16-core B200 host: 2 / 4 / 8 / 16 threads gave 144 / 223 / 263 / 233
    estimate_sequence frames/s, tools/seq_probe.py)."""
    import os

    default = max(2, min(8, (os.cpu_count() or 4) // 2))
    try:
        return max(1, int(os.environ.get("OXM_COPY_THREADS", default)))
    except ValueError:
        return default


def _copy_pool():
    global _COPY_POOL
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _COPY_POOL = ThreadPoolExecutor(max_workers=_copy_threads(), thread_name_prefix="oxm-copy")
    return _COPY_POOL


def _par_copy(pairs) -> None:
    """np.copyto for (dst, src) pairs, each split by rows over a small thread
    pool (NumPy releases the GIL for large copies): the host-side memcpys of
    50 MB frames and maps are what bound estimate_sequence."""
    jobs = []
    for dst, src in pairs:
        rows = dst.shape[0]
        step = max(1, -(-rows // _copy_threads()))
        for r in range(0, rows, step):
            jobs.append(_copy_pool().submit(np.copyto, dst[r : r + step], src[r : r + step]))
    for j in jobs:
        j.result()


_STAGING: dict = {}


def _download_large(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> fresh host array for the big drop-in outputs (a 1080p
    cube is 431 MB): DMA into a cached pinned staging buffer, then a
    row-parallel copy into the new array, instead of one pageable copy that
    also faults in every destination page on a single thread."""
    t = t.contiguous()
    key = (t.numel(), t.dtype)
    buf = _STAGING.get(key)
    if buf is None:
        _STAGING.clear()  # one staging buffer at a time (the largest recent shape)
        buf = _STAGING[key] = torch.empty(t.numel(), dtype=t.dtype).pin_memory()
    host = buf[: t.numel()].view(t.shape)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    src = host.numpy()
    dst = np.empty(src.shape, dtype=src.dtype)
    _par_copy([(dst, src)])
    return dst


class _SequenceRunner:
    """Two pipeline slots for estimate_sequence: pinned host staging, device
    frame, workspace and fp64 map planes per slot, each on its own stream."""

    def __init__(self, sensitivity, basis, cfg: PipelineConfig, dims):
        check_grids(sensitivity.grid, basis.grid)
        H, W = dims
        n = cfg.n_levels
        if H < 2**n or W < 2**n:
            raise ArgumentError(f"frame {H}x{W} is smaller than 2^{n} in one dimension")
        self.lib = _native.load()
        self.dev = require_cuda()
        self.ctx = context(_hybrid_operators(sensitivity, basis, cfg), self.dev.index)
        self.H, self.W, self.n, self.cal = H, W, n, float(cfg.calibration_scale)
        hL, wL = level_dims(H, W, n)[-1]
        self.ws_bytes = int(self.lib.oxm_hybrid_workspace_bytes(self.ctx.handle, 1, H, W, n))
        d = dict(device=self.dev)
        self.slots = []
        for _ in range(2):
            self.slots.append({
                "stream": torch.cuda.Stream(device=self.dev),
                "h_in": torch.empty((1, H, W, 3), dtype=torch.float64).pin_memory(),
                "d_in": torch.empty((1, H, W, 3), dtype=torch.float64, **d),
                "ws": torch.empty(self.ws_bytes, dtype=torch.uint8, **d),
                "x": torch.empty((3, 1, H, W), dtype=torch.float64, **d),
                "fits": torch.empty((1, hL, wL), dtype=torch.int32, **d),
                "flags": torch.zeros(1, dtype=torch.int32, **d),
                "h_x": torch.empty((3, 1, H, W), dtype=torch.float64).pin_memory(),
                "h_flags": torch.zeros(1, dtype=torch.int32).pin_memory(),
                "done": torch.cuda.Event(),
            })
        self.turn = 0

    def submit(self, frame: RgbImage):
        sl = self.slots[self.turn]
        self.turn ^= 1
        t_sub = time.perf_counter()
        sl["done"].synchronize()  # the slot's previous frame has been collected
        _par_copy([(sl["h_in"].numpy()[0], frame.data)])
        s = sl["stream"]
        with torch.cuda.stream(s):
            sl["d_in"].copy_(sl["h_in"], non_blocking=True)
            sl["flags"].zero_()
            x = sl["x"]
            st = self.lib.oxm_hybrid_frame_f64(
                self.ctx.handle, ptr(sl["d_in"]), 1, self.H, self.W, self.n, self.cal, ptr(sl["ws"]), self.ws_bytes,
                None, ptr(x[0]), ptr(x[1]), ptr(x[2]), ptr(sl["fits"]), ptr(sl["flags"]), stream_handle(s), None)
            _native.check(st, "hybrid_frame_f64")
            sl["h_x"].copy_(x, non_blocking=True)
            sl["h_flags"].copy_(sl["flags"], non_blocking=True)
            sl["done"].record(s)
        return sl, t_sub

    def collect(self, job):
        sl, t_sub = job
        sl["done"].synchronize()
        f = int(sl["h_flags"][0])
        if f & _native.FLAG_NONFINITE:
            raise ArgumentError("image contains non-finite values")
        if f & _native.FLAG_NEGATIVE_LL:
            raise ArgumentError("low-pass coefficients must be finite and non-negative")
        xs = sl["h_x"].numpy()[:, 0]
        planes = [np.empty_like(xs[k]) for k in range(3)]
        _par_copy([(planes[k], xs[k]) for k in range(3)])
        return trusted_map(planes[0], planes[1], planes[2]), t_sub
