"""Iterative shape-prior ("Bayes") low-pass estimator -- drop-in for
oximap.bayes (bayes.py:1-272).

Host side: config validation, the L x L prior (cond check + Cholesky) and
the operator context.  Device side: K4 (``oxm_em_lowpass``) runs the whole
fixed-point iteration per coefficient in fp64, K5 the Beer-Lambert fits.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .core import CameraSensitivity, ChromophoreBasis, ConcentrationMap
from .device import download, ptr, require_cuda, stream_handle, upload
from .errors import ArgumentError
from .operators import (
    DEFAULT_FALLBACK_BELOW,
    OperatorSet,
    ShapePrior,
    context,
    make_operator_set,
    second_difference,
)
from .unmix import TikhonovOperator

__all__ = [
    "BayesConfig",
    "LowPassBlock",
    "second_difference",
    "fit_concentration",
    "expected_spectrum",
    "expectation_step",
    "estimate_lowpass",
    "estimate_lowpass_fits",
    "em_operator_set",
]


@dataclass(frozen=True)
class BayesConfig:
    """Estimator knobs (bayes.py:36-58)."""

    beta: float = 0.1
    max_iters: int = 20
    rel_tol: float = 1e-4
    epsilon: float = 1e-6

    def __post_init__(self):
        if not self.beta > 0:
            raise ArgumentError(f"beta must be > 0, got {self.beta}")
        if self.max_iters < 1:
            raise ArgumentError(f"max_iters must be >= 1, got {self.max_iters}")
        if not 0 < self.epsilon < 1:
            raise ArgumentError(f"epsilon must be in (0, 1), got {self.epsilon}")
        if not self.rel_tol > 0:
            raise ArgumentError(f"rel_tol must be > 0, got {self.rel_tol}")


@dataclass(frozen=True)
class LowPassBlock:
    """Low-pass RGB plane (h, w, 3) and its accumulated gain 2^n (bayes.py:61-81)."""

    rgb_lp: np.ndarray
    scale: float

    def __post_init__(self):
        arr = np.asarray(self.rgb_lp, dtype=np.float64)
        if arr.ndim != 3 or arr.shape[2] != 3:
            raise ArgumentError(f"rgb_lp must be (h, w, 3), got shape {arr.shape}")
        if (arr < 0).any() or not np.isfinite(arr).all():
            raise ArgumentError("low-pass coefficients must be finite and non-negative")
        if not self.scale > 0:
            raise ArgumentError(f"scale must be > 0, got {self.scale}")
        object.__setattr__(self, "rgb_lp", arr)


def em_operator_set(
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: BayesConfig,
    init: TikhonovOperator,
    fallback_below: float = DEFAULT_FALLBACK_BELOW,
) -> OperatorSet:
    """Operators of the estimator; raises IllConditionedPriorError like
    _ShapePriorSolver (bayes.py:117-129)."""
    prior = ShapePrior.build(sensitivity.c, cfg.beta)
    return make_operator_set(
        n_bands=sensitivity.grid.count,
        solve=init.solve,
        xi=basis.xi,
        sens=sensitivity.c,
        gain=prior.gain,
        epsilon=cfg.epsilon,
        rel_tol=cfg.rel_tol,
        max_iters=cfg.max_iters,
        fallback_below=fallback_below,
    )


def _flat(arr: np.ndarray, width: int, what: str) -> tuple[np.ndarray, tuple[int, ...]]:
    a = np.asarray(arr, dtype=np.float64)
    if a.shape[-1] != width:
        raise ArgumentError(f"{what}")
    lead = a.shape[:-1]
    return a.reshape(-1, width), lead


def fit_concentration(spectrum: np.ndarray, basis: ChromophoreBasis, epsilon: float = 1e-6) -> np.ndarray:
    """(hbo, hb, offset) least-squares fit of -log(max(s, eps)) (bayes.py:138-151), K5."""
    L = basis.grid.count
    flat, lead = _flat(spectrum, L, f"spectrum has {np.shape(spectrum)[-1]} bands, basis expects {L}")
    ops = make_operator_set(n_bands=L, xi=basis.xi, epsilon=epsilon)
    x = fit_device(upload(flat, torch.float64, require_cuda()), ops, calibration=1.0)
    return download(x).reshape(lead + (3,))


def fit_device(cube: torch.Tensor, ops: OperatorSet, calibration: float = 1.0, *, stream=None) -> torch.Tensor:
    """K5 on an (n, L) device tensor; returns (n, 3) = (hbo*cal, hb*cal, offset)."""
    lib = _native.load()
    cube = cube.contiguous()
    n = cube.shape[0]
    ctx = context(ops, cube.device.index)
    planes = torch.empty((3, n), dtype=cube.dtype, device=cube.device)
    fn = lib.oxm_fit_f64 if cube.dtype == torch.float64 else lib.oxm_fit_f32
    _native.check(
        fn(ctx.handle, ptr(cube), n, float(calibration), ptr(planes[0]), ptr(planes[1]), ptr(planes[2]), stream_handle(stream)),
        "fit",
    )
    return planes.t()


def expected_spectrum(x: np.ndarray, basis: ChromophoreBasis) -> np.ndarray:
    """Beer-Lambert forward model exp(-xi x) (bayes.py:154-159)."""
    flat, lead = _flat(x, 3, f"concentration vectors must have 3 components, got {np.shape(x)}")
    L = basis.grid.count
    if flat.shape[0] == 0:
        return np.zeros(lead + (L,))
    lib = _native.load()
    dev = require_cuda()
    ops = make_operator_set(n_bands=L, xi=basis.xi)
    ctx = context(ops, dev.index)
    xd = upload(flat, torch.float64, dev)
    out = torch.empty((flat.shape[0], L), dtype=torch.float64, device=dev)
    _native.check(lib.oxm_expected_spectrum_f64(ctx.handle, ptr(xd), flat.shape[0], ptr(out), stream_handle()), "expected_spectrum")
    return download(out).reshape(lead + (L,))


def expectation_step(
    rgb_lp: np.ndarray, e_spectrum: np.ndarray, sensitivity: CameraSensitivity, cfg: BayesConfig
) -> np.ndarray:
    """Minimiser of ||C i - y||^2 + beta ||D2 (i - e)||^2 per (y, e) pair
    (bayes.py:162-182), evaluated on the GPU as e + N^-1 C^T (y - C e)."""
    y = np.asarray(rgb_lp, dtype=np.float64)
    e = np.asarray(e_spectrum, dtype=np.float64)
    if y.shape[-1] != 3:
        raise ArgumentError(f"rgb_lp must have 3 trailing channels, got {y.shape}")
    L = sensitivity.grid.count
    if e.shape[-1] != L:
        raise ArgumentError(f"expected spectrum has {e.shape[-1]} bands, sensitivity expects {L}")
    prior = ShapePrior.build(sensitivity.c, cfg.beta)
    lead = np.broadcast_shapes(y.shape[:-1], e.shape[:-1])
    yb = np.broadcast_to(y, lead + (3,)).reshape(-1, 3)
    eb = np.broadcast_to(e, lead + (L,)).reshape(-1, L)
    n = yb.shape[0]
    if n == 0:
        return np.zeros(lead + (L,))
    lib = _native.load()
    dev = require_cuda()
    ops = make_operator_set(n_bands=L, sens=sensitivity.c, gain=prior.gain)
    ctx = context(ops, dev.index)
    yd, ed = upload(yb, torch.float64, dev), upload(eb, torch.float64, dev)
    out = torch.empty((n, L), dtype=torch.float64, device=dev)
    _native.check(lib.oxm_expectation_step(ctx.handle, ptr(yd), ptr(ed), n, ptr(out), stream_handle()), "expectation_step")
    return download(out).reshape(lead + (L,))


def em_device(y: torch.Tensor, ops: OperatorSet, init: torch.Tensor | None = None, *, stream=None):
    """K4 on an (n, 3) unit-scale device tensor -> (spectra (n, L), x (n, 3), fits (n,))."""
    lib = _native.load()
    y = y.contiguous().to(torch.float64)
    n = y.shape[0]
    L = ops.n_bands
    ctx = context(ops, y.device.index)
    spectra = torch.empty((n, L), dtype=torch.float64, device=y.device)
    x = torch.empty((n, 3), dtype=torch.float64, device=y.device)
    fits = torch.empty((n,), dtype=torch.int32, device=y.device)
    init_p = ptr(init.contiguous().to(torch.float64)) if init is not None else None
    _native.check(
        lib.oxm_em_lowpass(ctx.handle, ptr(y), init_p, n, ptr(spectra), ptr(x), ptr(fits), stream_handle(stream)),
        "em_lowpass",
    )
    return spectra, x, fits


def estimate_lowpass_fits(
    block: LowPassBlock,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: BayesConfig,
    init: TikhonovOperator,
    *,
    threads: int = 1,
    init_spectra: np.ndarray | None = None,
) -> tuple[np.ndarray, ConcentrationMap, np.ndarray]:
    """``estimate_lowpass`` plus the per-coefficient fit counts (h, w)."""
    del threads  # the GPU path parallelises per coefficient
    h, w = block.rgb_lp.shape[:2]
    n = h * w
    L = sensitivity.grid.count
    ops = em_operator_set(sensitivity, basis, cfg, init)
    y = (block.rgb_lp / block.scale).reshape(n, 3)
    dev = require_cuda()
    init_t = None
    if init_spectra is not None:
        init_arr = np.asarray(init_spectra, dtype=np.float64)
        if init_arr.shape[-1] != L:
            raise ArgumentError(f"init_spectra has {init_arr.shape[-1]} bands, expected {L}")
        init_t = upload(init_arr.reshape(n, L), torch.float64, dev)
    if n == 0:
        z = np.zeros((h, w))
        return np.zeros((h, w, L)), ConcentrationMap(hbo=z, hb=z, offset=z), np.zeros((h, w), dtype=np.int32)
    spectra, x, fits = em_device(upload(y, torch.float64, dev), ops, init_t)
    xs = download(x)
    cmap = ConcentrationMap(hbo=xs[:, 0].reshape(h, w), hb=xs[:, 1].reshape(h, w), offset=xs[:, 2].reshape(h, w))
    return download(spectra).reshape(h, w, L), cmap, download(fits).reshape(h, w)


def estimate_lowpass(
    block: LowPassBlock,
    sensitivity: CameraSensitivity,
    basis: ChromophoreBasis,
    cfg: BayesConfig,
    init: TikhonovOperator,
    *,
    threads: int = 1,
    init_spectra: np.ndarray | None = None,
) -> tuple[np.ndarray, ConcentrationMap]:
    """Spectra (h, w, L) and concentrations of a low-pass plane (bayes.py:210-272)."""
    spectra, cmap, _ = estimate_lowpass_fits(
        block, sensitivity, basis, cfg, init, threads=threads, init_spectra=init_spectra
    )
    return spectra, cmap
