"""Closed-form RGB -> spectrum inverses -- drop-in for oximap.unmix
(unmix.py:1-105).  The operators are built on the host (3 x 3 solves); their
application to every 3-vector runs the K3 kernel in fp64."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .core import CameraSensitivity
from .device import download, ptr, require_cuda, stream_handle, upload
from .errors import ArgumentError, SingularOperatorError
from .haar import HaarLevel, HaarPyramid
from .operators import ridge_inverse


def apply_matrix(rgb: np.ndarray, matrix: np.ndarray) -> np.ndarray:
    """out[..., l] = sum_k matrix[l, k] rgb[..., k] on the GPU (K3)."""
    rgb = np.asarray(rgb, dtype=np.float64)
    if rgb.shape[-1] != 3:
        raise ArgumentError(f"expected trailing axis of 3 channels, got shape {rgb.shape}")
    L = matrix.shape[0]
    lead = rgb.shape[:-1]
    n = int(np.prod(lead)) if lead else 1
    if n == 0:
        return np.zeros(lead + (L,))
    dev = require_cuda()
    out = apply_matrix_device(upload(rgb.reshape(n, 3), torch.float64, dev), matrix)
    return download(out).reshape(lead + (L,))


def apply_matrix_device(rgb: torch.Tensor, matrix: np.ndarray, *, stream=None) -> torch.Tensor:
    """K3 on an (n, 3) device tensor (float32 or float64)."""
    lib = _native.load()
    m = np.ascontiguousarray(matrix, dtype=np.float64)
    L = m.shape[0]
    if not 1 <= L <= _native.MAX_BANDS:
        raise ArgumentError(f"the CUDA kernels support up to {_native.MAX_BANDS} bands, got {L}")
    rgb = rgb.contiguous()
    n = rgb.shape[0]
    out = torch.empty((n, L), dtype=rgb.dtype, device=rgb.device)
    fn = lib.oxm_unmix_f64 if rgb.dtype == torch.float64 else lib.oxm_unmix_f32
    _native.check(fn(L, m.ctypes.data, ptr(rgb), n, ptr(out), stream_handle(stream)), "unmix")
    return out


def lsq_unmix(rgb: np.ndarray, sensitivity: CameraSensitivity) -> np.ndarray:
    """Minimum-norm least squares s = C^T (C C^T)^-1 y (unmix.py:21-37)."""
    c = sensitivity.c
    gram = c @ c.T
    if np.linalg.matrix_rank(gram) < 3:
        raise SingularOperatorError("sensitivity matrix is rank deficient")
    return apply_matrix(rgb, np.linalg.solve(gram, c).T)


@dataclass(frozen=True)
class TikhonovOperator:
    """L x 3 ridge inverse (C^T C + gamma I)^-1 C^T (unmix.py:40-74)."""

    sensitivity: CameraSensitivity
    gamma: float
    solve: np.ndarray

    @classmethod
    def build(cls, sensitivity: CameraSensitivity, gamma: float) -> "TikhonovOperator":
        if gamma <= 0:
            raise ArgumentError(f"gamma must be > 0, got {gamma}")
        return cls(sensitivity=sensitivity, gamma=float(gamma), solve=ridge_inverse(sensitivity.c, gamma))

    @classmethod
    def from_relative(cls, sensitivity: CameraSensitivity, rel_gamma: float = 1e-3) -> "TikhonovOperator":
        """gamma = rel_gamma * trace(C^T C) / L."""
        c = sensitivity.c
        return cls.build(sensitivity, rel_gamma * (np.trace(c.T @ c) / c.shape[1]))


def tikhonov_unmix(rgb: np.ndarray, op: TikhonovOperator) -> np.ndarray:
    """rgb @ op.solve.T for every 3-vector (unmix.py:77-82)."""
    return apply_matrix(rgb, op.solve)


def unmix_pyramid_directional(pyramid: HaarPyramid, op: TikhonovOperator) -> HaarPyramid:
    """Unmix every directional plane; low-pass planes pass through
    (unmix.py:85-105)."""
    levels = []
    for level in pyramid.levels:
        if np.shape(level.dh)[-1] != 3:
            raise ArgumentError("pyramid must carry 3-channel (RGB) planes")
        levels.append(
            HaarLevel(
                lp=level.lp,
                dh=tikhonov_unmix(level.dh, op),
                dv=tikhonov_unmix(level.dv, op),
                dd=tikhonov_unmix(level.dd, op),
                orig_shape=level.orig_shape,
            )
        )
    return HaarPyramid(levels=tuple(levels))
