"""Multi-level 2D Haar transform -- drop-in for oximap.haar (haar.py:1-150).

``forward`` and ``inverse`` run the fused sm_100a kernels K1/K2 in fp64 (the
add order matches the reference, so coefficients are bit-identical).  The
containers and the host-side shape contract are the reference's.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .device import download, ptr, require_cuda, stream_handle, upload
from .errors import ArgumentError, DataError


def haar_matrix() -> np.ndarray:
    """Orthonormal, symmetric, involutory window matrix (haar.py:24-33).
    Window row vector order: (top-left, top-right, bottom-left, bottom-right)."""
    signs = np.array([[1, 1, 1, 1], [1, 1, -1, -1], [1, -1, -1, 1], [1, -1, 1, -1]], dtype=np.float64)
    return 0.5 * signs


@dataclass(frozen=True)
class HaarLevel:
    """Planes of one level; ``lp`` may be None below the coarsest level of an
    assembled pyramid.  ``orig_shape`` = pre-padding (rows, cols)."""

    lp: np.ndarray | None
    dh: np.ndarray
    dv: np.ndarray
    dd: np.ndarray
    orig_shape: tuple[int, int]


@dataclass(frozen=True)
class HaarPyramid:
    """Levels, finest first; the coarsest carries the residual low-pass."""

    levels: tuple[HaarLevel, ...]

    def __post_init__(self):
        if len(self.levels) == 0:
            raise ArgumentError("pyramid must have at least one level")
        if self.levels[-1].lp is None:
            raise ArgumentError("coarsest level must carry its low-pass plane")

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def residual_lp(self) -> np.ndarray:
        return self.levels[-1].lp


def _as_hwc(image: np.ndarray) -> tuple[np.ndarray, tuple[int, ...]]:
    """(H, W) or (H, W, C...) -> (H, W, C) plus the trailing shape."""
    tail = image.shape[2:]
    return image.reshape(image.shape[0], image.shape[1], -1), tail


def forward(image: np.ndarray, n_levels: int) -> HaarPyramid:
    """Decompose into ``n_levels`` levels (haar.py:120-142) on the GPU."""
    if n_levels < 1:
        raise ArgumentError(f"n_levels must be >= 1, got {n_levels}")
    img = np.asarray(image, dtype=np.float64)
    if img.ndim not in (2, 3):
        raise ArgumentError(f"image must be 2-D or 3-D, got shape {img.shape}")
    if img.shape[0] < 1 or img.shape[1] < 1:
        raise ArgumentError("image must have at least one pixel per axis")
    hwc, tail = _as_hwc(img)
    H, W, C = hwc.shape
    levels = pyramid_device(upload(hwc, torch.float64, require_cuda()), n_levels)
    out = []
    for (lp, dh, dv, dd), oshape in levels:
        planes = [download(p).reshape(p.shape[0], p.shape[1], *tail) for p in (lp, dh, dv, dd)]
        out.append(HaarLevel(lp=planes[0], dh=planes[1], dv=planes[2], dd=planes[3], orig_shape=oshape))
    return HaarPyramid(levels=tuple(out))


def level_dims(height: int, width: int, n_levels: int) -> list[tuple[int, int]]:
    dims = []
    h, w = height, width
    for _ in range(n_levels):
        h, w = (h + 1) // 2, (w + 1) // 2
        dims.append((h, w))
    return dims


def pyramid_device(image: torch.Tensor, n_levels: int, *, stream=None):
    """K1 on a device (H, W, C) float32/float64 tensor.  Returns per level
    ((lp, dh, dv, dd) device views, orig_shape).  Raises ArgumentError on
    non-finite input (haar.py:133-134)."""
    lib = _native.load()
    if image.dim() != 3 or not image.is_cuda:
        raise ArgumentError("pyramid_device expects a CUDA (H, W, C) tensor")
    image = image.contiguous()
    H, W, C = image.shape
    dims = level_dims(H, W, n_levels)
    total = sum(4 * h * w for h, w in dims) * C
    planes = torch.empty(total, dtype=image.dtype, device=image.device)
    flags = torch.zeros(1, dtype=torch.int32, device=image.device)
    fn = lib.oxm_haar_forward_f64 if image.dtype == torch.float64 else lib.oxm_haar_forward_f32
    if image.dtype not in (torch.float64, torch.float32):
        raise ArgumentError(f"unsupported dtype {image.dtype}")
    _native.check(fn(ptr(image), H, W, C, n_levels, ptr(planes), ptr(flags), stream_handle(stream)), "haar_forward")
    if int(flags.item()) & _native.FLAG_NONFINITE:
        raise ArgumentError("image contains non-finite values")
    out, off = [], 0
    prev = (H, W)
    for h, w in dims:
        sz = h * w * C
        quad = tuple(planes[off + q * sz : off + (q + 1) * sz].view(h, w, C) for q in range(4))
        out.append((quad, prev))
        prev = (h, w)
        off += 4 * sz
    return out


def _check_chain(pyramid: HaarPyramid) -> list[tuple[int, int, int, int]]:
    """Walk the levels coarse -> fine like haar.py:145-150 / 104-117 and raise
    the same DataError on a shape mismatch; returns (h, w, crop_h, crop_w)
    per level, finest first."""
    lp_shape = tuple(np.shape(pyramid.residual_lp))
    shapes: list[tuple[int, int, int, int]] = []
    for level in reversed(pyramid.levels):
        for name in ("dh", "dv", "dd"):
            got = tuple(np.shape(getattr(level, name)))
            if got != lp_shape:
                raise DataError(f"level plane {name} has shape {got}, expected {lp_shape}")
        h, w = lp_shape[0], lp_shape[1]
        oh, ow = level.orig_shape
        ch, cw = min(max(int(oh), 0), 2 * h), min(max(int(ow), 0), 2 * w)
        shapes.append((h, w, ch, cw))
        lp_shape = (ch, cw) + lp_shape[2:]
    shapes.reverse()
    return shapes


def inverse(pyramid: HaarPyramid) -> np.ndarray:
    """Reconstruct with per-level crop (haar.py:145-150) on the GPU."""
    shapes = _check_chain(pyramid)
    res = np.asarray(pyramid.residual_lp, dtype=np.float64)
    tail = res.shape[2:]
    C = int(np.prod(tail)) if tail else 1
    h0, w0, ch0, cw0 = shapes[0]
    if ch0 == 0 or cw0 == 0:
        return np.zeros((ch0, cw0) + tail)
    dev = require_cuda()
    dirs = np.concatenate(
        [np.asarray(getattr(lv, nm), dtype=np.float64).reshape(-1) for lv in pyramid.levels for nm in ("dh", "dv", "dd")]
    )
    out = inverse_device(
        upload(res.reshape(res.shape[0], res.shape[1], C), torch.float64, dev),
        upload(dirs, torch.float64, dev),
        shapes,
        C,
    )
    return download(out).reshape((ch0, cw0) + tail)


def inverse_device(coarse_lp: torch.Tensor, dirs: torch.Tensor, shapes, channels: int, *, stream=None) -> torch.Tensor:
    """K2 on device tensors.  ``shapes`` = [(h, w, crop_h, crop_w)] finest first."""
    lib = _native.load()
    n = len(shapes)
    shp = (ctypes.c_int64 * (4 * n))(*[int(v) for s in shapes for v in s])
    out = torch.empty((shapes[0][2], shapes[0][3], channels), dtype=coarse_lp.dtype, device=coarse_lp.device)
    fn = lib.oxm_haar_inverse_f64 if coarse_lp.dtype == torch.float64 else lib.oxm_haar_inverse_f32
    _native.check(
        fn(ptr(coarse_lp.contiguous()), ptr(dirs.contiguous()), ctypes.addressof(shp), n, channels, ptr(out), stream_handle(stream)),
        "haar_inverse",
    )
    return out
