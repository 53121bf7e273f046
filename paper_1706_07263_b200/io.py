"""GPU-native file path of ``oximap estimate`` (cli.py:317-340): 16-bit PPM
frames in, SPC1 maps out.

Only the two formats either side of the hot path are covered.  PPM rasters are
read as raw big-endian bytes and decoded on the device (oxm_hybrid_maps_u16,
value = count * scale exactly as io.py:139-162); maps are interleaved on the
device into the SPC1 payload (oxm_pack_hwc3_f32) and written with the
reference's header (io.py:34-39).  Header parsing follows io.py:112-137 with
the same DataError cases.
"""

from __future__ import annotations

import pathlib

import numpy as np
import torch

from . import _native
from .core import MAP_GRID, CameraSensitivity, ChromophoreBasis
from .device import ptr, require_cuda, stream_handle
from .errors import DataError

_SPC_MAGIC = "SPC1"


def _header_tokens(buf: bytes, path) -> tuple[list[bytes], float | None, int]:
    """Four header tokens (magic, width, height, maxval), the `# scale`
    comment and the raster offset (io.py:112-137)."""
    tokens: list[bytes] = []
    scale = None
    i = 0
    while len(tokens) < 4 and i < len(buf):
        ch = buf[i:i + 1]
        if ch == b"#":
            j = buf.find(b"\n", i)
            if j < 0:
                raise DataError(f"{path}: unterminated header comment")
            words = buf[i + 1:j].decode("ascii", errors="replace").split()
            if len(words) == 2 and words[0] == "scale":
                try:
                    scale = float(words[1])
                except ValueError as exc:
                    raise DataError(f"{path}: bad scale comment: {exc}") from exc
            i = j + 1
        elif ch.isspace():
            i += 1
        else:
            j = i
            while j < len(buf) and not buf[j:j + 1].isspace() and buf[j:j + 1] != b"#":
                j += 1
            tokens.append(buf[i:j])
            i = j
    if len(tokens) < 4:
        raise DataError(f"{path}: truncated pixmap header")
    return tokens, scale, i + 1


def read_ppm_raw(path) -> tuple[np.ndarray, float]:
    """(H, W, 3) uint16 counts in FILE byte order (big-endian, not swapped)
    and the scale; decode happens on the device."""
    path = pathlib.Path(path)
    buf = path.read_bytes()
    if not buf.startswith(b"P6"):
        raise DataError(f"{path}: not a binary pixmap (missing P6 magic)")
    tokens, scale, off = _header_tokens(buf, path)
    try:
        w, h, maxval = int(tokens[1]), int(tokens[2]), int(tokens[3])
    except ValueError as exc:
        raise DataError(f"{path}: malformed pixmap header: {exc}") from exc
    if maxval != 65535:
        raise DataError(f"{path}: expected 16-bit pixmap (maxval 65535), got {maxval}")
    if w < 1 or h < 1:
        raise DataError(f"{path}: non-positive pixmap dimensions {w}x{h}")
    raster = buf[off:]
    if len(raster) != w * h * 6:
        raise DataError(f"{path}: truncated raster, expected {w * h * 6} bytes, got {len(raster)}")
    return np.frombuffer(raster, dtype=np.uint16).reshape(h, w, 3), 1.0 if scale is None else scale


def spc1_map_bytes(hbo: torch.Tensor, hb: torch.Tensor, offset: torch.Tensor) -> bytes:
    """SPC1 file bytes for one (H, W) map given as CUDA float32 planes."""
    H, W = hbo.shape
    payload = torch.empty((H, W, 3), dtype=torch.float32, device=hbo.device)
    st = _native.load().oxm_pack_hwc3_f32(ptr(hbo.contiguous()), ptr(hb.contiguous()), ptr(offset.contiguous()),
                                          H * W, ptr(payload), stream_handle())
    _native.check(st, "pack_hwc3")
    header = f"{_SPC_MAGIC} {H} {W} 3 {MAP_GRID.start_nm!r} {MAP_GRID.step_nm!r}\n".encode("ascii")
    return header + payload.cpu().numpy().astype("<f4", copy=False).tobytes()


def estimate_files(inputs, outputs, sensitivity: CameraSensitivity, basis: ChromophoreBasis, cfg=None) -> int:
    """PPM frames -> SPC1 maps (the `oximap estimate` loop, cli.py:317-340) on
    the GPU: raw 16-bit rasters go to the device, maps come back as SPC1
    payloads.  Returns the number of frames processed."""
    from .engine import HybridMapEngine
    from .pipeline import PipelineConfig

    eng = HybridMapEngine(sensitivity, basis, cfg if cfg is not None else PipelineConfig())
    dev = require_cuda()
    n = 0
    for src, dst in zip(inputs, outputs):
        counts, scale = read_ppm_raw(src)
        frames = torch.from_numpy(counts[None].copy()).to(dev)
        out = eng.run(frames, planes=True, scale=scale, big_endian=True)
        pathlib.Path(dst).write_bytes(spc1_map_bytes(out.hbo[0], out.hb[0], out.offset[0]))
        n += 1
    return n
