"""Device plumbing: torch owns device memory and streams, the C ABI gets raw
pointers.  No compute happens here."""

from __future__ import annotations

import numpy as np
import torch

from .errors import NativeLibraryError


def require_cuda() -> torch.device:
    """The current CUDA device; raises when there is none (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device visible: the sm_100a path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return int(t.data_ptr()) if t.numel() > 0 else None


def upload(arr: np.ndarray, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Host array -> contiguous device tensor of ``dtype``."""
    host = torch.from_numpy(np.require(arr, requirements=("C", "W")))  # copies read-only / strided views
    return host.to(device=device, dtype=dtype, non_blocking=False).contiguous()


def download(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def empty(shape, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    return torch.empty(tuple(int(s) for s in shape), dtype=dtype, device=device)
