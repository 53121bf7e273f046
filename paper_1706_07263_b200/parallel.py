"""Multi-GPU plumbing for video batches.

Frames are independent (no temporal coupling), so a video is
split into contiguous per-rank blocks and every rank runs the hybrid path on
its own frames with no data-path collective.  The only collectives are the
timing reduction (max over ranks, as the benchmark contract requires) and an
optional gather of finished maps to one rank.  One process per GPU,
torch.distributed (NCCL on GPUs, gloo for the CPU tests).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n_frames: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of frames owned by ``rank``; blocks differ in
    size by at most one frame and cover 0..n_frames exactly once."""
    if world_size < 1 or not 0 <= rank < world_size or n_frames < 0:
        raise ValueError(f"bad shard request n={n_frames} rank={rank} world={world_size}")
    base, extra = divmod(n_frames, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device: torch.device | None = None) -> float:
    """Max of a per-rank scalar (step time) over all ranks; identity when
    torch.distributed is not initialised."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    if dist.get_backend() == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_root(local: torch.Tensor, n_frames: int, root: int = 0) -> torch.Tensor | None:
    """Gather per-rank map blocks (frames, H, W) into the full (n_frames, H, W)
    tensor on ``root`` (None elsewhere).  Ranks send their contiguous block
    with point-to-point sends, so uneven blocks need no padding."""
    if not (dist.is_available() and dist.is_initialized()):
        return local
    ws, rank = dist.get_world_size(), dist.get_rank()
    if rank != root:
        dist.send(local.contiguous(), dst=root)
        return None
    out = torch.empty((n_frames,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r in range(ws):
        lo, hi = shard_range(n_frames, r, ws)
        if r == root:
            out[lo:hi] = local
        elif hi > lo:
            buf = torch.empty((hi - lo,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
            dist.recv(buf, src=r)
            out[lo:hi] = buf
    return out


def gather_chunk_to_root(local: torch.Tensor, n_frames: int, chunk: int, c: int, root: int = 0):
    """Streamed variant of gather_to_root for videos processed chunk by chunk
    (the final NVLink gather overlapped with the next chunk's
    compute).  Every rank calls it for chunk ``c`` with its maps of frames
    [lo + c * chunk, lo + (c + 1) * chunk) of its block (possibly empty when its
    block is shorter); the root receives the other ranks' chunks with batched
    point-to-point transfers and returns [(first frame index, tensor)] for all
    ranks' chunk c (its own included); other ranks return None.  Identity
    (single entry) without torch.distributed."""
    if not (dist.is_available() and dist.is_initialized()):
        return [(c * chunk, local)]
    ws, rank = dist.get_world_size(), dist.get_rank()
    spans = []
    for r in range(ws):
        lo, hi = shard_range(n_frames, r, ws)
        a, b = min(hi, lo + c * chunk), min(hi, lo + (c + 1) * chunk)
        spans.append((a, b))
    # gloo moves host tensors only: CUDA maps are staged through host memory
    # (the multi-rank functional check on one GPU); NCCL sends device memory
    host = dist.get_backend() == "gloo" and local.is_cuda
    if rank != root:
        a, b = spans[rank]
        if b > a:
            t = local.contiguous().cpu() if host else local.contiguous()
            dist.batch_isend_irecv([dist.P2POp(dist.isend, t, root)])[0].wait()
        return None
    ops, out = [], []
    for r in range(ws):
        a, b = spans[r]
        if r == root:
            out.append((a, local))
        elif b > a:
            buf = torch.empty((b - a,) + tuple(local.shape[1:]), dtype=local.dtype,
                              device="cpu" if host else local.device)
            ops.append(dist.P2POp(dist.irecv, buf, r))
            out.append((a, buf))
    for w in (dist.batch_isend_irecv(ops) if ops else []):
        w.wait()
    if host:
        out = [(a, t if t.device == local.device else t.to(local.device)) for a, t in out]
    return sorted(out, key=lambda t: t[0])
