"""Multi-rank host logic on CPU: world_size 2 over gloo (no GPU needed)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_07263_b200.parallel import gather_chunk_to_root, gather_to_root, max_over_ranks, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 4096):
        for ws in (1, 2, 3, 8):
            seen = []
            for r in range(ws):
                lo, hi = shard_range(n, r, ws)
                seen.extend(range(lo, hi))
                assert hi - lo in (n // ws, n // ws + 1)
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        n = 5
        lo, hi = shard_range(n, rank, ws)
        # each rank's "maps": frame index broadcast over a 2x3 plane
        local = torch.arange(lo, hi, dtype=torch.float32)[:, None, None].expand(hi - lo, 2, 3).contiguous()
        full = gather_to_root(local, n)
        t = max_over_ranks(0.5 + rank)
        # streamed gather, chunks of 2 frames (rank blocks 0..2 and 3..4: uneven)
        streamed = []
        for c in range(2):
            cl = local[2 * c:2 * c + 2]
            got = gather_chunk_to_root(cl, n, 2, c)
            if got is not None:
                streamed.extend((a, t_[:, 0, 0].tolist()) for a, t_ in got)
        q.put((rank, t, None if full is None else full[:, 0, 0].tolist(), streamed if rank == 0 else None))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1] == 1.5  # max over ranks
    assert res[0][2] == [0.0, 1.0, 2.0, 3.0, 4.0]  # gathered in frame order on rank 0
    assert res[1][2] is None
    # streamed gather: chunk 0 of both blocks, then chunk 1 (rank 1's block is exhausted)
    assert res[0][3] == [(0, [0.0, 1.0]), (3, [3.0, 4.0]), (2, [2.0])]
