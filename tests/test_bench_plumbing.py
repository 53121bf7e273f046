"""bench.py's multi-rank path on CPU: `--gpus 2` outside torchrun re-launches
itself with two ranks (gloo), reduces the step time over ranks and gathers
every rank's maps to rank 0 (`--plumbing-check` swaps the kernels for a host
surrogate; the same code path runs the GPU bench)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_bench_spawns_ranks_and_gathers():
    env = dict(os.environ, OXM_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    env.pop("LOCAL_RANK", None)
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plumbing-check", "--batch", "2",
                          "--height", "4", "--width", "6", "--steps", "2"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["plumbing_check"]
    assert rec["gathered"]["value"] > 0 and rec["gathered"]["bytes_to_root_per_step"] == 2 * 4 * 6 * 8
    assert rec["gathered_blocks"] == [[0, 0.0], [2, 1.0]]  # rank r's block lands at frame 2r


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--plumbing-check"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert res.returncode != 0 and "WORLD_SIZE=1" in res.stderr
