#!/usr/bin/env python3
"""Benchmark: THb/SO2 frames per second at 1080p, 2-level Haar (BASELINE.json
config 3, "1920x1080 RGB frame, 2-level Haar, single B200 throughput sweep").

One "step" = the hybrid hot path over one batch of `--batch` synthetic frames
(frames already in HBM): low-pass chain -> fp64 EM -> fused per-pixel
reconstruction + Beer-Lambert fit + THb/SO2.  Frames are independent, so
multi-GPU runs (torchrun) shard frames with no data-path collective
("scaling": "weak"): every rank processes its own batch; the step time is the
max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N` outside torchrun re-launches itself under torch.distributed.run
with N ranks (one per GPU).  Besides the sharded `value`, the line carries
`gathered` (the same steps with every rank's maps gathered to rank 0, SURVEY
§8e), `parity` (the timed batch against the oracle and against the all-fp64 EM
schedule), `cpu_baseline` (both reference thread settings), `e2e` and
`dropin` (the reference user's estimate_frame / estimate_sequence calls).

`--impl reference` times the reference CPU implementation of the path (the
pinned NumPy oracle port, oracle/oximap_oracle.py: the reference is pure
Python and cannot travel to the GPU box) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "THb/SO2 frames/sec at 1080p, 2-level Haar"
UNIT = "frames/s"
WORKLOAD = "1920x1080 RGB, 2-level Haar, hybrid (Tikhonov detail + iterative Bayes LL), THb+SO2 maps"
CPU_SAMPLE_FRAMES = 6  # ~8 s of host work per reference thread setting at 1080p n=2 (10-30 s in all)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--batch", type=int, default=DEFAULT_BATCH, help="frames per step per GPU")
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--levels", type=int, default=2)
    p.add_argument("--texture", type=float, default=0.3, help="phantom texture_density")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-dropin", action="store_true")
    p.add_argument("--plumbing-check", action="store_true",
                   help="CPU dry run of the multi-rank plumbing (tests only; no kernels, not a measurement)")
    return p.parse_args()


def workload_config(args) -> dict:
    """The `config` object, identical for both arms (the driver pairs lines on it)."""
    return {"workload": WORKLOAD, "height": args.height, "width": args.width, "levels": args.levels,
            "texture_density": args.texture}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def operators():
    from paper_1706_07263_b200 import fixtures

    return fixtures.default_sensitivity(), fixtures.default_basis()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md): the
    sampler runs every 20 ms and is up (first sample written) before the timed
    region starts; `mark()` brackets the region in wall-clock time and the
    summary keeps the samples whose nvidia-smi timestamps fall inside it (or,
    for a region shorter than the sampling period, the first one after its
    start)."""

    FIELD_SETS = [
        ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,timestamp"),
        ("index,clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active,"
         "clocks_throttle_reasons.hw_slowdown,clocks_throttle_reasons.hw_thermal_slowdown,"
         "clocks_throttle_reasons.sw_thermal_slowdown,clocks_throttle_reasons.sw_power_cap,timestamp"),
    ]
    PERIOD_MS = 20

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def _fields(self):
        for f in self.FIELD_SETS:
            try:
                r = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={f}", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=20)
            except (OSError, subprocess.TimeoutExpired):
                return None
            if r.returncode == 0 and r.stdout.strip():
                return f
        return None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        fields = self._fields()
        self.proc = None
        if fields:
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                     "-lms", str(self.PERIOD_MS)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
                deadline = time.time() + 5.0  # wait for the sampler's first line (NVML start-up)
                while time.time() < deadline and os.path.getsize(self.path) == 0:
                    time.sleep(0.02)
            except OSError:
                self.proc = None
        return self

    def mark(self, start: bool) -> None:
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(2 * self.PERIOD_MS / 1000)  # let the sample covering the region's end land
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    @staticmethod
    def _ts(text: str):
        import datetime

        try:
            return datetime.datetime.strptime(text.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 10 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        window = rows
        if self.t0 is not None and self.t1 is not None:
            stamped = [(self._ts(r[9]), r) for r in rows]
            window = [r for t, r in stamped if t is not None and self.t0 <= t <= self.t1]
            if not window:  # region shorter than the sampling period: the first sample after its start
                after = [r for t, r in stamped if t is not None and t >= self.t0]
                window = after[:1] or rows[-1:]
        sm = [float(r[1]) for r in window]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in window for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        pw = [float(r[3]) for r in window if r[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(window[0][2]), "reasons": reasons,
                "samples": len(window), "sample_period_ms": self.PERIOD_MS,
                "window_s": round(self.t1 - self.t0, 4) if self.t0 is not None and self.t1 is not None else None,
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------- inputs
def make_frames(batch, H, W, texture, rank, device):
    """(batch, H, W, 3) float32 phantom frames on `device`: 4 distinct truth
    maps per rank (seeded), forward model + per-frame Philox noise by the
    oxm_synth_frames_f32 kernel (untimed input staging)."""
    import torch

    from paper_1706_07263_b200 import synth

    sens, basis = operators()
    out = torch.empty((batch, H, W, 3), dtype=torch.float32, device=device)
    n_truth = min(4, batch)
    per = -(-batch // n_truth)
    for t in range(n_truth):
        spec = synth.tissue_phantom_spec(H, W, seed=100 * rank + t, noise_sigma=0.0, texture_density=texture)
        truth = synth.truth_map(spec)
        lo, hi = t * per, min(batch, (t + 1) * per)
        if lo < hi:
            out[lo:hi] = synth.device_frames(truth, sens, basis, hi - lo, noise_sigma=0.01, seed=1000 * rank + t,
                                             device=device)
    return out


# ---------------------------------------------------------------- cpu baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _oracle_frames(frames_host: np.ndarray, levels: int, threads: int, blas: int):
    """Oracle port (= reference arithmetic) over the frames with `threads`
    worker threads and BLAS capped at `blas`; returns (seconds, outputs)."""
    from threadpoolctl import threadpool_limits

    from oracle import oximap_oracle as O

    sens, basis = operators()
    outs = []
    with threadpool_limits(limits=blas):
        O.estimate_frame(frames_host[0].astype(np.float64)[:64, :64], sens.c, basis.xi, n_levels=levels)  # warm
        t0 = time.perf_counter()
        for f in frames_host:
            outs.append(O.estimate_frame(f.astype(np.float64), sens.c, basis.xi, n_levels=levels, threads=threads,
                                         want_cube=False))
        dt = time.perf_counter() - t0
    return dt, outs


def cpu_baseline(frames_host: np.ndarray, levels: int, n_other: int) -> tuple[dict, list]:
    """SURVEY.md §8d protocol on the host cores: the reference's two thread
    settings -- threads = nproc with BLAS 1 thread, and threads = 1 with BLAS
    on every core -- the better one reported, with nproc and the CPU model.
    The second setting runs on the first `n_other` frames of the sample.
    Returns the record and the oracle outputs of the first setting (the
    bench's parity sample)."""
    from oracle import oximap_oracle as O

    nproc = O.default_threads()
    dt_a, outs = _oracle_frames(frames_host, levels, nproc, 1)
    dt_b, _ = _oracle_frames(frames_host[:n_other], levels, 1, nproc)
    fps_a, fps_b = len(frames_host) / dt_a, n_other / dt_b
    best_a = fps_a >= fps_b
    settings = {"threads=nproc, BLAS=1": {"value": fps_a, "frames": len(frames_host), "seconds": dt_a},
                "threads=1, BLAS=nproc": {"value": fps_b, "frames": n_other, "seconds": dt_b}}
    H, W = frames_host.shape[1:3]
    rec = {"value": max(fps_a, fps_b), "unit": UNIT, "cores": nproc, "kind": "port", "nproc": nproc,
           "cpu_model": cpu_model(),
           "setting": "threads=nproc, BLAS=1" if best_a else "threads=1, BLAS=nproc",
           "settings": settings,
           "sample": f"frames 0..{len(frames_host) - 1} of the timed batch ({H}x{W}, n={levels}), hybrid via "
                     f"oracle/oximap_oracle.py (bit-identical to the reference); both reference thread settings, "
                     f"the better reported"}
    return rec, outs


def parity_record(out, ref_outs: list, frames_idx: list) -> dict:
    """The timed batch's maps against the oracle on `frames_idx`: fit counts
    (bit-exact), THb relative, SO2 absolute, NaN pattern (north-star
    tolerances 1e-4 / 1e-5)."""
    thb, so2, fits = out.thb.cpu().numpy(), out.so2.cpu().numpy(), out.fits.cpu().numpy()
    flips, ncoef, thb_rel, so2_abs, nan_eq = 0, 0, 0.0, 0.0, True
    for b, ref in zip(frames_idx, ref_outs):
        flips += int(np.sum(fits[b] != ref["fits"]))
        ncoef += ref["fits"].size
        rt = ref["thb"]
        nz = rt != 0
        thb_rel = max(thb_rel, float(np.max(np.abs(thb[b][nz] - rt[nz]) / np.abs(rt[nz]), initial=0.0)))
        ok = ~np.isnan(ref["so2"])
        nan_eq &= bool(np.array_equal(np.isnan(so2[b]), ~ok))
        so2_abs = max(so2_abs, float(np.max(np.abs(so2[b][ok] - ref["so2"][ok]), initial=0.0)))
    return {"vs": "oracle/oximap_oracle.py (pinned bit-for-bit to the reference's outputs)",
            "frames": list(frames_idx), "coefficients": ncoef, "fit_count_flips": flips, "max_thb_rel": thb_rel,
            "max_so2_abs": so2_abs, "so2_nan_pattern_equal": nan_eq,
            "pass": flips == 0 and nan_eq and thb_rel <= 1e-4 and so2_abs <= 1e-5}


def schedule_check(eng, frames, out) -> dict:
    """Runtime flip detector for the EM precision schedule: the whole timed
    batch through the all-fp64 EM schedule (HybridMapEngine.audit), every
    low-pass coefficient's fit count compared, maps compared (outside the
    timed region)."""
    return {"vs": "all-fp64 EM schedule (em_lead=None) on the whole timed batch (HybridMapEngine.audit)",
            **eng.audit(frames, out)}


def dropin_record(frames_host: np.ndarray, levels: int, n_seq: int) -> dict:
    """The reference user's own calls at config 3 (fp64 drop-in path,
    pipeline.py:117-245): estimate_frame latency including the (H, W, 26)
    fp64 SpectralCube it returns, and estimate_sequence throughput over host
    frames (maps as fp64 ConcentrationMaps in host memory)."""
    import paper_1706_07263_b200 as ox

    sens, basis = operators()
    cfg = ox.PipelineConfig(n_levels=levels)
    imgs = [ox.RgbImage(f.astype(np.float64)) for f in frames_host[:n_seq]]
    ox.estimate_frame(imgs[0], sens, basis, cfg)  # warm
    lat = []
    for k in range(3):
        t0 = time.perf_counter()
        cube, cmap = ox.estimate_frame(imgs[k % len(imgs)], sens, basis, cfg)
        lat.append(time.perf_counter() - t0)
    del cube, cmap
    list(ox.estimate_sequence(imgs[:2], sens, basis, cfg))  # warm
    timings = []
    t0 = time.perf_counter()
    n = sum(1 for _ in ox.estimate_sequence(imgs, sens, basis, cfg, timings=timings))
    dt = time.perf_counter() - t0
    H, W = frames_host.shape[1:3]
    return {"estimate_frame_ms": 1e3 * statistics.median(lat),
            "estimate_frame_note": f"one {H}x{W} host fp64 frame -> SpectralCube ({H * W * 26 * 8 / 1e6:.0f} MB fp64) "
                                   "+ fp64 ConcentrationMap in host memory, median of 3",
            "estimate_sequence_fps": n / dt, "estimate_sequence_frames": n,
            "estimate_sequence_note": "host fp64 RgbImage frames -> fp64 ConcentrationMaps (pipelined: H2D / "
                                      "kernels / D2H of consecutive frames overlap)"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1706_07263_b200 import synth

    sens, basis = operators()
    frames = [synth.phantom_rgb_f32(args.height, args.width, s, sens, basis, texture_density=args.texture)
              .astype(np.float32) for s in range(2)]
    from threadpoolctl import threadpool_limits

    from oracle import oximap_oracle as O

    threads = O.default_threads()
    times = []
    with threadpool_limits(limits=1):
        for i in range(args.warmup + args.steps):
            f = frames[i % 2].astype(np.float64)
            t0 = time.perf_counter()
            O.estimate_frame(f, sens.c, basis.xi, n_levels=args.levels, threads=threads, want_cube=False)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                times.append(dt)
    total = sum(times)
    value = len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "run": {"frames_per_step": 1, "arm": "oracle port of the reference on host cores"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"1 frame per step ({args.height}x{args.width}, n={args.levels}) through the "
                                   "oracle port of the reference (bit-identical outputs), threads=all cores, BLAS 1"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- ours
def probe_peaks(lib, torch, dev):
    """Measured fp64-FMA and MUFU-lg2 pipe peaks on this GPU (probe.cu)."""
    import ctypes

    sm = torch.cuda.get_device_properties(dev).multi_processor_count
    sink64 = torch.zeros(256, dtype=torch.float64, device=dev)
    sink32 = torch.zeros(256, dtype=torch.float32, device=dev)
    out = {}
    for name, fn, sink, iters in (("fp64_fma", lib.oxm_probe_fp64_fma, sink64, 400),
                                  ("mufu_lg2", lib.oxm_probe_mufu_lg2, sink32, 400)):
        ops = ctypes.c_double()
        s = torch.cuda.current_stream()
        best = float("inf")
        for rep in range(4):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn(sm * 8, iters, sink.data_ptr(), ctypes.byref(ops), s.cuda_stream)
            b.record()
            b.synchronize()
            if rep:
                best = min(best, a.elapsed_time(b) * 1e-3)
        out[name] = ops.value / best
    return out


def copy_bandwidth(torch, dev) -> dict:
    """Pinned H2D / D2H GB/s, each direction alone and both running at once
    (512 MiB per copy, best of 3 rounds; tools/pcie_probe.py has the full
    probe).  The e2e bound is the best schedule of a step's copies: both
    directions at the concurrent rate while both have bytes left, the
    remainder of the larger one at its alone rate."""
    n = 512 * 2**20
    h_in, h_out = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a, d_b = torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def rate(h2d: bool, d2h: bool) -> float:
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(4):
                if h2d:
                    with torch.cuda.stream(s1):
                        d_a.copy_(h_in, non_blocking=True)
                if d2h:
                    with torch.cuda.stream(s2):
                        h_out.copy_(d_b, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, 4 * n / (time.perf_counter() - t0) / 1e9)
        return best

    return {"h2d_alone_gbs": rate(True, False), "d2h_alone_gbs": rate(False, True), "concurrent_gbs": rate(True, True)}


def pcie_bound(frames: float, h2d_bytes: float, d2h_bytes: float, bw: dict) -> float:
    """Frames/s if a step's copies ran at the measured rates (compute hidden)."""
    both = min(h2d_bytes, d2h_bytes)
    rest_rate = bw["h2d_alone_gbs"] if h2d_bytes >= d2h_bytes else bw["d2h_alone_gbs"]
    t = both / (bw["concurrent_gbs"] * 1e9) + abs(h2d_bytes - d2h_bytes) / (rest_rate * 1e9)
    return frames / t


def init_dist(args):
    """One process per GPU.  Under torchrun WORLD_SIZE must equal --gpus;
    OXM_BENCH_BACKEND=gloo runs several ranks on one GPU (functional check of
    the multi-rank path, not a scaling number)."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one process per GPU)")
    backend = os.environ.get("OXM_BENCH_BACKEND", "nccl")
    if args.plumbing_check:
        if world > 1:
            dist.init_process_group("gloo")
        return world, rank, torch.device("cpu")
    ndev = torch.cuda.device_count()
    if world > 1:
        if backend == "nccl" and ndev < world:
            raise SystemExit(f"bench.py: {world} ranks need {world} GPUs over NCCL, {ndev} visible "
                             "(OXM_BENCH_BACKEND=gloo shares one GPU for a functional check)")
        local = local % ndev
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local if world > 1 else torch.cuda.current_device())
    torch.cuda.set_device(dev)
    return world, rank, dev


def gathered_leg(args, world, step, gather_maps, dev) -> dict:
    """the same steps with every rank's THb + SO2 maps gathered
    to rank 0 (NCCL point-to-point over NVLink; the identity at N = 1),
    device-timed, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1706_07263_b200.parallel import max_over_ranks

    if world > 1:
        dist.barrier()
    if dev.type == "cuda":
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            step()
            gather_maps()
        b.record()
        b.synchronize()
        dt = a.elapsed_time(b) * 1e-3
    else:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
            gather_maps()
        dt = time.perf_counter() - t0
    dt = max_over_ranks(dt, dev if dev.type == "cuda" else None)
    return {"value": world * args.batch * args.steps / dt, "unit": UNIT, "ms_per_step": 1e3 * dt / args.steps,
            "bytes_to_root_per_step": (world - 1) * args.batch * args.height * args.width * 8,
            "how": "each step: the hybrid batch on every rank, then parallel.gather_chunk_to_root of its THb and "
                   "SO2 maps (NCCL p2p) to rank 0"}


def run_plumbing_check(args):
    """CPU dry run of the multi-rank bench plumbing (spawn, barrier, max over
    ranks, map gather) with a host surrogate for the kernels: exercised by
    tests/test_bench_plumbing.py without a GPU.  Prints a line marked
    "plumbing_check" (not a measurement)."""
    import torch

    from paper_1706_07263_b200.parallel import gather_chunk_to_root, max_over_ranks

    world, rank, dev = init_dist(args)
    B, H, W = args.batch, args.height, args.width
    thb = torch.full((B, H, W), float(rank), dtype=torch.float32)
    so2 = torch.zeros((B, H, W), dtype=torch.float32)

    def step():
        thb.add_(0.0)

    got = {}

    def gather():
        r = gather_chunk_to_root(thb, world * B, B, 0)
        gather_chunk_to_root(so2, world * B, B, 0)
        if r is not None:
            got["first"] = [(a, float(t[0, 0, 0])) for a, t in r]

    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = max_over_ranks(time.perf_counter() - t0)
    g = gathered_leg(args, world, step, gather, dev)
    if rank == 0:
        print(json.dumps({"plumbing_check": True, "metric": METRIC, "n_gpus": world, "steps": args.steps,
                          "value": world * B * args.steps / dt, "gathered": g, "gathered_blocks": got.get("first")}),
              flush=True)
    import torch.distributed as dist

    if world > 1:
        dist.destroy_process_group()


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, dev = init_dist(args)

    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200 import _native
    from paper_1706_07263_b200.parallel import gather_chunk_to_root, max_over_ranks

    lib = _native.load()
    sens, basis = operators()
    H, W, n, B = args.height, args.width, args.levels, args.batch
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev)
    frames = make_frames(B, H, W, args.texture, rank, dev)
    out = eng.allocate(B, H, W, fits=True)
    nll = B * (-(-H // 2**n)) * (-(-W // 2**n))
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        eng.launch(frames, out)
    eng.check_flags(out)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        clk.mark(True)
        start.record(stream)
        for k in range(args.steps):
            eng.launch(frames, out, stage_events=ev[k])
        stop.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
    if world > 1:
        dist.barrier()
    elapsed = start.elapsed_time(stop) * 1e-3
    elapsed_max = max_over_ranks(elapsed, dev)
    stage_s = [statistics.mean(e[i].elapsed_time(e[i + 1]) * 1e-3 for e in ev) for i in range(5)]
    fits_total = int(out.fits.sum().item())
    emc = eng.em_counters(B, H, W)  # the last timed launch's EM work split
    eng.check_flags(out)
    clocks = clk.summary()

    # ---- gathered: the same steps plus the maps of every rank on rank 0
    gout = eng.allocate(B, H, W)
    gathered = gathered_leg(
        args, world, lambda: eng.launch(frames, gout),
        lambda: (gather_chunk_to_root(gout.thb, world * B, B, 0), gather_chunk_to_root(gout.so2, world * B, B, 0)),
        dev)
    del gout

    # ---- end to end: pinned host frames -> maps in pinned host memory
    e2e = None
    if not args.no_e2e:
        host_in = frames.cpu().pin_memory()
        thb_h = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
        so2_h = torch.empty((B, H, W), dtype=torch.float32).pin_memory()
        state = {}
        chunk = 4
        eng.maps_from_host(host_in, thb_h, so2_h, chunk=chunk, _state=state)  # warm
        e2e_steps = max(2, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            eng.maps_from_host(host_in, thb_h, so2_h, chunk=chunk, _state=state)
        e2e_dt = max_over_ranks(time.perf_counter() - t0, dev)
        e2e = {"value": world * B * e2e_steps / e2e_dt, "unit": UNIT,
               "h2d_bytes_per_step": B * H * W * 3 * 4, "d2h_bytes_per_step": B * H * W * 2 * 4,
               "steps": e2e_steps, "chunk_frames": chunk, "api": "HybridMapEngine.maps_from_host -> oxm_hybrid_maps_f32"}
        # the CLI's own input format: 16-bit PPM rasters (io.py:88-162), decoded on the device
        scale = float(frames.max().item()) / 65535.0
        counts = torch.clamp(torch.round(frames / scale), 0, 65535).to(torch.int32).to(torch.uint16)
        host_u16 = counts.cpu().pin_memory()
        del counts
        eng.maps_from_host(host_u16, thb_h, so2_h, chunk=chunk, _state=state, scale=scale, big_endian=False)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            eng.maps_from_host(host_u16, thb_h, so2_h, chunk=chunk, _state=state, scale=scale, big_endian=False)
        e2e_dt16 = max_over_ranks(time.perf_counter() - t0, dev)
        e2e["ppm_u16"] = {"value": world * B * e2e_steps / e2e_dt16, "unit": UNIT,
                          "h2d_bytes_per_step": B * H * W * 3 * 2, "d2h_bytes_per_step": B * H * W * 2 * 4,
                          "api": "maps_from_host(uint16 PPM counts) -> oxm_hybrid_maps_u16"}
        bw = copy_bandwidth(torch, dev)
        for rec in (e2e, e2e["ppm_u16"]):
            bound = world * pcie_bound(B, rec["h2d_bytes_per_step"], rec["d2h_bytes_per_step"], bw)
            rec["pcie_bound"] = bound
            rec["frac_of_pcie_bound"] = rec["value"] / bound
        e2e["copy_bandwidth"] = bw

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- correctness of what was timed (outside every timed region)
    sched = schedule_check(eng, frames, out)
    cpu = None
    sample = frames[:CPU_SAMPLE_FRAMES if world == 1 and not args.no_cpu else 1].cpu().numpy()
    if world == 1 and not args.no_cpu:
        cpu, ref_outs = cpu_baseline(sample, n, CPU_OTHER_FRAMES)
    else:
        _, ref_outs = _oracle_frames(sample, n, os.cpu_count() or 1, 1)
    parity = parity_record(out, ref_outs, list(range(len(ref_outs))))
    parity["schedule"] = sched
    dropin = None
    if world == 1 and not args.no_dropin:
        dropin = dropin_record(frames[:DROPIN_SEQ_FRAMES].cpu().numpy(), n, DROPIN_SEQ_FRAMES)

    peaks = probe_peaks(lib, torch, dev)
    mp = ROOT / "MEASURED_PEAKS.json"
    hbm = json.loads(mp.read_text()).get("hbm_gbs") if mp.exists() else None
    # per-stage algorithmic work
    px = B * H * W
    bytes_ll = px * 12 + nll * (3 * 8 + 3 * 8 + 1)  # frame in; ybar, fit #1, exact-block flag out
    lead_mufu = emc["lead_fits"] * MUFU_PER_LEAD_FIT
    px_lg2 = px * 26
    stage_t = {"ll_kernel": stage_s[0], "em_lead": stage_s[1], "em": stage_s[2], "px_f32_kernel": stage_s[3],
               "fixup": stage_s[4]}
    fp64_rate = peaks["fp64_fma"]  # fp64-pipe instructions (lane ops) per second, DFMA probe
    rooflines = {
        "ll_kernel": {"bound": "hbm", "achieved": bytes_ll / stage_s[0] / 1e9, "peak": hbm, "unit": "GB/s",
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                      "work": f"{px} px x 12 B in + {nll} coefficients x 49 B out (ybar, fit #1, exact flag)"},
        "em_lead": {"bound": "xu", "achieved": lead_mufu / stage_s[1] / 1e12 if stage_s[1] > 0 else None,
                    "peak": peaks["mufu_lg2"] / 1e12, "unit": "TMUFU/s",
                    "peak_source": "MUFU lg2 probe (oxm_probe_mufu_lg2) in this run",
                    "kernels": "em_lead_kernel (fp32 fits)",
                    "work": f"{emc['lead_fits']} fp32 fits x {MUFU_PER_LEAD_FIT} MUFU (ex2 + lg2 per band)"},
        "em": {"bound": "fp64 pipe", "achieved": emc["tail_fits"] * FP64_INST_PER_FIT / stage_s[2] / 1e12,
               "peak": fp64_rate / 1e12, "unit": "T fp64-pipe lane-ops/s",
               "peak_source": "fp64 DFMA probe (oxm_probe_fp64_fma) in this run: one DFMA per lane per pipe slot",
               "kernels": "em_persistent_kernel (fp64 tail)",
               "work": f"{emc['tail_fits']} fp64 fits (incl. {emc['restarts']} exact-mode restarts) x "
                       f"{FP64_INST_PER_FIT} fp64-pipe thread instructions per fit (DFMA/DADD/DMUL/DSETP; ncu "
                       f"SASS counts of this batch's tail launch / its fits, profiles/r02_em_tail_sass_counts.txt)",
               "flops": {"achieved": emc["tail_fits"] * FLOPS_PER_FIT / stage_s[2] / 1e12,
                         "peak": 2 * fp64_rate / 1e12, "unit": "TFLOP/s",
                         "per_fit": FLOPS_PER_FIT, "note": "FMA = 2 flops, DADD/DMUL = 1, compares 0 (same counts)"}},
        "px_f32_kernel": {"bound": "xu", "achieved": px_lg2 / stage_s[3] / 1e12, "peak": peaks["mufu_lg2"] / 1e12,
                          "unit": "Tlg2/s", "peak_source": "MUFU lg2 probe (oxm_probe_mufu_lg2) in this run",
                          "kernels": "px_f32_kernel", "work": f"{px} px x 26 lg2"},
        "fixup": {"bound": "latency", "achieved": None, "peak": None, "unit": None,
                  "kernels": "exact pass (em_persistent_kernel on the block list) + px_fallback_kernel (deferred)",
                  "note": f"all-fp64 EM of {emc['exact_blocks']} blocks, then fp64 recompute of "
                          f"{emc['deferred_px']} deferred pixels (of {emc['queued_px']} fallback pixels; "
                          f"the rest are finished in place by px_f32_kernel)"},
    }
    for k, r in rooflines.items():
        r["ms"] = stage_t[k] * 1e3
        r["frac"] = r["achieved"] / r["peak"] if r["peak"] and r["achieved"] is not None else None
    rooflines["em"]["flops"]["frac"] = rooflines["em"]["flops"]["achieved"] / rooflines["em"]["flops"]["peak"]
    traffic = {}
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        per_frame = json.loads(tf.read_text()).get("dram_bytes_per_frame", {})
        traffic = {k: v * B for k, v in per_frame.items()}
    dominant = max(stage_t, key=stage_t.get)
    roof = dict(rooflines[dominant])
    roof["kernel"] = dominant
    roof["traffic"] = traffic.get(dominant)
    roof["traffic_note"] = "ncu dram__bytes_read+write per launch (profiles/traffic.json, scaled to this batch)"

    value = world * B * args.steps / elapsed_max
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 low-pass; EM f32 lead-in + f64 tail (fit counts exact); f32 per-pixel (f64 fallback)",
        "data": "synthetic (tissue phantoms, seeded; forward model + noise on GPU)",
        "config": workload_config(args),
        "run": {"frames_per_step_per_gpu": B, "global_batch": world * B,
                "l2": f"inputs {B * H * W * 12 / 1e6:.0f} MB per step > 126 MB L2 (no flush needed)",
                "parallelism": f"frame-sharded x{world}, no data-path collective"},
        "gathered": gathered,
        "roofline": roof,
        "stage_rooflines": rooflines,
        "parity": parity,
        "fits_per_coefficient": fits_total / nll,
        "em_work_last_step": {**emc, "coefficients": nll},
        "probes": {"fp64_fma_T/s": peaks["fp64_fma"] / 1e12, "mufu_lg2_T/s": peaks["mufu_lg2"] / 1e12},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "dropin": dropin,
        "gpu_launches": HybridMapLaunches * args.steps,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# EM tail work per fp64 fit, measured rather than assumed: ncu's
# SASS-level thread-instruction counts of the tail launch of this exact bench
# batch (tools/ncu_thread_counts.py -> profiles/r02_em_tail_sass_counts.txt)
# divided by its 60,605,987 fits -- DFMA + DADD + DMUL + DSETP = 714.3
# fp64-pipe instructions per fit, 1239.4 flops (FMA = 2).  Per band that is the
# exp (DADD + 3 DFMA + DMUL + DFMA), its argument (2 DFMA), C e (3 DFMA),
# e + G r (3 DFMA), the eps clamp (DSETP), the table log (DFMA + 3 DFMA + DMUL
# + 2 DFMA + DADD) and the fit (3 DFMA), plus the per-step norms.  `frac` =
# fp64-pipe instructions issued / the DFMA probe's rate, the quantity ncu
# reports as sm__inst_executed_pipe_fp64.
FP64_INST_PER_FIT = 714.3
FLOPS_PER_FIT = 1239.4
MUFU_PER_LEAD_FIT = 2 * 26  # fp32 lead-in: one ex2 and one lg2 per band
CPU_OTHER_FRAMES = 3   # frames for the slower reference thread setting (threads=1, BLAS=nproc)
DROPIN_SEQ_FRAMES = 16
DEFAULT_BATCH = 128
# frames per step per GPU: 64 / 128 / 256 frames per launch measured 12.86 / 13.04 /
# 13.14 k fps (fewer kernel ramp-ups and drains per frame); 128 keeps the
# N = 8 gather to rank 0 at 17 GB per step
# kernels launched per step: zero_counters, ll_tma (+ fit #1), em_lead, em_persistent (tail),
# px_f32 (+ in-warp fp64 fallback), exact pass, px_fallback (deferred)
HybridMapLaunches = 7


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N local ranks (127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(pathlib.Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "LOCAL_RANK" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.plumbing_check:
        run_plumbing_check(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
