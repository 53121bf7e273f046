"""Builds the sm_100a shared library behind include/oximap_b200.h.

Plain nvcc (no torch extension machinery): every ``csrc/*.cu`` is compiled
with ``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and linked into
``paper_1706_07263_b200/_lib/liboximap_b200.so``, which lives in-tree so it
travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import shutil
import subprocess

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIBDIR = PKG / "_lib"
LIBNAME = "liboximap_b200.so"
LIBPATH = LIBDIR / LIBNAME
OBJDIR = ROOT / "build" / "obj"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC,-fvisibility=hidden",
    "-Xptxas",
    "-v",
    "--cudart",
    "static",
    "-I",
    str(INCLUDE),
    "-I",
    str(CSRC),
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build the CUDA library")
    return cand


def _sources() -> list[pathlib.Path]:
    return sorted(CSRC.glob("*.cu"))


def _deps() -> list[pathlib.Path]:
    return _sources() + sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h")) + [pathlib.Path(__file__)]


def up_to_date() -> bool:
    if not LIBPATH.exists():
        return False
    t = LIBPATH.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in _deps())


def build(force: bool = False, verbose: bool = False, defines: tuple[str, ...] = (),
          out: pathlib.Path | None = None) -> pathlib.Path:
    """Compile (if stale) and return the path of the shared library.
    ``defines``/``out`` build a tuning variant elsewhere (tools/em_variants.py)."""
    libpath = LIBPATH if out is None else out
    if out is None and not defines and not force and up_to_date():
        return LIBPATH
    nvcc = _nvcc()
    objdir = OBJDIR if out is None else out.parent / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    libpath.parent.mkdir(parents=True, exist_ok=True)
    logs = {}

    def compile_one(src: pathlib.Path) -> pathlib.Path:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs[src.name] = res.stdout + res.stderr
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, _sources()))
    tmp = libpath.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, libpath)
    (libpath.parent / "ptxas.log" if out is not None else ROOT / "build" / "ptxas.log").write_text(
        "\n".join(f"== {k}\n{v}" for k, v in sorted(logs.items())))
    if verbose:
        for k, v in sorted(logs.items()):
            print(f"== {k}\n{v}")
    return libpath


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
