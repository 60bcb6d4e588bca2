"""In-tree build of libdash_b200.so for sm_100a (nvcc, no JIT cache).

    python -m paper_2305_18376_b200.build        # rebuild if sources changed
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
INCLUDE = HERE.parent / "include"
LIB = HERE / "libdash_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]
SOURCES = ["dash_update.cu"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-I", str(INCLUDE), "-o", str(LIB) + ".tmp",
           *[str(CSRC / s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = HERE / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(str(LIB) + ".tmp", LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_host_ext(force: bool = False, verbose: bool = False) -> Path:
    """The host-side gather helper (_dashhost, CPython extension, gcc): walks a
    batch's per-slice arrays in C for StreamState.update(UpdateBatch)."""
    import sysconfig
    src = CSRC / "host_gather.c"
    out = HERE / ("_dashhost" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = [os.environ.get("CC", "gcc"), "-O3", "-shared", "-fPIC", "-pthread", "-I", sysconfig.get_paths()["include"],
           str(src), "-o", str(out) + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("gcc failed on host_gather.c")
    os.replace(str(out) + ".tmp", out)
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build_host_ext(force="--force" in sys.argv, verbose=True)
    build_library(force="--force" in sys.argv, verbose=True)
