"""Build libwoit.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2201_00094_b200.build        # or __graft_entry__.build()

Objects go to build/, the shared library to paper_2201_00094_b200/libwoit.so
(git-ignored, shipped to the GPU box by gpurun). ptxas resource usage of every
kernel is written to build/ptxas.log.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(REPO, "build")
LIB = os.path.join(PKG, "libwoit.so")
SOURCES = ("frame.cu", "batch.cu", "binning.cu", "synth.cu", "resolve.cu", "build_atomic.cu", "baselines.cu", "cast.cu", "abi.cu")
HEADERS = ("common.cuh", "frame.cuh", "packing.cuh", "internal.cuh")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I" + os.path.join(REPO, "include")]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; libwoit.so cannot be built")
    return exe


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile and link. ``defines`` (e.g. ("WOIT_UNROLL=4",)) build a tuning variant into
    its own object directory and ``out`` library."""
    build_dir = BUILD if not defines else os.path.join(BUILD, "v_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(build_dir, exist_ok=True)
    dflags = ["-D" + d for d in defines]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(REPO, "include", "woit.h")]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc(), *ARCH, *FLAGS, *dflags, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    logs = []
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        for cmd, r in pool.map(run, jobs):
            logs.append(r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if logs:
        with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    if force or jobs or _stale(out, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", out, *objs, "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of libwoit.so failed")
    if verbose:
        print(out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
