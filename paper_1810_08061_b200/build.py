"""Build libskb.so (all CUDA sources under csrc/) in-tree for sm_100a.

Usage: python -m paper_1810_08061_b200.build   (or __graft_entry__.build()).
The shared library is written next to this file so it travels with the
repository snapshot to the GPU box; nothing is installed into site-packages.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("SKB_BUILD_OUT") or os.path.join(HERE, "libskb.so")   # override: A/B or trace builds
REPO = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--use_fast_math", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "-I", os.path.join(REPO, "include")]
if os.environ.get("SKB_TRACE") == "1":   # clock64 role-event tracing (tools/trace_c1.py)
    FLAGS.append("-DSKB_TRACE_ENABLED")
    FLAGS.append("-DSKB_STREAM_TIMING")    # stream kernel phase totals (tools/stream_phases.py)


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    mtime = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) \
        + glob.glob(os.path.join(REPO, "include", "*.h"))
    return any(os.path.getmtime(p) > mtime for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "build", os.path.basename(LIB)[:-3]) if os.environ.get("SKB_BUILD_OUT") \
        else os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode:
            sys.stderr.write(res.stdout + res.stderr)
        if res.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda", "-lcublas", "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("link of libskb.so failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
