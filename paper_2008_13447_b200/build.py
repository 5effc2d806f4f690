"""Build libvlmp.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRCS = [os.path.join(HERE, "csrc", f) for f in ("profile.cu", "filter32.cu", "readout.cu", "pruned.cu", "session.cu")]
SRC = SRCS[0]   # the tile kernels (variant builds)
HDRS = [os.path.join(HERE, "csrc", "vlmp_internal.cuh")]
OUT = os.path.join(HERE, "libvlmp.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", f"-I{os.path.join(ROOT, 'include')}"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    deps = SRCS + HDRS + [os.path.join(ROOT, "include", "vlmp.h")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, *SRCS]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
