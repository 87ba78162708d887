"""Build the sm_100a C-ABI library ``libkfp.so`` in-tree with nvcc (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "kfp_api.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "kfp_fused.cuh"), os.path.join(HERE, "csrc", "kfp_window.cuh"), os.path.join(HERE, "csrc", "kfp_col.cuh"), os.path.join(HERE, "csrc", "kfp_device.cuh"), os.path.join(ROOT, "include", "kfp.h")]
LIB = os.path.join(HERE, "libkfp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [NVCC, *FLAGS, "--cudart=static", "-o", LIB, *SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libkfp.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
