"""Build the sm_100a C-ABI library ``libkfp.so`` in-tree with nvcc (no JIT, no torch extension).

``libkfp_mut.so`` is a test-only mutant of the same sources (``-DKFP_MUTATE``: one coefficient of the step
kernel perturbed by 1e-3, kfp_api.cu base_params); tests/test_gpu_parity.py checks that the parity suite
fails on it (the suite is sensitive to a plausible kernel mistake).  Never loaded by the product path."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "kfp_api.cu")]
DEPS = SRC + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "kfp.h")]
LIB = os.path.join(HERE, "libkfp.so")
MUTANT = os.path.join(HERE, "libkfp_mut.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in DEPS)


def _cmd(lib: str, extra=()):
    return [NVCC, *FLAGS, *extra, "--cudart=static", "-o", lib, *SRC]


def build(force: bool = False, verbose: bool = False, mutant: bool = True) -> str:
    """Compile libkfp.so (and the test-only mutant) when a source is newer; both nvcc runs in parallel."""
    jobs = []
    if force or needs_build(LIB):
        jobs.append((LIB, subprocess.Popen(_cmd(LIB), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    if mutant and (force or needs_build(MUTANT)):
        jobs.append((MUTANT, subprocess.Popen(_cmd(MUTANT, ["-DKFP_MUTATE"]), stdout=subprocess.PIPE,
                                              stderr=subprocess.PIPE, text=True)))
    failed = []
    for lib, p in jobs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            failed.append(os.path.basename(lib))
        elif verbose and lib == LIB:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError(f"nvcc failed building {', '.join(failed)}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, mutant="--no-mutant" not in sys.argv)
    print(LIB)
