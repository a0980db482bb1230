"""Build libustfwi_b200.so in-tree (sm_100a) with nvcc.

Usage: python -m paper_2102_00755_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libustfwi_b200.so")
SOURCES = ["engine.cu", "kernels.cu", "passes.cu", "passes_y.cu", "lbfgs.cu", "resample.cu", "host_setup.cpp", "host_fft.cpp"]
HEADERS = ["passes.cu", "fft_smem.cuh", "fft_reg.cuh", "async_copy.cuh", "kernels.cuh", "host_setup.hpp", os.path.join("..", "..", "include", "ustfwi_capi.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return False


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs, procs = [], []
    for src in SOURCES:  # translation units compile in parallel
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{out}\n{err}")
        if verbose:
            sys.stderr.write(err)
    tmp = LIB + ".tmp"
    # --no-undefined: a missing symbol fails the build, not the first dlopen on the GPU box
    cmd = [NVCC, *ARCH, "-shared", *objs, "-o", tmp, "-ldl", "-lpthread", "-lrt", "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
