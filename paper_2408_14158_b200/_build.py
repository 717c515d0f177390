"""In-tree build of libhfr.so (sm_100a) — no JIT cache, the .so travels with gpurun."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "hfr_runtime.cu")]
# every source the library is built from (the list missed hfr_nvls.cuh)
DEPS = sorted(set(SRC + glob.glob(os.path.join(PKG, "csrc", "*.cu")) + glob.glob(os.path.join(PKG, "csrc", "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h"))))
LIB = os.path.join(PKG, "libhfr.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# No --use_fast_math (keeps IEEE RNE, no FTZ: DESIGN.md reading R4).
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    """Build libhfr.so in-tree (one library, no variants: every behaviour
    switch is a field of hfr_config_t)."""
    lib = LIB
    if force or stale():
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [NVCC, *FLAGS, "-o", tmp, *SRC]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libhfr.so")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
