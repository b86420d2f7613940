"""In-tree build of the sm_100a shared library (no JIT cache: the .so lives in
the package directory so it travels with the repo snapshot to the GPU box).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false ...

``-fmad=false`` forbids implicit FMA contraction so that every rounding in
the kernels is the one written in the source (the fp64 path relies on it to
stay bit-identical to the reference's x86 build; the fp32/u8 paths spell out
their FMAs explicitly); ``-ffp-contract=off`` does the same for host code
(the tone thresholds, the metric's host Lab).
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

from ._lib import LIB_PATH, PKG_DIR

CSRC = os.path.join(PKG_DIR, "csrc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    mtime = os.path.getmtime(LIB_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(PKG_DIR, "..", "include", "warmgray_b200.h"))
    return any(os.path.getmtime(p) > mtime for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every .cu under csrc/ into _build/libwarmgray_b200.so."""
    if not force and not _stale():
        return LIB_PATH
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
           "-Xcompiler", "-fPIC,-fvisibility=hidden,-O3,-ffp-contract=off", "-shared", "-o", tmp, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
