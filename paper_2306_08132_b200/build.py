"""Build libdgx_cuda.so in-tree for sm_100a (nvcc; no JIT, no torch extension).

The kernels TU is compiled with --fmad=false so the forward path performs
exactly the reference's IEEE operation sequence (bit-exact contact decisions);
the adjoint opts into FMA explicitly via fma()."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libdgx_cuda.so")
SOURCES = ["dgx_kernels.cu", "dgx_capi.cu", "dgx_peak.cu", "dgx_mesh_host.cu", "dgx_drop.cu"]
HEADERS = ["dgx_math.h", "dgx_geom.h", "dgx_mesh.h", "dgx_mesh_host.h", "dgx_adjoint.cuh", "dgx_kernel.cuh", "dgx_sdf_fast.cuh", "dgx_drop.cuh", "dgx_lane_adj.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(PKG, "..", "include", "dgx.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", OUT]
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
