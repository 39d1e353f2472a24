#!/bin/bash
# Checked build of libdgx_cuda.so (device-side bounds checks, DGX_ASSERT in
# csrc/dgx_kernel.cuh) into exp/libdgx_checked.so. compute-sanitizer is closed
# on the GPU pool, so the tests run against this build instead:
#   DGX_LIBRARY=exp/libdgx_checked.so python -m pytest tests -m gpu
set -e
cd "$(dirname "$0")/../paper_2306_08132_b200/csrc"
mkdir -p ../../exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared \
  -DDGX_CHECKS dgx_kernels.cu dgx_capi.cu dgx_peak.cu dgx_mesh_host.cu dgx_drop.cu -o ../../exp/libdgx_checked.so
echo built exp/libdgx_checked.so
