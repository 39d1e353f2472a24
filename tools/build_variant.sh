#!/bin/bash
# Build an A/B variant of libdgx_cuda.so with extra -D flags into exp/:
#   tools/build_variant.sh NAME -DFOO=1 ...   -> exp/libdgx_NAME.so (select with DGX_LIBRARY=exp/libdgx_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p exp
src=paper_2306_08132_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -shared "$@" \
  $src/dgx_kernels.cu $src/dgx_capi.cu $src/dgx_peak.cu $src/dgx_mesh_host.cu $src/dgx_drop.cu -o exp/libdgx_$name.so
