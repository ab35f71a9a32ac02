#!/bin/sh
# Builds libspamm_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).
set -e
cd "$(dirname "$0")"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC ${SPAMM_PTXAS_V:+-Xptxas -v} --shared -ccbin /usr/bin/g++ \
      -o libspamm_b200.so abi.cu tree.cu plan.cu execute.cu pipeline.cu exchange.cu -ldl "$@"
