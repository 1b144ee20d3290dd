#!/bin/bash
# build_variant.sh <csrc dir> <out .so> [extra nvcc flags] — dev tool for A/B timing
src=$1; out=$2; shift 2
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  -I/root/repo/include -I$src "$@" -o $out $src/kstep.cu $src/kernels.cu $src/sim_api.cu 2>&1 | grep -E "error"
exit 0
