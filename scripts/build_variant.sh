#!/bin/bash
# Build an experiment variant of the library: scripts/build_variant.sh <name> <nvcc flags...>
# -> paper_2603_02599_b200/libsun_b200_<name>.so (load it with SUN_LIB=...)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2603_02599_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -cudart static --expt-relaxed-constexpr "$@" -o ../libsun_b200_$name.so sun_capi.cu
