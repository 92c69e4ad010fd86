#!/bin/bash
# Build experimental variants of libacpf.so into exp/ (git-ignored, gpurun-ignored), e.g.
#   tools/build_exp.sh nocomp -DACPF_EXP_NOCOMPUTE
#   tools/build_exp.sh dbg -DACPF_DEBUG_BOUNDS      # bounds-checked build
# and run against one with ACPF_LIB=exp/libacpf_<name>.so
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p exp
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O3 -shared -I include "$@" -o exp/libacpf_$name.so \
  ${SRC:-paper_2605_14103_b200/csrc}/*.cu ${SRC:-paper_2605_14103_b200/csrc}/*.cpp -lcusolver
