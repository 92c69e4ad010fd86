#!/bin/bash
# Build experimental variants of libacpf.so into exp/ (git-ignored), e.g.
#   tools/build_exp.sh nocomp -DACPF_EXP_NOCOMPUTE
set -e
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O3 -shared -I include "$@" -o exp/libacpf_$name.so \
  ${SRC:-paper_2605_14103_b200/csrc}/*.cu ${SRC:-paper_2605_14103_b200/csrc}/*.cpp -lcusolver -lcublas
