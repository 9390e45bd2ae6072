#!/bin/bash
# build a variant of libevogp.so with extra nvcc flags into variants/<name>/libevogp.so
# usage: tools/build_variant.sh NAME "-DFLAG1 -DFLAG2"
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $ROOT/variants/$NAME
/usr/local/cuda/bin/nvcc $FLAGS -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -ftz=false \
  -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -shared -o $ROOT/variants/$NAME/libevogp.so \
  $ROOT/paper_2501_17168_b200/csrc/kernels.cu $ROOT/paper_2501_17168_b200/csrc/paired.cu $ROOT/paper_2501_17168_b200/csrc/variation.cu $ROOT/paper_2501_17168_b200/csrc/tensorize_dev.cu $ROOT/paper_2501_17168_b200/csrc/capi.cu $ROOT/paper_2501_17168_b200/csrc/tensorize.cpp
echo built variants/$NAME
