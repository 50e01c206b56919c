#!/bin/bash
# build a libgirg_<tag>.so variant with extra -D flags:  tools/build_variant.sh tag -DGIRG_X=1 ...
tag=$1; shift
cd $(dirname $0)/..
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -shared "$@" -o paper_1905_06706_b200/libgirg_$tag.so paper_1905_06706_b200/csrc/girg.cu
