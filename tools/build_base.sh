#!/bin/bash
# build libgirg_m_base.so from a git revision (default HEAD) for A/B sweeps: tools/build_base.sh [rev] [tag]
rev=${1:-HEAD}; tag=${2:-m_base}
cd $(dirname $0)/..
tmp=$(mktemp -d)
mkdir -p $tmp/paper_1905_06706_b200/csrc $tmp/include
for f in $(git ls-tree --name-only $rev paper_1905_06706_b200/csrc/); do git show $rev:$f > $tmp/$f; done
git show $rev:include/girg.h > $tmp/include/girg.h
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -shared -o paper_1905_06706_b200/libgirg_$tag.so $tmp/paper_1905_06706_b200/csrc/girg.cu
rm -rf $tmp
