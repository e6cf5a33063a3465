#!/bin/bash
# Build A/B variants of libdr.so into paper_1906_11633_b200/variants/ (selected with DR_LIB=variants/<name>.so).
cd "$(dirname "$0")/.."
mkdir -p paper_1906_11633_b200/variants
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --shared -Xcompiler -fPIC $flags \
       -Iinclude -Ipaper_1906_11633_b200/csrc -o paper_1906_11633_b200/variants/$name.so \
       paper_1906_11633_b200/csrc/dr_kernels.cu paper_1906_11633_b200/csrc/dr_api.cu paper_1906_11633_b200/csrc/dr_vision.cu || exit 1
done
