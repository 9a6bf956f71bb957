#!/bin/bash
# Build tuning variants of libhrb200.so into paper_1211_3056_b200/_lib/variants/
# (git-ignored, travels with gpurun); bench them with HRB_LIB=<path>.
cd "$(dirname "$0")/.."
mkdir -p paper_1211_3056_b200/_lib/variants
build() {  # name, extra nvcc flags
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $2 \
    -o paper_1211_3056_b200/_lib/variants/$1.so paper_1211_3056_b200/csrc/hrb200.cu &
}
for spec in "$@"; do build "${spec%%:*}" "${spec#*:}"; done
wait
ls paper_1211_3056_b200/_lib/variants/
