#!/bin/bash
# Build K1s microbenchmark variants: tools/kbench.sh NAME "-DFLAGS..." ; binaries in build/kbench_NAME
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas -v \
  -Iinclude -Ipaper_2312_07743_b200/csrc -DKB_NAME="\"$NAME\"" "$@" -o build/kbench_$NAME tools/kbench.cu \
  -Lpaper_2312_07743_b200/_lib -lfw2v -Xlinker -rpath,'$ORIGIN/../paper_2312_07743_b200/_lib' 2>&1 | grep -E "error|registers|spill" | head -5
