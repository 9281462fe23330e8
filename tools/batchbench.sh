#!/bin/bash
set -e
cd "$(dirname "$0")/.."
g++ -O3 -std=c++17 -march=x86-64-v3 -Iinclude -Ipaper_2312_07743_b200/csrc -I/usr/local/cuda/include -o build/batchbench tools/batchbench.cpp \
  build/fw2v_kernels.o build/fw2v_snapshot.o build/k1s_*.o build/fw2v_corpus.o build/fw2v_io.o build/fw2v_eval.o -L/usr/local/cuda/lib64 -lcudart_static -lpthread -ldl -lrt
