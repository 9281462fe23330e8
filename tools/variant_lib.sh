#!/bin/bash
# Experiment build: libfw2v with one K1s shape TU recompiled with extra nvcc flags.
# usage: tools/variant_lib.sh NAME SHAPE "FLAGS"   e.g. tools/variant_lib.sh rb6 l16v8 "-DFW2V_STAIR_REG_BLOCKS=6"
# -> paper_2312_07743_b200/_lib/libfw2v_NAME.so (select with FW2V_LIB=...)
set -e
cd "$(dirname "$0")/.."
NAME=$1; SHAPE=$2; FLAGS=$3
mkdir -p build_var
/usr/local/cuda/bin/nvcc $FLAGS -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
  -Iinclude -Ipaper_2312_07743_b200/csrc -c -o build_var/k1s_${SHAPE}_$NAME.o paper_2312_07743_b200/csrc/k1s_$SHAPE.cu 2> build_var/ptxas_$NAME.log
OBJS=$(ls build/*.o | grep -v "build/k1s_$SHAPE.o" | grep -v href_)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2312_07743_b200/_lib/libfw2v_$NAME.so \
  $OBJS build_var/k1s_${SHAPE}_$NAME.o -lpthread -ldl -lrt
grep -A2 "k1s_stair" build_var/ptxas_$NAME.log | grep -i "spill\|regis" | head -6
