#!/bin/bash
# Experiment build: libcc.so with kernels/dataflow.cu compiled with extra defines, into
# variants/<name>/libcc.so (load it with CC_LIB=...).  Usage: tools/variant.sh name -DX=1 ...
set -e
name=$1; shift
mkdir -p variants/$name
NVCC=/usr/local/cuda/bin/nvcc
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-Wall -Iinclude "$@" \
  -c paper_2511_02257_b200/csrc/kernels/dataflow.cu -o variants/$name/dataflow.o
objs=$(ls paper_2511_02257_b200/build/*.o | grep -v kernels_dataflow.cu.o)
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libcc.so $objs variants/$name/dataflow.o
echo built variants/$name/libcc.so
