#!/bin/bash
# Build + run the GEMV microbenchmark against the library's objects (run under gpurun).
set -e
cd "$(dirname "$0")/.."
OBJ=paper_2605_06676_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o profiles/gemv_bench profiles/gemv_bench.cu \
    $OBJ/c_api.o $OBJ/budgets.o $OBJ/score.o $OBJ/select.o $OBJ/decode.o $OBJ/rope.o $OBJ/comm.o -ldl
