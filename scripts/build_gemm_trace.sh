#!/bin/bash
# Dev probe build: gemm.cu with -DDBS_GEMM_TRACE linked with the other library objects.
set -e
cd "$(dirname "$0")/.."
NV=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NV $ARCH -O3 -std=c++17 -DDBS_GEMM_TRACE -DDBS_GEMM_ATTRIB -Iinclude -c paper_2007_11831_b200/csrc/gemm.cu -o /tmp/gemm_trace_k.o
objs=$(ls paper_2007_11831_b200/_build/*.o | grep -v gemm.o)
$NV $ARCH -O3 -std=c++17 -Iinclude scripts/gemm_trace.cu /tmp/gemm_trace_k.o $objs -o scripts/_bin/gemm_trace -lpthread -ldl -lrt
