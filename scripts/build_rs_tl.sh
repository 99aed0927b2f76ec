#!/bin/bash
# Timeline variant of the library: flow_resident.cu with -DFCB_TIMELINE linked
# against the regular objects (build_variants/rstl, git-ignored).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2511_11514_b200/csrc
OUT=$ROOT/build_variants/rstl
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
     --expt-relaxed-constexpr -DFCB_TIMELINE $EXTRA -c $CS/flow_resident.cu -o $OUT/flow_resident.o
nvcc $ARCH -shared -Xcompiler -fPIC $CS/build/abi.o $CS/build/sinkhorn.o $CS/build/stein.o \
     $CS/build/dynamics.o $OUT/flow_resident.o -o $OUT/libflowcover_b200.so -lcudart_static -lrt -ldl -lpthread
