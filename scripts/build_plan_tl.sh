#!/bin/bash
# Timeline variant: flow_resident.cu and dynamics.cu (fused planner) with
# -DFCB_TIMELINE, linked against the regular objects (build_variants/pltl).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2511_11514_b200/csrc
OUT=$ROOT/build_variants/pltl
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -DFCB_TIMELINE"
nvcc $FL -c $CS/dynamics.cu -o $OUT/dynamics.o &
nvcc $FL -c $CS/flow_resident.cu -o $OUT/flow_resident.o &
wait
nvcc $ARCH -shared -Xcompiler -fPIC $CS/build/abi.o $CS/build/sinkhorn.o $CS/build/stein.o \
     $OUT/dynamics.o $OUT/flow_resident.o -o $OUT/libflowcover_b200.so -lcudart_static -lrt -ldl -lpthread
