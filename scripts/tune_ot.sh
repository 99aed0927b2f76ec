#!/bin/bash
# Build variants of libflowcover_b200.so with different sweep knobs into
# build_variants/ (git-ignored; travels to the GPU box with gpurun).
# usage: scripts/tune_ot.sh "NAME:-DFCB_SMEM_TILE=1 -DFCB_MINB=2" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build_variants
mkdir -p $OUT
CS=$ROOT/paper_2511_11514_b200/csrc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="$ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  mkdir -p $OUT/$name
  for f in abi stein dynamics; do
    [ -f $OUT/common_$f.o ] || nvcc $FL -c $CS/$f.cu -o $OUT/common_$f.o
  done
  nvcc $FL $defs -c $CS/sinkhorn.cu -o $OUT/$name/sinkhorn.o -Xptxas -v 2> $OUT/$name/ptxas.log
  nvcc $ARCH -shared -Xcompiler -fPIC $OUT/common_abi.o $OUT/common_stein.o $OUT/common_dynamics.o \
       $OUT/$name/sinkhorn.o -o $OUT/$name/libflowcover_b200.so -lcudart_static -lrt -ldl -lpthread
  echo "$name: $(grep -A3 'ot_solve_kernelIfLi2ELi2ELb0' $OUT/$name/ptxas.log | grep -o 'Used [0-9]* registers')"
done
