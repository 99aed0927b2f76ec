#!/bin/bash
# Build variants of libflowcover_b200.so with different compile-time knobs into
# build_variants/NAME/ (git-ignored; travels to the GPU box with gpurun), then
# select one at run time with FCB_LIB_PATH=build_variants/NAME/libflowcover_b200.so.
# usage: scripts/tune_ot.sh "NAME:-DFCB_RPT32=4 -DFCB_MINB=1" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2511_11514_b200/csrc
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  make -C $CS -j8 BUILD=$ROOT/build_variants/$name/obj \
       OUT=$ROOT/build_variants/$name/libflowcover_b200.so EXTRA="$defs"
done
