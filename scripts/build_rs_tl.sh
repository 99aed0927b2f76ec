#!/bin/bash
# Timeline variant of the library (-DFCB_TIMELINE: globaltimer stamps at the
# grid barriers of the resident flow and the fused planner, read back with
# fcb_debug_timeline / fcb_debug_rs_timeline) in build_variants/rstl.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -C $ROOT/paper_2511_11514_b200/csrc -j8 BUILD=$ROOT/build_variants/rstl/obj \
     OUT=$ROOT/build_variants/rstl/libflowcover_b200.so EXTRA="-DFCB_TIMELINE $EXTRA"
