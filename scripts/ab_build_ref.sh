#!/bin/bash
# scripts/ab_build_ref.sh NAME GITREF [file ...]: the product library as of GITREF (with each given
# file, basename-matched, replacing csrc's copy) into scratch/libpcdn_NAME.so
set -e
NAME=$1; REF=$2; shift 2
D=$(mktemp -d); git archive $REF paper_1306_4080_b200/csrc include | tar -x -C $D
for f in "$@"; do cp "$f" $D/paper_1306_4080_b200/csrc/$(basename "$f"); done
mkdir -p scratch
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -shared $ABFLAGS \
    -o scratch/libpcdn_$NAME.so $D/paper_1306_4080_b200/csrc/pcdn_api.cu
rm -rf $D; echo scratch/libpcdn_$NAME.so
