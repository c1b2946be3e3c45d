#!/bin/bash
# A/B variant of libpcdn.so: scripts/ab_build.sh NAME [file-to-substitute ...] builds the product
# library with each given header/source (basename-matched) replacing csrc's copy, into
# scratch/libpcdn_NAME.so (load it with PCDN_LIB=scratch/libpcdn_NAME.so).  Extra nvcc flags: $ABFLAGS.
set -e
NAME=$1; shift
D=$(mktemp -d); mkdir -p $D/p; cp -r paper_1306_4080_b200/csrc $D/p/; cp -r include $D/; for f in "$@"; do cp "$f" $D/p/csrc/$(basename "$f"); done
mkdir -p scratch
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false -Xcompiler -fPIC -shared $ABFLAGS \
    -o scratch/libpcdn_$NAME.so $D/p/csrc/pcdn_api.cu
rm -rf $D; echo scratch/libpcdn_$NAME.so
