#!/bin/bash
# Build an A/B variant library: p2p.cu from git revision $1 (or a file path),
# linked with the current objects -> paper_1209_3516_b200/libfmm_b200_$2.so
set -e
cd "$(dirname "$0")/.."
SRC=$1; NAME=$2; shift 2
T=$(mktemp -d)
if [ -f "$SRC" ]; then cp "$SRC" $T/p2p.cu; else git show "$SRC":paper_1209_3516_b200/csrc/p2p.cu > $T/p2p.cu; fi
O=paper_1209_3516_b200/_objs
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I paper_1209_3516_b200/csrc "$@" -c $T/p2p.cu -o $T/p2p.o
OBJS=$(ls $O/*.o | grep -v "/p2p.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_1209_3516_b200/libfmm_b200_$NAME.so $OBJS $T/p2p.o
rm -rf $T
