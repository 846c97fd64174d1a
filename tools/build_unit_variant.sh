#!/bin/bash
# Build an A/B variant library with one translation unit recompiled:
#   tools/build_unit_variant.sh UNIT NAME [nvcc flags...]
# compiles paper_1209_3516_b200/csrc/UNIT.cu with the extra flags and links
# it with the other current objects -> paper_1209_3516_b200/libfmm_b200_NAME.so
set -e
cd "$(dirname "$0")/.."
UNIT=$1; NAME=$2; shift 2
T=$(mktemp -d)
O=paper_1209_3516_b200/_objs
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I paper_1209_3516_b200/csrc "$@" -c paper_1209_3516_b200/csrc/$UNIT.cu -o $T/$UNIT.o
OBJS=$(ls $O/*.o | grep -v "/$UNIT.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_1209_3516_b200/libfmm_b200_$NAME.so $OBJS $T/$UNIT.o
rm -rf $T
