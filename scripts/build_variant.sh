#!/bin/bash
# Build a variant of libegfem.so with extra nvcc flags on one translation unit (A/B experiments).
# usage: scripts/build_variant.sh NAME TU.cu "-DFLAG=1 ..."  -> paper_2005_06193_b200/lib/variants/NAME.so
set -e
cd "$(dirname "$0")/.."
L=paper_2005_06193_b200/lib; mkdir -p $L/variants $L/variants/obj
TU=$2; base=$(basename $TU .cu)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC $3 -I include \
  -c -o $L/variants/obj/$1_$base.o paper_2005_06193_b200/csrc/$TU
objs=""; for o in $L/obj/*.o; do [ "$(basename $o)" = "$base.o" ] && objs="$objs $L/variants/obj/$1_$base.o" || objs="$objs $o"; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -o $L/variants/$1.so $objs -lnvrtc -ldl
echo built $L/variants/$1.so
