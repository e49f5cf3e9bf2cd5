#!/bin/bash
# Build a kernel-variant copy of libsthk.so with extra -D flags (experiments only).
# usage: tools/build_variant.sh NAME "-DSTHK_SYM_G=2 ..."
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2005_10123_b200/csrc
OUT=${VOUT:-$ROOT/tools/variants}; mkdir -p $OUT/obj_$NAME
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $DEFS -c $C/sthk_kernels.cu -o $OUT/obj_$NAME/k.o -Xptxas -v 2> $OUT/obj_$NAME/ptxas.log
grep -A2 "sym_kernelILb1" $OUT/obj_$NAME/ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo
nvcc $ARCH -shared -o $OUT/libsthk_$NAME.so $OUT/obj_$NAME/k.o $C/sthk_diag.o $C/sthk_engine.o $C/sthk_sim.o -L/usr/local/cuda/lib64 -lcudart_static -lnccl -lrt -ldl -lpthread
