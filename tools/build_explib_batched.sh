#!/bin/bash
# Developer experiment: rebuild lsb_batched.cu with extra -D defines and link it with the regular
# objects into _explibs/NAME.so (tools/swap_c5.sh times every library found there).
# Usage: tools/build_explib_batched.sh NAME "-DLSB_H3_MINB=3 ..."
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
SRC=paper_2409_03807_b200/csrc; OBJ=paper_2409_03807_b200/_lib/obj
mkdir -p _explibs/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
$NV $DEFS -c $SRC/lsb_batched.cu -o _explibs/obj/bat_$NAME.o
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _explibs/$NAME.so _explibs/obj/bat_$NAME.o \
    $OBJ/lsb_api.o $OBJ/lsb_context.o $OBJ/lsb_bench.o $OBJ/lsb_refops.o $OBJ/lsb_setup.o -lpthread
echo "built _explibs/$NAME.so"
