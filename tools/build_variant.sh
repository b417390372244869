#!/bin/bash
# Builds an A/B variant of the engine library with extra nvcc flags (dev tool):
#   tools/build_variant.sh NAME "-DGDEV_FOO=3 ..."  ->  paper_2412_16490_b200/_lib/variants/libgrasp_b200_NAME.so
# Use it with GRASP_LIB=<that path> python bench.py ...
set -e
cd "$(dirname "$0")/../paper_2412_16490_b200/csrc"
NAME=$1; EXTRA=$2
OUT=../_lib/variants; OBJ=../_lib/obj
mkdir -p $OUT/$NAME
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20 -Xcompiler -fPIC -Iinclude -Xptxas -v --expt-relaxed-constexpr $EXTRA"
$NV --fmad=false -c cuda/engine.cu -o $OUT/$NAME/engine.o 2> $OUT/$NAME/ptxas_engine.log &
$NV -c cuda/qp.cu -o $OUT/$NAME/qp.o 2> $OUT/$NAME/ptxas_qp.log &
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -o $OUT/libgrasp_b200_$NAME.so \
  $(ls $OBJ/*.o | grep -v -e engine.o -e qp.o -e engine_debug.o) $OUT/$NAME/engine.o $OUT/$NAME/qp.o -lpthread
echo built $OUT/libgrasp_b200_$NAME.so
