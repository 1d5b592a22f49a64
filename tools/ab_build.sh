#!/bin/bash
# A/B experiment build: tools/ab_build.sh NAME "-DFLAG ..." [sources...]
# Recompiles the listed kernel sources (default: k_stats_i8 k_score_i8) with extra defines on top of
# the regular build objects and links ab/NAME.so (git-ignored, travels to the GPU box).
set -e
NAME=$1; DEFS=$2; shift 2
SRCS=${@:-k_stats_i8 k_score_i8}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2408_14947_b200/csrc
OUT=$ROOT/ab/$NAME; mkdir -p $OUT
cp $C/build/*.o $OUT/
rm -f $OUT/k_probe.o $OUT/k_stream_probe.o $OUT/k_tc_selftest.o $OUT/probe_api.o
for s in $SRCS; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 $DEFS -c $C/$s.cu -o $OUT/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/ab/$NAME.so $OUT/*.o -lpthread
rm -rf $OUT
echo built ab/$NAME.so
