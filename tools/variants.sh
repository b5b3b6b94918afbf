#!/bin/bash
# Build sortbench variants with different onesweep compile flags.
set -e
cd "$(dirname "$0")"
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
SRC=../paper_2503_05168_b200/csrc
OBJ=$SRC/_obj
for v in "${@:-base: trace:-DSEELE_SORT_TRACE}"; do
  name=${v%%:*}; flags=${v#*:}
  $NVCC -std=c++17 -O3 -lineinfo $ARCH $flags -c $SRC/binning.cu -o /tmp/binning_$name.o
  $NVCC -std=c++17 -O3 $ARCH $flags -c $SRC/api.cu -o /tmp/api_$name.o
  $NVCC -std=c++17 -O3 $ARCH $flags -o sortbench_$name sortbench.cu /tmp/api_$name.o /tmp/binning_$name.o $OBJ/preprocess.o $OBJ/raster.o $OBJ/raster_fast.o -lcudart
done
