#!/bin/bash
# Builds an experimental variant of the library with extra -D flags for gemm.cu:
#   scripts/build_variant.sh NAME "-DABFT_KS256=1 -DABFT_STAGING_BUFS=1"  -> scripts/bin/lib_NAME.so
set -e
cd "$(dirname "$0")/.."
python paper_2103_00130_b200/build.py > /dev/null
name=$1; shift
mkdir -p scripts/bin/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-fvisibility=hidden -I include -I paper_2103_00130_b200/csrc $@ \
  -c paper_2103_00130_b200/csrc/gemm.cu -o scripts/bin/var_$name/gemm.o
objs=$(ls build/abftlp/*.o | grep -v gemm.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/bin/lib_$name.so scripts/bin/var_$name/gemm.o $objs -lpthread
echo scripts/bin/lib_$name.so
