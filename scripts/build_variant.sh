#!/bin/bash
# Builds an experimental variant of the library with extra -D flags for one translation unit:
#   scripts/build_variant.sh NAME "-DABFT_KS256=1" [gemm.cu|eb.cu]  -> scripts/bin/lib_NAME.so
set -e
cd "$(dirname "$0")/.."
python paper_2103_00130_b200/build.py > /dev/null
name=$1; flags=$2; unit=${3:-gemm.cu}
mkdir -p scripts/bin/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-fvisibility=hidden -I include -I paper_2103_00130_b200/csrc $flags \
  -c paper_2103_00130_b200/csrc/$unit -o scripts/bin/var_$name/unit.o
objs=$(ls build/abftlp/*.o | grep -v "/$unit.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/bin/lib_$name.so scripts/bin/var_$name/unit.o $objs -lpthread
echo scripts/bin/lib_$name.so
