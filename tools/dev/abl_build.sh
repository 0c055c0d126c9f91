#!/bin/bash
# Development tool: build ablation variants of the library into
# paper_2112_12965_b200/csrc/build/abl_<name>.so (git-ignored, travels with gpurun).
# usage: tools/abl_build.sh name "-DFLAG ..." [name "-DFLAGS"]...
set -e
cd "$(dirname "$0")/../../paper_2112_12965_b200/csrc"
ARCH="-gencode arch=compute_100a,code=sm_100a"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p build/abl_$name
  for f in stats ${JOIN:-join} heads_fft learn dprofile capi peak; do
    nvcc $ARCH -O3 -lineinfo -std=c++20 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $f.cu -o build/abl_$name/$f.o &
  done
  wait
  nvcc $ARCH -shared -cudart static -o build/abl_$name.so build/abl_$name/*.o
  echo "built build/abl_$name.so"
done
