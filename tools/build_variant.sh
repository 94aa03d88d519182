#!/bin/bash
# A/B builds of the product library with extra nvcc flags (profiling only):
#   tools/build_variant.sh NAME "-DFOO -DBAR"  ->  paper_2002_02145_b200/libpsconv_NAME.so
set -e
cd "$(dirname "$0")/.."
make -s build/desc.o build/recipe.o build/select.o build/emit.o build/microkernel_cpu.o build/nest.o build/dnnrank.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
  --expt-relaxed-constexpr -Iinclude -Ipaper_2002_02145_b200/csrc $2 -c paper_2002_02145_b200/csrc/conv_fwd.cu -o build/var_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2002_02145_b200/libpsconv_$1.so \
  build/var_$1.o build/desc.o build/recipe.o build/select.o build/emit.o build/microkernel_cpu.o build/nest.o build/dnnrank.o -Xcompiler -fopenmp -lgomp
