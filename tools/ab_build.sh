#!/bin/bash
# A/B variant of the CUDA library: recompiles one source (default program.cu; AB_SRC=gemm_tc to
# pick another) with extra nvcc flags and links paper_2506_12024_b200/lib/ab/libfq_cuda_<name>.so
# (select at run time with FQ_CUDA_LIB=<path>).
#   tools/ab_build.sh B -DFQ_SOMETHING=1
#   AB_SRC=gemm_tc tools/ab_build.sh a3 -DFQ_A32=3 -DFQ_IN32=5
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=${AB_SRC:-program}
mkdir -p build/ab paper_2506_12024_b200/lib/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2506_12024_b200/csrc --expt-relaxed-constexpr "$@" -c paper_2506_12024_b200/csrc/$src.cu -o build/ab/${src}_$name.o
objs=$(ls build/cuda/*.o | grep -v "/$src.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2506_12024_b200/lib/ab/libfq_cuda_$name.so $objs build/ab/${src}_$name.o -lcudart
echo paper_2506_12024_b200/lib/ab/libfq_cuda_$name.so
