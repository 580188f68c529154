#!/bin/bash
# A/B variant of the CUDA library: recompiles program.cu with extra nvcc flags and links
# paper_2506_12024_b200/lib/ab/libfq_cuda_<name>.so (select at run time with FQ_CUDA_LIB=<path>).
#   tools/ab_build.sh B -DFQ_SOMETHING=1
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/ab paper_2506_12024_b200/lib/ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
  -Ipaper_2506_12024_b200/csrc --expt-relaxed-constexpr "$@" -c paper_2506_12024_b200/csrc/program.cu -o build/ab/program_$name.o
objs=$(ls build/cuda/*.o | grep -v program.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2506_12024_b200/lib/ab/libfq_cuda_$name.so $objs build/ab/program_$name.o -lcudart
echo paper_2506_12024_b200/lib/ab/libfq_cuda_$name.so
