# Build recipe for the B200 FlexQuant engine (sm_100a only).
#   make            -> CUDA C-ABI library (libfq_cuda.so)
#   make oracle     -> CPU oracle restatement + reference build (oracle/Makefile)
NVCC      ?= nvcc
CXX       := /usr/bin/g++
PKG       := paper_2506_12024_b200
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc --expt-relaxed-constexpr
CU_SRCS   := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,build/cuda/%.o,$(CU_SRCS))
CUDA_LIB  := $(PKG)/lib/libfq_cuda.so

all: $(CUDA_LIB)

build/cuda/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/fq_internal.cuh include/fq_cuda.h $(PKG)/csrc/gemv_program.cuh
	@mkdir -p build/cuda
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(CUDA_LIB): $(CU_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/lib/*.so

.PHONY: all oracle clean
