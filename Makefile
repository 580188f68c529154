# Build recipe for the B200 FlexQuant engine (sm_100a only).
#   make            -> CUDA C-ABI library (libfq_cuda.so), C++ host library (libflexquant_b200.so)
#                      and its Python module (_flexquant*.so)
#   make oracle     -> CPU oracle restatement + reference build (oracle/Makefile)
NVCC      ?= nvcc
CXX       := /usr/bin/g++
PYTHON    ?= python
PKG       := paper_2506_12024_b200
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc --expt-relaxed-constexpr
CU_SRCS   := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,build/cuda/%.o,$(CU_SRCS))
CUDA_LIB  := $(PKG)/lib/libfq_cuda.so
CUDA_HOME ?= /usr/local/cuda
HOST_SRCS := $(filter-out $(PKG)/host/bindings.cpp,$(wildcard $(PKG)/host/*.cpp))
HOST_OBJS := $(patsubst $(PKG)/host/%.cpp,build/host/%.o,$(HOST_SRCS))
HOST_LIB  := $(PKG)/lib/libflexquant_b200.so
CXXFLAGS  := -O2 -std=c++20 -fPIC -Wall -Iinclude -I$(PKG)/host -I$(CUDA_HOME)/include
PYEXT     := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))" 2>/dev/null)
PYINC     := $(shell $(PYTHON) -c "import sysconfig, pybind11; print('-I'+sysconfig.get_paths()['include'], '-I'+pybind11.get_include())" 2>/dev/null)
PYMOD     := $(PKG)/_flexquant$(PYEXT)
RPATH     := -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/lib'

all: $(CUDA_LIB) $(HOST_LIB) $(PYMOD)

build/cuda/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/fq_internal.cuh include/fq_cuda.h $(PKG)/csrc/gemv_program.cuh
	@mkdir -p build/cuda
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(CUDA_LIB): $(CU_OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

build/host/%.o: $(PKG)/host/%.cpp $(wildcard include/flexquant/*.hpp) include/fq_cuda.h $(wildcard $(PKG)/host/*.hpp)
	@mkdir -p build/host
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(HOST_LIB): $(HOST_OBJS) $(CUDA_LIB)
	$(CXX) -shared -o $@ $(HOST_OBJS) -L$(PKG)/lib -lfq_cuda -L$(CUDA_HOME)/lib64 -lcudart $(RPATH)

$(PYMOD): $(PKG)/host/bindings.cpp $(HOST_LIB) $(wildcard include/flexquant/*.hpp)
	$(CXX) $(CXXFLAGS) -shared $(PYINC) -o $@ $< -L$(PKG)/lib -lflexquant_b200 -lfq_cuda -L$(CUDA_HOME)/lib64 -lcudart $(RPATH)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/lib/*.so $(PKG)/_flexquant*.so

.PHONY: all oracle clean
