# Builds the in-tree CUDA library (sm_100a) and the oracle's C pieces.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
PKG := paper_2405_05079_b200
LIB := $(PKG)/libpovar.so
SRC := $(PKG)/csrc/povar.cu
HDR := $(PKG)/csrc/pv_kernels.cuh $(PKG)/csrc/pv_device.cuh $(PKG)/csrc/pv_pcg.cuh $(PKG)/csrc/pv_pipe.cuh include/povar.h
BALSRC := $(PKG)/csrc/pv_bal.cpp
BALOBJ := build/pv_bal.o

all: $(LIB)

$(BALOBJ): $(BALSRC) include/povar_bal.h
	mkdir -p build
	g++ -O3 -std=c++17 -fPIC -pthread -Wall -c -o $@ $(BALSRC)

$(LIB): $(SRC) $(HDR) $(BALOBJ)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) $(BALOBJ) -lnccl -Xcompiler -pthread

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/povar_ptxas.o $(SRC) 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" 

clean:
	rm -f $(LIB) $(BALOBJ)

.PHONY: all clean ptxas
