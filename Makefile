# Build every native artefact in-tree (the .so files travel to the GPU box).
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
CXXFLAGS  := -O2 -std=c++17 -fPIC

DFR_SO    := paper_2207_14334_b200/libdfr.so
ORACLE_SO := oracle/liboracle.so
DATAGEN_SO:= datagen/libdatagen.so
DFR_SRC   := $(wildcard paper_2207_14334_b200/csrc/*.cu)
DFR_HDR   := $(wildcard paper_2207_14334_b200/csrc/*.cuh) include/dfr.h

all: $(DATAGEN_SO) $(ORACLE_SO) $(DFR_SO)
host: $(DATAGEN_SO) $(ORACLE_SO)

$(DATAGEN_SO): datagen/datagen.cpp
	$(CXX) $(CXXFLAGS) -O3 -fopenmp -shared $< -o $@

# the oracle is deliberately plain: -O2, single-threaded, no OpenMP
$(ORACLE_SO): oracle/oracle.cpp
	$(CXX) $(CXXFLAGS) -shared $< -o $@

$(DFR_SO): $(DFR_SRC) $(DFR_HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -shared $(DFR_SRC) -o $@ 2> paper_2207_14334_b200/ptxas.log || (cat paper_2207_14334_b200/ptxas.log; false)

clean:
	rm -f $(DFR_SO) $(ORACLE_SO) $(DATAGEN_SO)

.PHONY: all host clean

# debug variant: sync + error check after every launch, device bounds asserts
paper_2207_14334_b200/libdfr_debug.so: $(DFR_SRC) $(DFR_HDR)
	$(NVCC) $(NVFLAGS) -DDFR_DEBUG -shared $(DFR_SRC) -o $@
