# Builds the three native libraries (all in-tree so gpurun ships them):
#   paper_2008_03909_b200/libcc.so   the product: CUDA kernels + C ABI (include/cc.h)
#   inputs/libccgen.so               seeded CUDA graph/stream generator (inputs, not the method)
#   oracle/liboracle.so              the CPU oracle (test infrastructure)
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PTXASV    ?=

CC_SRC    := $(wildcard paper_2008_03909_b200/csrc/*.cu)
CC_HDR    := $(wildcard paper_2008_03909_b200/csrc/*.cuh paper_2008_03909_b200/csrc/*.h include/*.h)
CC_OBJ    := $(patsubst paper_2008_03909_b200/csrc/%.cu,build/cc/%.o,$(CC_SRC))

all: paper_2008_03909_b200/libcc.so inputs/libccgen.so oracle/liboracle.so

build/cc/%.o: paper_2008_03909_b200/csrc/%.cu $(CC_HDR)
	@mkdir -p build/cc
	$(NVCC) $(NVFLAGS) $(PTXASV) -c $< -o $@

paper_2008_03909_b200/libcc.so: $(CC_OBJ)
	$(NVCC) $(ARCH) -shared $^ -o $@ -lcudart

inputs/libccgen.so: inputs/csrc/gen.cu
	$(NVCC) $(NVFLAGS) -shared $< -o $@ -lcudart

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c99 -Wall -shared -fPIC $< -o $@

clean:
	rm -rf build paper_2008_03909_b200/libcc.so inputs/libccgen.so oracle/liboracle.so

.PHONY: all clean

# measurement probes (not product code; binaries are git-ignored, built on demand)
probes: scripts/probe/randgather scripts/probe/zerocopy scripts/probe/incr_latency
scripts/probe/incr_latency: scripts/probe/incr_latency.cu paper_2008_03909_b200/libcc.so
	$(NVCC) $(ARCH) -O3 --cudart shared $< -o $@ -Lpaper_2008_03909_b200 -lcc -Xlinker -rpath=$(CURDIR)/paper_2008_03909_b200
scripts/probe/%: scripts/probe/%.cu
	$(NVCC) $(ARCH) -O3 --cudart shared $< -o $@

.PHONY: probes
