# Builds the three native libraries in-tree (they travel to the GPU box with the snapshot):
#   datagen/libflern_gen.so                      seeded input generator (shared by both sides)
#   oracle/liboracle.so                          CPU oracle (test infrastructure)
#   paper_2311_02781_b200/lib/libflern.so        the product: C-ABI + sm_100a kernels
NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -cudart static --expt-relaxed-constexpr -Iinclude -Xptxas -v
PKG := paper_2311_02781_b200
CSRC := $(PKG)/csrc
KERNEL_SRCS := $(wildcard $(CSRC)/*.cu)
KERNEL_HDRS := $(wildcard $(CSRC)/*.cuh) include/flern.h

all: datagen/libflern_gen.so oracle/liboracle.so $(PKG)/lib/libflern.so

datagen/libflern_gen.so: datagen/flern_gen.cpp
	$(CXX) -O2 -std=c++17 -fPIC -shared -pthread -o $@ $<

# -ffp-contract=off: every fp64 op separately rounded, in source order
oracle/liboracle.so: oracle/oracle.cpp oracle/oracle.h
	$(CXX) -O2 -std=c++17 -ffp-contract=off -fPIC -shared -pthread -o $@ oracle/oracle.cpp

$(PKG)/lib/libflern.so: $(KERNEL_SRCS) $(KERNEL_HDRS)
	@mkdir -p $(PKG)/lib build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(KERNEL_SRCS) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)
	@grep -E "error|spill|Used" build/ptxas.log | grep -v " 0 bytes spill" | head -40 || true

# diagnostic variant: reads the FLERN_DBG_* / FLERN_NO_* / FLERN_WAIT_HINT A/B knobs from the environment
# (scripts/ab_env.sh runs with FLERN_LIB=libflern_diag.so); the release library never reads the environment
$(PKG)/lib/libflern_diag.so: $(KERNEL_SRCS) $(KERNEL_HDRS)
	@mkdir -p $(PKG)/lib build
	$(NVCC) $(NVFLAGS) -DFLERN_DIAG -shared -o $@ $(KERNEL_SRCS) 2> build/ptxas_diag.log || (cat build/ptxas_diag.log; exit 1)

# diagnostic variant: per-role mbarrier wait accounting (scripts/trace.py)
$(PKG)/lib/libflern_tw.so: $(KERNEL_SRCS) $(KERNEL_HDRS)
	@mkdir -p $(PKG)/lib build
	$(NVCC) $(NVFLAGS) -DFLERN_TRACE_WAITS -shared -o $@ $(KERNEL_SRCS) 2> build/ptxas_tw.log || (cat build/ptxas_tw.log; exit 1)

$(PKG)/lib/libflern_seq.so: $(KERNEL_SRCS) $(KERNEL_HDRS)
	@mkdir -p $(PKG)/lib build
	$(NVCC) $(NVFLAGS) -DFLERN_SEQ_TRACE -shared -o $@ $(KERNEL_SRCS) 2> build/ptxas_seq.log || (cat build/ptxas_seq.log; exit 1)

clean:
	rm -f datagen/libflern_gen.so oracle/liboracle.so $(PKG)/lib/libflern.so

.PHONY: all clean
