# Top-level build.  `make` builds the product library and the CPU checkers.
#   paper_2505_05950_b200/libfloe_b200.so : sm_100a kernels + C ABI (include/floe_gpu.h)
#   oracle/liboracle.so, oracle/_ref/libfloe_ref.so : test infrastructure
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG      := paper_2505_05950_b200
LIB      := $(PKG)/libfloe_b200.so
SRCS     := $(PKG)/csrc/floe_gpu.cu
HDRS     := $(wildcard $(PKG)/csrc/*.cuh) include/floe_gpu.h

all: $(LIB) oracle integration

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $(SRCS) -lcublasLt 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

oracle:
	$(MAKE) -C oracle

# INTEGRATION.md build: the reference core compiled in place + floe_b200.hpp (reference types)
integration: $(LIB)
	$(MAKE) -C tests/cpp

clean:
	rm -f $(LIB) build_ptxas.log
	$(MAKE) -C oracle clean
	$(MAKE) -C tests/cpp clean

.PHONY: all oracle integration clean

# Sanitizer build: same sources, a 600 s barrier watchdog (compute-sanitizer
# slows the kernels by orders of magnitude), separate output used through
# FLOE_LIB=tools/libfloe_b200_sanitize.so.
tools/libfloe_b200_sanitize.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -DFLOE_WATCHDOG_NS=600000000000ull -shared -cudart static -o $@ $(SRCS) -lcublasLt 2> /dev/null

# racecheck build: as above, with the early record polling compiled out
# (racecheck does not model shared-memory release/acquire; floe_v2.cuh).
tools/libfloe_b200_racecheck.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -DFLOE_WATCHDOG_NS=600000000000ull -DFLOE_RACECHECK -shared -cudart static -o $@ $(SRCS) -lcublasLt 2> /dev/null
