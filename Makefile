# Build the product library (CUDA, sm_100a) and the CPU oracle (test infrastructure).
NVCC      ?= nvcc
ARCH      ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   ?= -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall -Iinclude \
             -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_2110_06196_b200
SRCS      := $(wildcard $(PKG)/csrc/*.cu)
HDRS      := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/grape_walk.h
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
LIB       := $(PKG)/libgrape_walk.so

LIBCHK    := $(PKG)/libgrape_walk_checked.so
OBJSCHK   := $(patsubst $(PKG)/csrc/%.cu,build_checked/%.o,$(SRCS))

all: $(LIB) $(LIBCHK) oracle/liboracle.so tools/libgrape_dram_probe.so

# measurement aid for bench.py (DRAM bytes of one launch from the GPU counters; CUPTI), not the product
tools/libgrape_dram_probe.so: tools/dram_probe.cpp
	g++ -O2 -std=c++17 -shared -fPIC $< -I/usr/local/cuda/include -L/usr/local/cuda/lib64 \
	    -Wl,-rpath,/usr/local/cuda/lib64 -lcupti -lnvperf_host -lcuda -o $@

# bounds-checked build (GRAPE_CHECKED: every table access, row write and derived index
# checked in the kernels; tests/test_gpu_checked.py) — same sources, same ABI
checked: $(LIBCHK)

build_checked/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build_checked
	$(NVCC) $(NVFLAGS) -DGRAPE_CHECKED=1 -c $< -o $@ 2> build_checked/$*.ptxas.log || (cat build_checked/$*.ptxas.log; false)

$(LIBCHK): $(OBJSCHK)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJSCHK) -cudart static

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

oracle/liboracle.so: oracle/grape_oracle.c
	gcc -O2 -std=gnu99 -fPIC -shared -ffp-contract=off -fno-fast-math -Wall -o $@ $< -lm

clean:
	rm -rf build build_checked $(LIB) $(LIBCHK) oracle/liboracle.so tools/libgrape_dram_probe.so

.PHONY: all clean checked
