# B200 (sm_100a) build of the DiffKV memory-manager C-ABI library + the CPU oracle (test infrastructure).
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $(EXTRA) \
           --expt-relaxed-constexpr -Iinclude -Xptxas -v
PKG     := paper_2412_03131_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) include/dkv.h
LIB     := $(PKG)/libdkv.so
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

all: $(LIB) oracle/liboracle.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@.tmp $(OBJS) && mv $@.tmp $@

oracle/liboracle.so: oracle/dkv_oracle.c oracle/dkv_oracle.h
	gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -Wall -o $@ oracle/dkv_oracle.c -lm

clean:
	rm -rf build $(LIB) oracle/liboracle.so

.PHONY: all clean
