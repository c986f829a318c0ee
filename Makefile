# Builds the B200 product library (libbfly.so, in-tree so it travels with gpurun)
# and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-O2,-Wall -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2507_17766_b200
SRCS := $(PKG)/csrc/bfly_plan.cu $(PKG)/csrc/bfly_merge.cu $(PKG)/csrc/bfly_peer.cu $(PKG)/csrc/bfly_host.cu \
        $(PKG)/csrc/bfly_validate.cu $(PKG)/csrc/bfly_ring.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/bfly.h
LIB := $(PKG)/libbfly.so

all: $(LIB) oracle

HOSTSRC := $(PKG)/csrc/bfly_convert.cpp
HOSTOBJ := build/bfly_convert.o

$(HOSTOBJ): $(HOSTSRC)
	g++ -O3 -fPIC -Wall -c -o $@ $<

$(LIB): $(SRCS) $(HDRS) $(HOSTOBJ)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) $(HOSTOBJ) 2> build/ptxas.log || (cat build/ptxas.log; false)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(LIB)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean

# tuning build (not the product): adds bfly_tune_reduce for tools/tune_reduce.py
tune: build/libbfly_tune.so
build/libbfly_tune.so: $(SRCS) $(HDRS) $(HOSTOBJ)
	$(NVCC) $(NVFLAGS) -DBFLY_TUNING -shared -o $@ $(SRCS) $(HOSTOBJ) 2> build/ptxas_tune.log || (cat build/ptxas_tune.log; false)
.PHONY: tune
