# Build the product library (CUDA, sm_100a) and the CPU oracle.
#   make            -> paper_1501_06625_b200/libpathtrack_b200.so + oracle/liborc.so
#   make ref        -> oracle/_ref/liborc_ref.so (needs /root/reference)
NVCC     ?= /usr/local/cuda/bin/nvcc
HOSTCXX  := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH     := -gencode arch=compute_100a,code=sm_100a
# --fmad=false + explicit _rn intrinsics: no FMA contraction anywhere (bit parity)
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -ccbin $(HOSTCXX) \
            -Xcompiler -fPIC,-ffp-contract=off -Xptxas -warn-spills --split-compile=0 $(EXTRA_NVFLAGS)
PKG      := paper_1501_06625_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/libpathtrack_b200.so
HDRS     := $(SRC)/mp.cuh $(SRC)/device.cuh $(SRC)/mgs_warp.cuh $(SRC)/plan.hpp $(SRC)/work.hpp include/pathtrack_b200.h

all: $(LIB) oracle

$(SRC)/tracker.o: $(SRC)/tracker.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(SRC)/gen.o: $(SRC)/gen.cpp $(SRC)/mp.cuh include/pathtrack_b200.h
	$(HOSTCXX) -std=c++20 -O2 -fPIC -ffp-contract=off -c $< -o $@

$(LIB): $(SRC)/tracker.o $(SRC)/gen.o
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -o $@ $^

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(SRC)/*.o $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean
