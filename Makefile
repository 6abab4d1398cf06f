# Build the product library (CUDA, sm_100a), the host-only inputs library and
# the CPU oracle.
#   make            -> paper_1501_06625_b200/libpathtrack_b200.so   (the tracker: C-ABI + kernels)
#                      paper_1501_06625_b200/libpt_inputs.so        (host: generators, system/solution
#                                                                    files, Pieri minors; no CUDA)
#                      oracle/liborc.so                             (test infrastructure)
#   make ref        -> oracle/_ref/liborc_ref.so (needs /root/reference)
NVCC     ?= /usr/local/cuda/bin/nvcc
HOSTCXX  := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH     := -gencode arch=compute_100a,code=sm_100a
# --fmad=false + explicit _rn intrinsics: no FMA contraction anywhere (bit parity).
# No --split-compile: its parallel optimisation is not deterministic (two
# builds of the same sources gave different register / stack allocations and
# single-path times 7-18 % apart); the TUs still compile in parallel (make -j).
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -ccbin $(HOSTCXX) \
            -Xcompiler -fPIC,-ffp-contract=off -Xptxas -warn-spills $(EXTRA_NVFLAGS)
HOSTFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wno-unknown-pragmas
PKG      := paper_1501_06625_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/libpathtrack_b200.so
INLIB    := $(PKG)/libpt_inputs.so
HDRS     := $(SRC)/mp.cuh $(SRC)/mp_qdfast.cuh $(SRC)/mgs_batch.cuh $(SRC)/device.cuh $(SRC)/mgs_warp.cuh $(SRC)/plan.hpp $(SRC)/work.hpp \
            $(SRC)/kernels.cuh $(SRC)/kernel_set.hpp include/pathtrack_b200.h
# one translation unit per precision: the three ptxas runs proceed in parallel
KOBJS    := $(SRC)/kern_d.o $(SRC)/kern_dd.o $(SRC)/kern_dd_exact.o $(SRC)/kern_qd.o $(SRC)/kern_qd_fast.o $(SRC)/kern_misc.o \
            $(SRC)/tracker.o
INOBJS   := $(SRC)/gen.o $(SRC)/sysio.o $(SRC)/pieri.o

all: $(LIB) $(INLIB) oracle

$(SRC)/%.o: $(SRC)/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) $(KFLAGS) -c $< -o $@

# the fast DD tracking kernels: dd_norm without the non-finite select (paths
# that meet inf / NaN are re-tracked by kern_dd_exact.o, pathtrack_b200.h)
$(SRC)/kern_dd.o: KFLAGS := -DPT_DD_FAST_NONFINITE
# the tolerance-parity QD kernels (mp_qdfast.cuh, pt_plan_set_arith); the QD ops stay
# out-of-line calls (inlined, the column chain ran 30 % slower: instruction cache)
$(SRC)/kern_qd_fast.o: KFLAGS := -DPT_QD_FAST

$(SRC)/%.o: $(SRC)/%.cpp $(SRC)/mp.cuh $(SRC)/inputs.hpp include/pathtrack_inputs.h
	$(HOSTCXX) $(HOSTFLAGS) -c $< -o $@

$(LIB): $(KOBJS)
	$(NVCC) $(ARCH) -shared -ccbin $(HOSTCXX) -o $@ $^

$(INLIB): $(INOBJS)
	$(HOSTCXX) -shared -o $@ $^

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(SRC)/*.o $(LIB) $(INLIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean
