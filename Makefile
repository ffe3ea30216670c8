# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
#   make            -> paper_2503_01066_b200/libcolo_b200.so + oracle libs
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2503_01066_b200
SRC := $(PKG)/csrc/colo_host.cu $(PKG)/csrc/colo_runtime.cu $(PKG)/csrc/colo_decide.cu $(PKG)/csrc/colo_replay.cu
HDR := include/colo_abi.h $(PKG)/csrc/colo_common.cuh $(PKG)/csrc/colo_internal.h
# -fmad=false: no FMA contraction anywhere (bit-exact f64 vs the x86 reference)
NVFLAGS := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Iinclude -Xcompiler -fPIC,-O2 -Xptxas -v

all: $(PKG)/libcolo_b200.so oracle

$(PKG)/libcolo_b200.so: $(SRC) $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(PKG)/libcolo_b200.so

.PHONY: all oracle clean
