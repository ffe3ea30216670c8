# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
#   make            -> paper_2503_01066_b200/libcolo_b200.so + oracle libs
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2503_01066_b200
SRC := $(PKG)/csrc/colo_host.cu $(PKG)/csrc/colo_runtime.cu $(PKG)/csrc/colo_decide.cu $(PKG)/csrc/colo_serving.cu $(PKG)/csrc/colo_sweep.cu $(PKG)/csrc/colo_io.cu $(PKG)/csrc/colo_colocated.cu $(PKG)/csrc/colo_report.cpp $(PKG)/csrc/colo_nccl.cu $(PKG)/csrc/colo_trace.cu
HDR := include/colo_abi.h $(PKG)/csrc/colo_common.cuh $(PKG)/csrc/colo_internal.h $(PKG)/csrc/colo_replay.cuh
# -fmad=false: no FMA contraction anywhere (bit-exact f64 vs the x86 reference)
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
NVFLAGS := $(ARCH) -O3 -lineinfo -fmad=false -std=c++17 -Iinclude -I$(JSON_DIR) -Xcompiler -fPIC,-O2 -Xptxas -v

all: $(PKG)/libcolo_b200.so oracle dropin cli

$(PKG)/libcolo_b200.so: $(SRC) $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -ldl 2> build/ptxas.log || (cat build/ptxas.log; false)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -f $(PKG)/libcolo_b200.so

.PHONY: all oracle clean

# C++ drop-in parity program: the unchanged reference headers + colosim_gpu.hpp
# (build-time dependency on /root/reference; the binary travels to the GPU box)
REF ?= /root/reference/proj
dropin: build/dropin_parity

build/dropin_parity: tests/cpp/dropin_parity.cpp $(PKG)/cpp/colosim_gpu.hpp include/colo_abi.h $(PKG)/libcolo_b200.so
	@if [ -d "$(REF)/include/colosim" ]; then mkdir -p build && \
	  g++ -std=c++20 -O2 -ffp-contract=off -I$(REF)/include -I$(JSON_DIR) -Iinclude -I$(PKG)/cpp -I/usr/local/cuda/include \
	    -o $@ tests/cpp/dropin_parity.cpp -L$(PKG) -lcolo_b200 -lnccl -Wl,-rpath,'$$ORIGIN/../$(PKG)'; \
	else echo "dropin: $(REF) absent, keeping prebuilt build/dropin_parity"; fi

.PHONY: dropin

# The reference's own CLI driver, tools/colosim.cpp UNCHANGED, compiled
# against the include overlay (paper_2503_01066_b200/cpp/overlay: Simulation,
# run_simulation and the map builders on the GPU) and linked to
# libcolo_b200.so.  Build-time dependency on /root/reference (the source is
# compiled where it lies, never copied); the binary travels to the GPU box.
cli: $(PKG)/bin/colosim

$(PKG)/bin/colosim: $(PKG)/cpp/overlay/colosim/engine.hpp $(PKG)/cpp/overlay/colosim/maps.hpp $(PKG)/cpp/overlay/colosim_gpu_context.hpp $(PKG)/cpp/colosim_gpu.hpp include/colo_abi.h $(PKG)/libcolo_b200.so
	@if [ -f "$(REF)/tools/colosim.cpp" ]; then mkdir -p $(PKG)/bin && \
	  g++ -std=c++20 -O2 -ffp-contract=off -I$(PKG)/cpp/overlay -I$(REF)/include -I$(JSON_DIR) -Iinclude -I$(PKG)/cpp \
	    -I$(PKG)/cpp/cli11 -o $@ $(REF)/tools/colosim.cpp -L$(PKG) -lcolo_b200 -Wl,-rpath,'$$ORIGIN/..'; \
	else echo "cli: $(REF) absent, keeping prebuilt $(PKG)/bin/colosim"; fi

.PHONY: cli
