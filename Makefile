# Builds the B200 engine (product) and the CPU oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-Wall -Xptxas -v \
           --expt-relaxed-constexpr -Iinclude
PKG := paper_2504_15302_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/rd.h include/rd_format.h
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))
LIB := $(PKG)/lib/librd_b200.so

all: $(LIB) oracle

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# test-only probe of the tcgen05 building blocks (tests/test_gpu_tcgen05.py)
tests/cuda/libtcprobe.so: tests/cuda/tc_probe.cu $(PKG)/csrc/rd_device.cuh
	$(NVCC) $(ARCH) -O2 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -o $@ $<
all: tests/cuda/libtcprobe.so

# C++ adapter test (include/rd_ragsim.hpp) against each implementation of rd.h
tests/cpp/ragsim_adapter_cpu: tests/cpp/ragsim_adapter_test.cpp include/rd_ragsim.hpp include/rd.h oracle
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude -o $@ $< -Loracle -l:librd_cpu.so -Wl,-rpath,'$$ORIGIN/../../oracle'
tests/cpp/ragsim_adapter_b200: tests/cpp/ragsim_adapter_test.cpp include/rd_ragsim.hpp include/rd.h $(LIB)
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude -o $@ $< -L$(PKG)/lib -l:librd_b200.so -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib'
all: tests/cpp/ragsim_adapter_cpu tests/cpp/ragsim_adapter_b200
tests/cpp/fit_pin: tests/cpp/fit_pin.cpp include/rd_ragsim.hpp include/rd.h oracle
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude -o $@ $< -Loracle -l:librd_cpu.so -Wl,-rpath,'$$ORIGIN/../../oracle'
all: tests/cpp/fit_pin

# C++ end-to-end latency of rd_search through the C ABI (tools/e2e_latency.cpp)
tools/e2e_latency: tools/e2e_latency.cpp include/rd.h $(LIB)
	g++ -std=c++17 -O2 -Wall -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG)/lib -l:librd_b200.so \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../$(PKG)/lib' -Wl,-rpath,/usr/local/cuda/lib64
