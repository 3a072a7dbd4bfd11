# Native build: libgls.so (CUDA, sm_100a) and the test-only oracle (plain C).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_2304_13398_b200
SRC := $(PKG)/csrc/gls_api.cu $(PKG)/csrc/gls_kernels.cu
HDR := $(PKG)/csrc/gls_internal.cuh $(PKG)/csrc/gls_lanes.cuh $(PKG)/csrc/gls_csrp.cuh include/gls.h

all: $(PKG)/libgls.so oracle/liboracle.so

$(PKG)/libgls.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) -lcudart

oracle/liboracle.so: oracle/gls_oracle.c
	gcc -O2 -std=c11 -shared -fPIC -o $@ $<

# bounds-checked build (device asserts on every hot-path access; tests: GLS_LIB=... pytest -m gpu)
check: $(PKG)/libgls_check.so

$(PKG)/libgls_check.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DGLS_CHECK -shared -o $@ $(SRC) -lcudart

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/gls_kernels.o $(PKG)/csrc/gls_kernels.cu

clean:
	rm -f $(PKG)/libgls.so oracle/liboracle.so

.PHONY: all clean ptxas check

# A/B variants for performance experiments (not used by tests)
variant-%: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -DGLS_MINB=$* -shared -o /tmp/libgls_minb$*.so $(SRC) -lcudart

# named A/B variant with extra flags: make var V=name F="-DGLS_ROUND=16"
var: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) $(F) -shared -o $(PKG)/libgls_$(V).so $(SRC) -lcudart
