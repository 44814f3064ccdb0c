# Product build: the C-ABI library with the sm_100a kernels, built in-tree so
# it travels to the GPU box with the repo snapshot.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2012_14792_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/slicecraft_b200.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr -Xptxas -v

all: $(PKG)/libslicecraft_b200.so oracle

$(PKG)/libslicecraft_b200.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared $(SRCS) -o $@ -lpthread 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle:
	$(MAKE) -C oracle

# Drop-in check binary (needs the reference headers; built where they exist,
# runs on the GPU box): the reference library and the B200 binding side by side.
REF_INC ?= /root/reference/proj/include
dropin: dropin/dropin_test
dropin/dropin_test: dropin/dropin_test.cpp dropin/slicecraft_b200.hpp $(PKG)/libslicecraft_b200.so oracle
	g++ -std=c++20 -O2 -I$(REF_INC) -Iinclude -Idropin $< \
	    -Loracle/_ref -lslicecraft_ref -L$(PKG) -lslicecraft_b200 \
	    -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

clean:
	rm -f $(PKG)/libslicecraft_b200.so build_ptxas.log
	$(MAKE) -C oracle clean

.PHONY: all oracle clean dropin
