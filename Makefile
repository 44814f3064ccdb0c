# Product build: the C-ABI library with the sm_100a kernels, built in-tree so
# it travels to the GPU box with the repo snapshot.
NVCC ?= /usr/local/cuda/bin/nvcc
# system host compiler (see oracle/Makefile: the inherited $(CXX) is not used)
CXX := g++
PKG := paper_2012_14792_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cpp)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/slicecraft_b200.h
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr -Xptxas -v

all: $(PKG)/libslicecraft_b200.so synth oracle

# synthetic-input generator shared by the bench arms and the tests (not the
# product, not the oracle)
synth: synth/libscsynth.so
synth/libscsynth.so: synth/sc_synth.c
	gcc -std=gnu11 -O2 -fPIC -shared -pthread $< -o $@ -lm

$(PKG)/libslicecraft_b200.so: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared $(SRCS) -o $@ -lpthread 2> build_ptxas.log || (cat build_ptxas.log; false)

oracle:
	$(MAKE) -C oracle

# Link-level drop-in for the reference API (dropin/slicecraft_api.cpp, built
# against the reference HEADERS -- the API contract -- and linked only to the
# product library), and its check: one caller program (dropin/dropin_cases.cpp)
# linked against the drop-in (cases_b200) and, as test infrastructure, against
# the unmodified reference (cases_ref, whose transcript is the golden file).
REF_INC ?= /root/reference/proj/include
DROPIN_FLAGS := -std=c++20 -O2 -Wall -I$(REF_INC) -Iinclude -Idropin
dropin: dropin/libslicecraft_dropin.so dropin/cases_b200 dropin/cases_ref
dropin/libslicecraft_dropin.so: dropin/slicecraft_api.cpp dropin/slicecraft_b200.hpp $(PKG)/libslicecraft_b200.so
	$(CXX) $(DROPIN_FLAGS) -fPIC -shared $< -L$(PKG) -lslicecraft_b200 \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@
dropin/cases_b200: dropin/dropin_cases.cpp dropin/libslicecraft_dropin.so
	$(CXX) $(DROPIN_FLAGS) $< -Ldropin -lslicecraft_dropin -L$(PKG) -lslicecraft_b200 \
	    -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@
dropin/cases_ref: dropin/dropin_cases.cpp oracle
	$(CXX) $(DROPIN_FLAGS) $< -Loracle/_ref -lslicecraft_ref -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -o $@

clean:
	rm -f $(PKG)/libslicecraft_b200.so build_ptxas.log dropin/*.so dropin/cases_b200 dropin/cases_ref synth/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean dropin synth
