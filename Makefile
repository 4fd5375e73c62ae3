# Top-level build (driven by __graft_entry__.build()).
#
#   paper_2604_25422_b200/libks_dwconv1d.so   sm_100a kernels + C ABI + C++ drop-in
#   tests/cpp/test_dropin                      C++ tests of the drop-in API (GPU)
#   oracle/liboracle.so, oracle/_ref/*         CPU parity checkers (oracle/Makefile)
#   oracle/_ref/ref_test_conv_core             the reference's own operator tests
#                                              compiled against OUR headers + library
#
# Every .so/binary is git-ignored and travels to the GPU box with the snapshot.

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2604_25422_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/libks_dwconv1d.so
REF_ROOT ?= /root/reference/proj

NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Iinclude -I$(CSRC) \
            --expt-relaxed-constexpr -Xptxas -v -Xcompiler -Wall
CU_SRCS  := $(CSRC)/capi.cu $(CSRC)/conv_fwd.cu $(CSRC)/conv_dw.cu $(CSRC)/conv_tma.cu \
            $(CSRC)/stencil_tma.cu $(CSRC)/dw_tma.cu $(CSRC)/bwd_short_dw.cu $(CSRC)/bwd_short_dx.cu $(CSRC)/bwd_short_st.cu $(CSRC)/stencil_ldg.cu $(CSRC)/dw_pairwise_tma.cu $(CSRC)/paper_variants.cu $(CSRC)/stencil_pad.cu $(CSRC)/rows_short.cu $(CSRC)/dw_pad.cu \
            $(CSRC)/host_api.cu $(CSRC)/dist.cu $(CSRC)/peer.cu $(CSRC)/options.cu
CPP_SRCS := $(CSRC)/conv_core.cpp
OBJDIR   := build/obj
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRCS))
HDRS     := include/ks_dwconv1d.h $(wildcard include/kernelscope/*.hpp) $(wildcard $(CSRC)/*.cuh)

.PHONY: all lib oracle tests clean
all: lib oracle tests

lib: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -O2 -std=c++20 -fPIC -Wall -Wextra -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lnccl -Xlinker -soname=libks_dwconv1d.so

oracle:
	$(MAKE) -C oracle

TEST_BIN := tests/cpp/test_dropin
tests: $(TEST_BIN) refsuite

$(TEST_BIN): tests/cpp/test_dropin.cpp $(LIB) tests/cpp/doctest_shim/doctest.h oracle
	$(CXX) -O2 -std=c++20 -Wall -Iinclude -Itests/cpp/doctest_shim -Ioracle -o $@ $< -lpthread \
	    -L$(PKG) -lks_dwconv1d -Loracle -loracle \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../oracle'

# The reference's own tests/test_conv_core.cpp, compiled from /root/reference
# (never copied) against this repo's kernelscope/*.hpp and linked to the B200
# library: the drop-in acceptance test.  Skipped when the reference is absent.
ifneq ($(wildcard $(REF_ROOT)/tests/test_conv_core.cpp),)
refsuite: oracle/_ref/ref_test_conv_core
oracle/_ref/ref_test_conv_core: $(REF_ROOT)/tests/test_conv_core.cpp $(LIB) tests/cpp/doctest_shim/doctest.h
	@mkdir -p oracle/_ref
	$(CXX) -O2 -std=c++20 -Iinclude -Itests/cpp/doctest_shim -I$(REF_ROOT)/tests -o $@ $< -lpthread \
	    -L$(PKG) -lks_dwconv1d -Wl,-rpath,'$$ORIGIN/../../$(PKG)'
else
refsuite:
	@echo "refsuite: $(REF_ROOT) absent; using prebuilt oracle/_ref/ref_test_conv_core if present"
endif

clean:
	rm -rf build $(LIB) $(TEST_BIN) oracle/_ref/ref_test_conv_core
	$(MAKE) -C oracle clean
