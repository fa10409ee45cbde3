# Builds the product library (paper_1907_06154_b200/libssam_b200.so, sm_100a)
# and the test-only checkers (oracle/).  `make -j` from the repo root.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX := g++
CUDA_HOME ?= /usr/local/cuda
PKG := paper_1907_06154_b200
SRC := $(PKG)/csrc
BUILD := build
LIB := $(PKG)/libssam_b200.so
CLI := $(PKG)/bin/ssam

ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(SRC) \
           --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -std=c++17 -O2 -fPIC -Wall -Iinclude -I$(SRC) -I$(CUDA_HOME)/include

CU_SRCS := $(wildcard $(SRC)/*.cu)
CU_OBJS := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS := $(BUILD)/abi.o $(BUILD)/tmap.o $(BUILD)/grid_io.o $(BUILD)/multi.o
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.hpp) include/ssam_b200.h

all: $(LIB) $(CLI) oracle dropin

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/abi.o: $(SRC)/abi.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xlinker -soname=libssam_b200.so $^ -o $@

# The `ssam` command line (proj/tools/ssam_cli.cpp mirror) over the C ABI.
$(CLI): $(PKG)/cli/ssam_cli.cpp include/ssam_b200.h $(LIB)
	@mkdir -p $(PKG)/bin
	$(CXX) -std=c++17 -O2 -Wall -Iinclude $< $(LIB) -Wl,-rpath,'$$ORIGIN/..' -o $@

oracle:
	$(MAKE) -C oracle

# Variant builds for A/B experiments: make variant VAR=name VFLAGS="-D..." ->
# build/var_name/libssam_b200.so (load with SSAM_B200_LIB=...).  `make debug`
# is the variant with bounded mbarrier waits that report and trap.
VAR ?= dbg
VFLAGS ?= -DSSAM_DEBUG_HANG
VDIR := build/var_$(VAR)
V_OBJS := $(patsubst $(SRC)/%.cu,$(VDIR)/%.o,$(CU_SRCS))
$(VDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(VDIR)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $< -o $@
$(VDIR)/libssam_b200.so: $(V_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -Xlinker -soname=libssam_b200.so $^ -o $@
variant: $(VDIR)/libssam_b200.so
# Quick A/B of one translation unit: recompile only $(VSRC) with VFLAGS and
# link it with the main build's other objects -> build/qv_$(VAR)/libssam_b200.so
VSRC ?= star3d
QDIR := build/qv_$(VAR)
$(QDIR)/libssam_b200.so: $(SRC)/$(VSRC).cu $(HDRS) $(CU_OBJS) $(CPP_OBJS)
	@mkdir -p $(QDIR)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -c $(SRC)/$(VSRC).cu -o $(QDIR)/$(VSRC).o
	$(NVCC) $(ARCH) -shared -cudart static -Xlinker -soname=libssam_b200.so $(QDIR)/$(VSRC).o $(filter-out $(BUILD)/$(VSRC).o,$(CU_OBJS)) $(CPP_OBJS) -o $@
qvariant: $(QDIR)/libssam_b200.so
.PHONY: qvariant
debug:
	$(MAKE) variant VAR=dbg VFLAGS=-DSSAM_DEBUG_HANG
.PHONY: variant debug

clean:
	rm -rf $(BUILD) $(LIB) $(CLI)

.PHONY: all oracle clean

$(BUILD)/grid_io.o: $(SRC)/grid_io.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/tmap.o: $(SRC)/tmap.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# C++ drop-in parity test: the reference's own hot-path tests against
# include/ssam_b200/kernels.hpp (types + oracle from the reference headers).
REF ?= /root/reference/proj
DROPIN := tests/cpp/bin/dropin_parity
ifneq ($(wildcard $(REF)/include/ssam/oracle.hpp),)
dropin: $(DROPIN)
$(DROPIN): tests/cpp/dropin_parity.cpp include/ssam_b200/kernels.hpp include/ssam_b200.h $(LIB) oracle
	@mkdir -p tests/cpp/bin
	$(CXX) -std=c++20 -O2 -Iinclude -I$(REF)/include $< $(LIB) oracle/_ref/libssam_ref.so \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)' -Wl,-rpath,'$$ORIGIN/../../../oracle/_ref' -o $@
else
dropin:
	@echo "reference headers absent; keeping prebuilt $(DROPIN) (if any)"
endif

.PHONY: dropin

$(BUILD)/multi.o: $(SRC)/multi.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@
