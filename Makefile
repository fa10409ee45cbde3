# Builds the product library (paper_1907_06154_b200/libssam_b200.so, sm_100a)
# and the test-only checkers (oracle/).  `make -j` from the repo root.
NVCC ?= /usr/local/cuda/bin/nvcc
CXX := g++
CUDA_HOME ?= /usr/local/cuda
PKG := paper_1907_06154_b200
SRC := $(PKG)/csrc
BUILD := build
LIB := $(PKG)/libssam_b200.so

ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(SRC) \
           --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -std=c++17 -O2 -fPIC -Wall -Iinclude -I$(SRC) -I$(CUDA_HOME)/include

CU_SRCS := $(wildcard $(SRC)/*.cu)
CU_OBJS := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS := $(BUILD)/abi.o $(BUILD)/tmap.o
HDRS := $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.hpp) include/ssam_b200.h

all: $(LIB) oracle

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/abi.o: $(SRC)/abi.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -cudart static $^ -o $@

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all oracle clean

$(BUILD)/tmap.o: $(SRC)/tmap.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@
