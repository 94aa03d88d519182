# Builds the product library (sm_100a kernels + C ABI) and the CPU oracle.
# `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC    ?= /usr/local/cuda/bin/nvcc
CXX     := /usr/bin/g++
CC      := /usr/bin/gcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2002_02145_b200
CSRC    := $(PKG)/csrc
BUILD   := build
INC     := -Iinclude -I$(CSRC)
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $(INC)
CXXFLAGS:= -O3 -std=c++17 -fPIC -fopenmp $(INC)

LIB     := $(PKG)/libpsconv.so
CU_OBJS := $(BUILD)/conv_fwd.o
CC_OBJS := $(BUILD)/desc.o $(BUILD)/recipe.o $(BUILD)/select.o $(BUILD)/emit.o $(BUILD)/microkernel_cpu.o $(BUILD)/nest.o $(BUILD)/dnnrank.o
HDRS    := include/psconv.h $(wildcard $(CSRC)/*.hpp) $(wildcard $(CSRC)/*.cuh)

ORACLE  := oracle/liboracle.so

.PHONY: all lib oracle clean
all: lib oracle

lib: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/conv_fwd.o: $(CSRC)/conv_fwd.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_conv_fwd.txt || (cat $(BUILD)/ptxas_conv_fwd.txt; exit 1)

$(BUILD)/%.o: $(CSRC)/%.cpp $(HDRS) | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CC_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fopenmp -lgomp

# CPU oracle: test infrastructure only (tests/, smoke(), bench.py cpu_baseline).
# -ffp-contract=off: no FMA contraction, so the fp32 restatement accumulates
# exactly like the reference IR interpreter (bit-exact pin).
$(ORACLE): oracle/oracle.c oracle/oracle.h | $(BUILD)
	$(CC) -O3 -std=c11 -fPIC -shared -fopenmp -ffp-contract=off -march=x86-64-v3 -Ioracle -o $@ $<

oracle: $(ORACLE)

clean:
	rm -rf $(BUILD) $(LIB) $(ORACLE)
