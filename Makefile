# Product library (sm_100a) + test-infrastructure oracles.
#   make            -> paper_2407_11349_b200/libhawkes_b200.so, oracle/liboracle.so
#   make ref        -> oracle/_ref/libhawkes_ref.so (needs /root/reference; not shipped)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v
CSRC := paper_2407_11349_b200/csrc
LIB := paper_2407_11349_b200/libhawkes_b200.so
SRCS := $(CSRC)/hk_kernels.cu $(CSRC)/hk_capi.cu $(CSRC)/hk_regions.cu $(CSRC)/hk_fgt.cu $(CSRC)/hk_cells.cu $(CSRC)/hk_host.cpp
HDRS := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/hawkes_b200.h

all: $(LIB) oracle

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared $(SRCS) -o $@ 2> build_ptxas.log || (cat build_ptxas.log; false)

# Device bounds checks (HK_ASSERT) on: run the GPU tests against it with
# HK_LIB=paper_2407_11349_b200/libhawkes_b200_debug.so.
debug: $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -DHK_DEBUG -shared $(SRCS) -o paper_2407_11349_b200/libhawkes_b200_debug.so 2> build_ptxas_debug.log || (cat build_ptxas_debug.log; false)

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(LIB) paper_2407_11349_b200/libhawkes_b200_debug.so build_ptxas.log build_ptxas_debug.log
	$(MAKE) -C oracle clean

.PHONY: all oracle ref clean debug
