# libclimber.so for sm_100a (B200).  `make` or __graft_entry__.build().
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) $(EXTRA) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := paper_2502_09888_b200/csrc
OUT := paper_2502_09888_b200/lib
OBJS := $(OUT)/api.o $(OUT)/kernels.o $(OUT)/gemm_tc.o $(OUT)/attn_mma.o $(OUT)/attn_fa.o
HDRS := $(wildcard $(SRC)/*.cuh) include/climber.h

all: $(OUT)/libclimber.so

$(OUT)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OUT)/libclimber.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

clean:
	rm -rf $(OUT)

.PHONY: all clean
