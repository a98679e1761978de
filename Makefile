# Build the C-ABI shared library for sm_100a (B200).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
SRC_DIR := paper_1204_0556_b200/csrc
BUILD := build
LIB := paper_1204_0556_b200/libadmm_b200.so
OBJS := $(BUILD)/abi.o $(BUILD)/resident_f32.o $(BUILD)/resident_f64.o $(BUILD)/project.o $(BUILD)/streaming.o $(BUILD)/steps.o $(BUILD)/cluster.o $(BUILD)/bp.o $(BUILD)/wide.o
HDRS := $(wildcard $(SRC_DIR)/*.cuh) $(wildcard $(SRC_DIR)/*.h) include/admm_b200.h

all: $(LIB)

$(BUILD)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $(BUILD)/$*.ptxas.log 2>&1 || (cat $(BUILD)/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

$(SRC_DIR)/sortnet.cuh: tools/gen_sortnet.py
	python tools/gen_sortnet.py

clean:
	rm -rf $(BUILD) $(LIB)

.PHONY: all clean
