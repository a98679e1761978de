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

# Checked build: bounds checks, asserts and barrier jitter (common.cuh ADMM_CHECKED).
#   make checked; ADMM_B200_LIB=$(CHECKED_LIB) python -m pytest tests -m gpu
CHECKED_LIB := paper_1204_0556_b200/libadmm_b200_checked.so
CHECKED_OBJS := $(patsubst $(BUILD)/%,build_checked/%,$(OBJS))

checked: $(CHECKED_LIB)

build_checked/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build_checked
	$(NVCC) $(NVFLAGS) -DADMM_CHECKED -c $< -o $@ > build_checked/$*.ptxas.log 2>&1 || (cat build_checked/$*.ptxas.log; exit 1)

$(CHECKED_LIB): $(CHECKED_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CHECKED_OBJS) -lcudart

clean:
	rm -rf $(BUILD) build_checked $(LIB) $(CHECKED_LIB)

.PHONY: all clean checked
