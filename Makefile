# Builds the B200-native C-ABI library in-tree (it travels to the GPU box with the snapshot).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
SRC_DIR := paper_1407_7506_b200/csrc
SRCS := $(wildcard $(SRC_DIR)/*.cu)
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_1407_7506_b200/libppcg_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(SRC_DIR)/common.cuh include/ppcg_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L/usr/local/cuda/lib64 -lcusolver -lcublas -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
