# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
SRC := $(wildcard paper_1303_5466_b200/csrc/*.cu)
OBJ := $(patsubst paper_1303_5466_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1303_5466_b200/_lib/libvief_b200.so

all: $(LIB)

build/%.o: paper_1303_5466_b200/csrc/%.cu paper_1303_5466_b200/csrc/common.cuh include/vief_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p paper_1303_5466_b200/_lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
