# Builds the sm_100a C-ABI library in-tree (travels to the GPU box with gpurun).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr $(GTK_EXTRA_FLAGS)
PKG := paper_1901_04359_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
HDR := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/gtopk_b200.h
LIB := $(PKG)/libgtopk_b200.so
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB) oracle

build/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all clean oracle
