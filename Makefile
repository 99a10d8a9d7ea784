# Builds the sm_100a shared library in-tree (travels to the GPU box with the snapshot).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -Xptxas -v $(EXTRA)
SRC := paper_1608_03589_b200/csrc
LIB := paper_1608_03589_b200/liblpbp.so
OBJS := build/kernels.o build/direct_kernels.o build/sector_kernels.o build/bst_kernels.o build/resample_kernels.o build/capi.o build/plan_host.o build/sector_host.o build/bst_host.o

all: $(LIB)

build/%.o: $(SRC)/%.cu $(SRC)/*.cuh include/lpbp.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

build/%.o: $(SRC)/%.cpp $(SRC)/*.h
	@mkdir -p build
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC,-O3 -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread

clean:
	rm -rf build $(LIB)
.PHONY: all clean
