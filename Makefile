# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with
# the gpurun snapshot).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           --expt-relaxed-constexpr -Iinclude -Ipaper_1707_07803_b200/csrc
SRC := $(wildcard paper_1707_07803_b200/csrc/*.cu)
OBJ := $(patsubst paper_1707_07803_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1707_07803_b200/lib/libmpo_b200.so

all: $(LIB)

build/%.o: paper_1707_07803_b200/csrc/%.cu $(wildcard paper_1707_07803_b200/csrc/*.cuh) include/mpo_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

clean:
	rm -rf build $(LIB)

.PHONY: all clean
