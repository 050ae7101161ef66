# Build libnef.so (C ABI + sm_100a kernels) in-tree.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -Wall $(ARCH) --expt-relaxed-constexpr
SRC := $(wildcard paper_2602_02759_b200/csrc/*.cu) $(wildcard paper_2602_02759_b200/csrc/*.cpp)
HDR := $(wildcard paper_2602_02759_b200/csrc/*.h) $(wildcard paper_2602_02759_b200/csrc/*.cuh) $(wildcard paper_2602_02759_b200/csrc/*.inc) include/nef.h
LIB := paper_2602_02759_b200/libnef.so
OBJDIR := build/obj
OBJ := $(patsubst paper_2602_02759_b200/csrc/%,$(OBJDIR)/%.o,$(SRC))

all: $(LIB)

$(OBJDIR)/%.o: paper_2602_02759_b200/csrc/% $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(FLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean
