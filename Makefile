# Builds the C-ABI shared library paper_2602_14449_b200/libots.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $(ARCH)
SRC := $(wildcard paper_2602_14449_b200/csrc/*.cu)
HDR := $(wildcard paper_2602_14449_b200/csrc/*.cuh) $(wildcard paper_2602_14449_b200/csrc/*.inc) include/ots.h
LIB := paper_2602_14449_b200/libots.so

all: $(LIB)

$(LIB): $(SRC) $(HDR)
	$(NVCC) $(FLAGS) -Iinclude -shared -o $@ $(SRC) -lcudart

ptxas: $(SRC) $(HDR)
	$(NVCC) $(FLAGS) -Iinclude -Xptxas -v -shared -o /tmp/ots_ptxas.so $(SRC) 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" 

timing: $(SRC) $(HDR)
	$(NVCC) $(FLAGS) -DOTS_TIMING -Iinclude -shared -o paper_2602_14449_b200/libots_timing.so $(SRC) -lcudart

clean:
	rm -f $(LIB)
