# Builds the C-ABI shared library paper_2602_14449_b200/libots.so for sm_100a.
# One object per translation unit (parallel with make -j), linked into one .so.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
FLAGS := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $(ARCH)
SRC := $(wildcard paper_2602_14449_b200/csrc/*.cu)
HDR := $(wildcard paper_2602_14449_b200/csrc/*.cuh) $(wildcard paper_2602_14449_b200/csrc/*.inc) include/ots.h
OBJDIR := build/obj
OBJ := $(patsubst paper_2602_14449_b200/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
TOBJ := $(patsubst paper_2602_14449_b200/csrc/%.cu,$(OBJDIR)/%.timing.o,$(SRC))
LIB := paper_2602_14449_b200/libots.so

all: $(LIB)

$(OBJDIR)/%.o: paper_2602_14449_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(FLAGS) -Iinclude -c -o $@ $<

$(OBJDIR)/%.timing.o: paper_2602_14449_b200/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(FLAGS) -DOTS_TIMING -Iinclude -c -o $@ $<

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

ptxas: $(SRC) $(HDR)
	$(NVCC) $(FLAGS) -Iinclude -Xptxas -v -shared -o /tmp/ots_ptxas.so $(SRC) 2>&1 | grep -E "Function properties|registers|spill|Compiling entry"

timing: $(TOBJ)
	$(NVCC) $(ARCH) -shared -o paper_2602_14449_b200/libots_timing.so $(TOBJ) -lcudart

clean:
	rm -rf $(LIB) $(OBJDIR)
