# Builds the in-tree C-ABI library paper_2504_07042_b200/_lib/libhx_axlocal.so
# for sm_100a.  `make -j` compiles the per-order kernel objects in parallel.
NVCC      ?= nvcc
ARCH      ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS   ?= -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $(ARCH)
SRC       := paper_2504_07042_b200/csrc
OBJ       := build/obj
LIB       := paper_2504_07042_b200/_lib/libhx_axlocal.so
ORDERS    := 2 3 4 5 6 7 8 9 10 11 12 13 14 15 16
FAST_ORDERS := 2 3 4 5 6 7 9 10 11 12 13 14 15 16
GEN_OBJS  := $(foreach n,$(ORDERS),$(OBJ)/ax_generic_$(n).o)
FASTN_OBJS := $(foreach n,$(FAST_ORDERS),$(OBJ)/ax_fastn_$(n).o)
LOW_OBJS  := $(OBJ)/ax_low_2.o $(OBJ)/ax_low_3.o
PLANE_OBJS := $(OBJ)/ax_plane_3.o $(OBJ)/ax_plane_4.o
OBJS      := $(GEN_OBJS) $(FASTN_OBJS) $(LOW_OBJS) $(PLANE_OBJS) $(OBJ)/ax_fast.o $(OBJ)/ax_mma.o $(OBJ)/setup.o $(OBJ)/bp5.o $(OBJ)/capi.o
HEADERS   := $(SRC)/hx_common.cuh include/hx_axlocal.h $(wildcard $(SRC)/*.cuh)

all: $(LIB)

$(OBJ):
	mkdir -p $(OBJ) paper_2504_07042_b200/_lib

$(OBJ)/ax_generic_%.o: $(SRC)/ax_generic.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -DHX_N1=$* -c $< -o $@

$(OBJ)/ax_low_%.o: $(SRC)/ax_low.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -DHX_N1=$* -c $< -o $@

$(OBJ)/ax_plane_%.o: $(SRC)/ax_plane.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -fmad=false -DHX_N1=$* -c $< -o $@

$(OBJ)/ax_fastn_%.o: $(SRC)/ax_fastn.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -DHX_N1=$* -c $< -o $@

# ax_mma: no implicit FMA contraction (bitwise n_col = 3 == 3 x n_col = 1 across instantiations)
$(OBJ)/ax_mma.o: $(SRC)/ax_mma.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -fmad=false -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cu $(HEADERS) | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static

clean:
	rm -rf build $(LIB)

.PHONY: all clean
