# Builds the B200 engine (libpfb200.so) and the C oracle.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $(EXTRA)
SRC := paper_1710_08826_b200/csrc
OUT := paper_1710_08826_b200/_native
LIB := $(OUT)/libpfb200.so
OBJS := $(OUT)/pfb_nll.o $(OUT)/pfb_nll_sop.o $(OUT)/pfb_nll_dal.o $(OUT)/pfb_dalitz.o $(OUT)/pfb_binned.o $(OUT)/pfb_pcg.o $(OUT)/pfb_io.o $(OUT)/pfb_peer.o $(OUT)/pfb_gen.o $(OUT)/pfb_api.o
HDRS := $(SRC)/pfb_objective.cuh $(SRC)/pfb_nll_task.cuh $(SRC)/pfb_internal.cuh $(SRC)/pfb_math.cuh $(SRC)/pfb_nll_kernel.cuh $(SRC)/pfb_nll_tma.cuh $(SRC)/pfb_nll_prod.cuh include/pfb200.h

all: $(LIB)

$(OUT)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OUT)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OUT)/$*.ptxas.log || (cat $(OUT)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

clean:
	rm -rf $(OUT)/*.o $(LIB)

.PHONY: all clean
