# Builds the product library (sm_100a) and the test-side C helpers.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2501_17168_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libevogp.so
# IEEE-faithful FP32 on the parity path: no fast math, no FTZ, IEEE div/sqrt (R5)
NVFLAGS := -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
           -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -Xptxas -v
# one translation unit per evaluation-kernel family so `make -j` builds them in parallel
CU := eval_full eval_inter_k16 eval_intra_k16 eval_inter_k8 eval_inter_k4 eval_inter_k2 eval_inter_k1 eval_intra_k8 eval_intra_k4 compile plan \
      paired variation tensorize_dev capi
OBJDIR := build/obj
OBJS := $(addprefix $(OBJDIR)/,$(addsuffix .o,$(CU))) $(OBJDIR)/tensorize.o
HDRS := $(CSRC)/evogp_internal.h $(CSRC)/fastmath.cuh $(CSRC)/decode.cuh $(CSRC)/interp.cuh $(CSRC)/hot.cuh $(CSRC)/hot_ptx.inc \
        $(CSRC)/selector_table.inc include/evogp.h

all: $(LIB) oracle/liboracle.so synth/libsynth.so

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJDIR)/tensorize.o: $(CSRC)/tensorize.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJS)
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -o $@ $(OBJS) -lcudart
	cat $(OBJDIR)/*.ptxas.log > $(PKG)/ptxas.log

# test infrastructure (never linked into the product)
oracle/liboracle.so: oracle/oracle.c oracle/variation.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -o $@ oracle/oracle.c oracle/variation.c -lm

synth/libsynth.so: synth/synth.c
	gcc -O2 -fPIC -shared -pthread -o $@ $< -lm

clean:
	rm -rf $(LIB) oracle/liboracle.so synth/libsynth.so $(PKG)/ptxas.log $(OBJDIR)

.PHONY: all clean
