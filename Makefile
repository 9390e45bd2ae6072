# Builds the product library (sm_100a) and the test-side C helpers.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2501_17168_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/libevogp.so
# IEEE-faithful FP32 on the parity path: no fast math, no FTZ, IEEE div/sqrt (R5)
NVFLAGS := -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
           -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-O2 -Xptxas -v
SRCS := $(CSRC)/kernels.cu $(CSRC)/paired.cu $(CSRC)/variation.cu $(CSRC)/tensorize_dev.cu $(CSRC)/capi.cu $(CSRC)/tensorize.cpp
HDRS := $(CSRC)/evogp_internal.h $(CSRC)/fastmath.cuh $(CSRC)/decode.cuh $(CSRC)/selector_table.inc include/evogp.h

all: $(LIB) oracle/liboracle.so synth/libsynth.so

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> $(PKG)/ptxas.log || (cat $(PKG)/ptxas.log; exit 1)

# test infrastructure (never linked into the product)
oracle/liboracle.so: oracle/oracle.c oracle/variation.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -o $@ oracle/oracle.c oracle/variation.c -lm

synth/libsynth.so: synth/synth.c
	gcc -O2 -fPIC -shared -pthread -o $@ $< -lm

clean:
	rm -f $(LIB) oracle/liboracle.so synth/libsynth.so $(PKG)/ptxas.log

.PHONY: all clean
