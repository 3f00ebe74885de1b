# Builds the product library (sm_100a), the oracle and the input generator.
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 -Xptxas -v
PKG       := paper_2201_02309_b200
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libkatsevich.so
OBJS      := $(CSRC)/precompute.o $(CSRC)/api.o $(CSRC)/filter.o $(CSRC)/backproject.o $(CSRC)/datagen.o
HDRS      := include/katsevich.h $(CSRC)/plan.hpp $(CSRC)/kernels.cuh

all: $(LIB) oracle/liboracle.so synth/libsynth.so

$(CSRC)/%.o: $(CSRC)/%.cu $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(CSRC)/precompute.o: $(CSRC)/precompute.cpp $(HDRS)
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC,-fopenmp,-O3 -x c++ -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fopenmp -lgomp -Xlinker -z,defs

oracle/liboracle.so: oracle/oracle.cpp
	g++ -O2 -std=c++17 -fopenmp -fPIC -shared -o $@ $<

synth/libsynth.so: synth/synth.c
	gcc -O2 -fopenmp -fPIC -shared -o $@ $< -lm

clean:
	rm -f $(CSRC)/*.o $(CSRC)/*.log $(LIB) oracle/liboracle.so synth/libsynth.so

.PHONY: all clean
