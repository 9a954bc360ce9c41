# Build every native artefact in-tree (same commands as __graft_entry__.build()).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared

all: paper_2110_07519_b200/libmessi.so datagen/libdatagen.so oracle/liboracle.so

paper_2110_07519_b200/libmessi.so: paper_2110_07519_b200/csrc/*.cu paper_2110_07519_b200/csrc/*.cuh include/messi.h
	$(NVCC) $(NVFLAGS) -o $@ paper_2110_07519_b200/csrc/api.cu

datagen/libdatagen.so: datagen/datagen.cu
	$(NVCC) $(ARCH) -O3 -lineinfo -fmad=false -Xcompiler -fPIC -shared -o $@ $<

oracle/liboracle.so: oracle/messi_oracle.c
	gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

clean:
	rm -f paper_2110_07519_b200/libmessi.so datagen/libdatagen.so oracle/liboracle.so

.PHONY: all clean
