# Builds: gen (input generators), oracle (CPU test oracle), spchol (the CUDA product library).
NVCC ?= nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2409_14009_b200
CSRC := $(PKG)/csrc
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Iinclude -I$(CSRC)

.PHONY: all gen oracle spchol spchol_check mocknccl clean
all: gen oracle spchol mocknccl

gen: gen/libgen.so
gen/libgen.so: gen/gen.c
	gcc -O2 -shared -fPIC -o $@ $<

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC -pthread -o $@ $< -lm

SPCHOL_SRC := $(wildcard $(CSRC)/*.cu) $(wildcard $(CSRC)/*.cpp)
SPCHOL_HDR := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/spchol.h
spchol: $(PKG)/libspchol.so
$(PKG)/libspchol.so: $(SPCHOL_SRC) $(SPCHOL_HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SPCHOL_SRC) -lcudart -ldl

# bounds-checked test build of the fused cdiv kernels (SPCHOL_PK_CHECK; load with SPCHOL_LIB=...)
spchol_check: $(PKG)/libspchol_check.so
$(PKG)/libspchol_check.so: $(SPCHOL_SRC) $(SPCHOL_HDR)
	$(NVCC) $(NVFLAGS) -DSPCHOL_PK_CHECK -shared -o $@ $(SPCHOL_SRC) -lcudart -ldl

# single-process NCCL stand-in for the multi-rank tests on one GPU (test infrastructure)
mocknccl: tests/mock_nccl/libmocknccl.so
tests/mock_nccl/libmocknccl.so: tests/mock_nccl/mock_nccl.cpp
	g++ -O2 -std=c++17 -shared -fPIC -I$(CUDA_HOME)/include -o $@ $< -L$(CUDA_HOME)/lib64 -lcudart

clean:
	rm -f gen/libgen.so oracle/liboracle.so $(PKG)/libspchol.so $(PKG)/libspchol_check.so tests/mock_nccl/libmocknccl.so
