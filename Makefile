# Builds the sm_100a product library and the CPU oracle (test infrastructure).
PY      ?= python
SITE    := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL    := $(SITE)/nvidia/nccl
CUDART  := $(SITE)/nvidia/cuda_runtime/lib
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -I$(NCCL)/include \
           -Xptxas -v -cudart shared
PKG     := paper_2210_17357_b200
SRCS    := $(wildcard $(PKG)/csrc/*.cu)
HDRS    := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/lgreco.h
LIB     := $(PKG)/liblgreco.so
ORACLE  := oracle/liblgreco_ref.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) -L$(NCCL)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL)/lib -Xlinker -rpath=$(CUDART) 2> build/ptxas.log || (cat build/ptxas.log; false)

$(ORACLE): oracle/lgreco_ref.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

clean:
	rm -f $(LIB) $(ORACLE)

.PHONY: all clean
