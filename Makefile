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
ORACLE_OMP := oracle/liblgreco_ref_omp.so

all: $(LIB) $(ORACLE) $(ORACLE_OMP)

OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRCS))

# one object per translation unit (parallel with make -j); the ptxas -v report of
# every unit is concatenated into build/ptxas.log
build/obj/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/obj/$*.ptxas.log || (cat build/obj/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -cudart shared -shared -o $@ $(OBJS) -L$(NCCL)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL)/lib -Xlinker -rpath=$(CUDART)
	cat build/obj/*.ptxas.log > build/ptxas.log

$(ORACLE): oracle/lgreco_ref.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

# the same oracle with its layer loops on all host cores (bench.py cpu_baseline only)
$(ORACLE_OMP): oracle/lgreco_ref.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -fopenmp -shared -o $@ $< -lm

clean:
	rm -f $(LIB) $(ORACLE) $(ORACLE_OMP)

.PHONY: all clean timing

# diagnostic build: k_solve_fast prints its phase cycle counts (scripts/dp_timing.py)
build/obj/dp_timing.o: $(PKG)/csrc/dp.cu $(HDRS)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -DLG_DP_TIMING -c -o $@ $< 2> /dev/null

build/liblgreco_timing.so: $(filter-out build/obj/dp.o,$(OBJS)) build/obj/dp_timing.o
	$(NVCC) $(ARCH) -cudart shared -shared -o $@ $^ -L$(NCCL)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath=$(NCCL)/lib -Xlinker -rpath=$(CUDART)

timing: build/liblgreco_timing.so
