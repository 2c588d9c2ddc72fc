#!/bin/bash
# Build liblgreco.so variants of one translation unit with extra -D flags (for A/B runs
# through LGRECO_LIB).  Usage: scripts/build_variants.sh qsgd "A:-DQP_XU_CEIL=0" "B:-DQP_XU_CEIL=4" ...
set -e
cd "$(dirname "$0")/.."
TU=$1; shift
PY=python
SITE=$($PY -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL=$SITE/nvidia/nccl; CUDART=$SITE/nvidia/cuda_runtime/lib
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build/var
OTHERS=$(for f in paper_2210_17357_b200/csrc/*.cu; do b=$(basename $f .cu); [ "$b" != "$TU" ] && echo build/obj/$b.o; done)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC -Iinclude -I$NCCL/include -cudart shared $flags \
    -c -o build/var/${TU}_$name.o paper_2210_17357_b200/csrc/$TU.cu &
done
wait
for spec in "$@"; do
  name=${spec%%:*}
  nvcc $ARCH -cudart shared -shared -o build/var/liblgreco_$name.so build/var/${TU}_$name.o $OTHERS \
    -L$NCCL/lib -l:libnccl.so.2 \
    -Xlinker -rpath=$NCCL/lib -Xlinker -rpath=$CUDART
done
ls build/var/*.so
