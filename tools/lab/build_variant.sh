#!/bin/bash
# Build a variant of liblddmm_cuda.so with extra -D flags for gather_pipe.cu only:
#   tools/lab/build_variant.sh NAME "-DGP_THREADS=384 -DGP_PREFETCH=0"
# -> tools/lab/build/NAME/liblddmm_cuda.so (use with LDDMM_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
CS=$ROOT/paper_2006_06823_b200/csrc
OUT=$ROOT/tools/lab/build/$1
mkdir -p $OUT
make -C $CS -j8 >/dev/null
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -I$ROOT/include $2 -Xptxas -v -c $CS/gather_pipe.cu -o $OUT/gather_pipe.o 2>&1 \
  | grep -A1 "ILi3ELi192" | grep -E "spill|registers" || true
OBJS=$(ls $CS/build/*.o | grep -v gather_pipe.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OBJS $OUT/gather_pipe.o -o $OUT/liblddmm_cuda.so -lcudart
echo built $OUT/liblddmm_cuda.so
