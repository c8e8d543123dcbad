#!/bin/bash
# Build a variant of liblddmm_cuda.so with extra -D flags for one source file (SRC,
# default gather_pipe.cu):
#   tools/lab/build_variant.sh NAME "-DGP_THREADS=384 -DGP_PREFETCH=0"
#   SRC=umma_gemm.cu tools/lab/build_variant.sh zp_nomma -DZP_NOMMA
# -> tools/lab/build/NAME/liblddmm_cuda.so (use with LDDMM_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
CS=$ROOT/paper_2006_06823_b200/csrc
OUT=$ROOT/tools/lab/build/$1
mkdir -p $OUT
make -C $CS -j8 >/dev/null
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -I$ROOT/include $2 -Xptxas -v -c $CS/${SRC:-gather_pipe.cu} -o $OUT/variant.o 2>&1 \
  | grep -E "spill" | sort | uniq -c || true
B=$(basename ${SRC:-gather_pipe.cu} .cu)
OBJS=$(ls $CS/build/*.o | grep -v "/$B.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OBJS $OUT/variant.o -o $OUT/liblddmm_cuda.so -lcudart
echo built $OUT/liblddmm_cuda.so
