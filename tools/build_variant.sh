#!/bin/bash
# Diagnostic builds: libesgd with one source (gemm_tc.cu, or $VARIANT_SRC)
# compiled under extra -D flags
#   tools/build_variant.sh <out.so> -DESGD_X_NOSPLITB ...
#   VARIANT_SRC=conv.cu tools/build_variant.sh <out.so> -DESGD_POOL_MINB=4
# (ESGD_X_* switch off one role's work - results are wrong, only timing counts;
#  ESGD_TRACE adds the clock64 timeline.)  Load with ESGD_LIB=<out.so>.
set -e
cd "$(dirname "$0")/.."
out=$1; shift
src=${VARIANT_SRC:-gemm_tc.cu}
python -c "from paper_1708_02983_b200 import _build; _build.build()"
obj=$(mktemp --suffix=.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
  --expt-relaxed-constexpr -Iinclude "$@" -c "paper_1708_02983_b200/csrc/$src" -o "$obj"
objs=$(ls paper_1708_02983_b200/csrc/_obj/*.o | grep -v "/${src%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" "$obj" $objs -lcudart_static -ldl -lpthread -lrt
rm -f "$obj"
echo "built $out ($*)"
