#!/bin/bash
# quick_e1.sh: recompile only search_e1.cu (the FBPQ search kernels) and
# relink libbpq_b200.so with the other objects already in build/ -- for
# FBPQ-only iterations.  Run `make` before committing.
set -e
cd "$(dirname "$0")"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xptxas -v --expt-relaxed-constexpr -I../../include -I. -c search_e1.cu -o build/search_e1.o > build/search_e1.ptxas.log 2>&1 \
  || (cat build/search_e1.ptxas.log; exit 1)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200.so build/capi.o build/prep.o \
  build/cells.o build/search.o build/search_e0.o build/search_e1.o build/search_e2.o build/encode.o -lcudart
grep -A3 "Compiling entry function.*search_kernel" build/search_e1.ptxas.log | grep -E "Compiling|spill" | \
  sed 's/.*search_kernel\(ILi[0-9]*ELi[0-9]*EfjLb[01]E\).*/\1/' | paste - - 
