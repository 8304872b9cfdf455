#!/bin/bash
# variant.sh NAME [extra nvcc flags...]: rebuild only search_e1.cu (FBPQ) from
# /tmp/var_NAME/ (a copy of csrc with edits) and link libbpq_b200_NAME.so
# with the main build's other objects.  For A/B timing experiments.
set -e
name=$1; shift
here="$(cd "$(dirname "$0")" && pwd)"
d=/tmp/var_$name
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Xptxas -v -I$here/../../include -I$d "$@" -c $d/search_e1.cu -o $d/search_e1.o > $d/ptxas.log 2>&1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $here/../libbpq_b200_$name.so \
  $here/build/capi.o $here/build/prep.o $here/build/cells.o $here/build/search.o $here/build/search_e0.o \
  $d/search_e1.o $here/build/search_e2.o $here/build/encode.o -lcudart
grep -A3 "search_kernelILi1ELi8EfjE" $d/ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo " <- $name"
