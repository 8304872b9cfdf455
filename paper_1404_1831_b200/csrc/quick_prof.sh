#!/bin/bash
# quick_prof.sh: phase-profiling variant (-DBPQ_PHASE_PROF) of search.cu and
# search_e1.cu only, linked with the other objects of build/ into
# libbpq_b200_prof.so (bench.py --phase-profile with BPQ_LIB=...).
set -e
cd "$(dirname "$0")"
mkdir -p build_prof
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBPQ_PHASE_PROF -I../../include -I."
/usr/local/cuda/bin/nvcc $F -c search.cu -o build_prof/search.o &
/usr/local/cuda/bin/nvcc $F -c search_e1.cu -o build_prof/search_e1.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200_prof.so build/capi.o build/prep.o \
  build/cells.o build_prof/search.o build/search_e0.o build_prof/search_e1.o build/search_e2.o build/encode.o -lcudart
