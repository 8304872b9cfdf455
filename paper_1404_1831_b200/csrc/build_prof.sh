#!/bin/bash
# Phase-profiling variant of the engine (-DBPQ_PHASE_PROF) for bench.py --phase-profile.
set -e
cd "$(dirname "$0")"
mkdir -p build_prof
for f in capi prep cells search search_e0 search_e1 search_e2 encode; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -DBPQ_PHASE_PROF -I../../include -I. -c $f.cu -o build_prof/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200_prof.so build_prof/*.o -lcudart
