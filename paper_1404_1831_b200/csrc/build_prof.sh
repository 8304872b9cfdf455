#!/bin/bash
# Phase-profiling variant of the engine (-DBPQ_PHASE_PROF) for bench.py
# --phase-profile (BPQ_LIB=.../libbpq_b200_prof.so).
set -e
cd "$(dirname "$0")"
mkdir -p build_prof
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBPQ_PHASE_PROF -I../../include -I."
for f in capi prep cells search encode; do /usr/local/cuda/bin/nvcc $F -c $f.cu -o build_prof/$f.o & done
for i in e1_m8 e1_m16 e2_m8 e2_m16 e0_m8 e0_m16 e1_m0 e2_m0 e0_m0; do
  e=${i%_m*}; e=${e#e}; m=${i#*_m}
  /usr/local/cuda/bin/nvcc $F -DBPQ_INST_ENGINE=$e -DBPQ_INST_M=$m -c search_inst.cu -o build_prof/search_$i.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200_prof.so build_prof/*.o -lcudart
