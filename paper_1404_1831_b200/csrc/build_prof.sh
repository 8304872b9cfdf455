#!/bin/bash
# Phase-profiling variant of the engine (-DBPQ_PHASE_PROF) for bench.py
# --phase-profile (BPQ_LIB=.../libbpq_b200_prof.so).  build_prof.sh [INST...]
# rebuilds only the named fused-search instantiations (default e1_m8) with
# the counters and links the others from build/ (run `make` first).
set -e
cd "$(dirname "$0")"
mkdir -p build_prof
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBPQ_PHASE_PROF -I../../include -I."
insts=("$@")
[ ${#insts[@]} -eq 0 ] && insts=(e1_m8)
for i in "${insts[@]}"; do
  e=${i%_m*}; e=${e#e}; m=${i#*_m}
  /usr/local/cuda/bin/nvcc $F -DBPQ_INST_ENGINE=$e -DBPQ_INST_M=$m -c search_inst.cu -o build_prof/search_$i.o &
done
# the large-cell stream kernels live in their own translation units
for m in 8 16; do
  /usr/local/cuda/bin/nvcc $F -DBPQ_INST_M=$m -c stream_inst.cu -o build_prof/stream_m$m.o &
done
wait
objs=()
for o in build/*.o; do
  b=$(basename $o)
  if [ -f build_prof/$b ] && { [[ " ${insts[*]/%/.o} " == *" ${b#search_} "* ]] || [[ $b == stream_m* ]]; }; then objs+=(build_prof/$b); else objs+=($o); fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200_prof.so "${objs[@]}" -lcudart
echo "linked: ${objs[*]}"
