#!/bin/bash
# Checked variant of the engine (-DBPQ_CHECKED): the large-cell stream kernel tests every index it forms
# against its array bound and counts violations into counter 19 of the diagnostics buffer.  Only the stream
# translation units are rebuilt; the others link from build/ (run `make` first).
set -e
cd "$(dirname "$0")"
mkdir -p build_checked
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBPQ_CHECKED -I../../include -I."
for m in 8 16; do
  /usr/local/cuda/bin/nvcc $F -DBPQ_INST_M=$m -c stream_inst.cu -o build_checked/stream_m$m.o &
done
wait
objs=()
for o in build/*.o; do
  b=$(basename $o)
  if [[ $b == stream_m* ]]; then objs+=(build_checked/$b); else objs+=($o); fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200_checked.so "${objs[@]}" -lcudart
