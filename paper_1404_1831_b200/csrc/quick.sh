#!/bin/bash
# quick.sh [-D...] INST... : recompile only the named fused-search
# instantiations (e.g. e1_m8 = FBPQ, M=8) and relink libbpq_b200.so with the
# other objects already in build/ (development iterations; run `make`
# before committing).  Prints each instantiation's registers / spills.
set -e
cd "$(dirname "$0")"
defs=()
while [[ "$1" == -D* ]]; do defs+=("$1"); shift; done
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -I../../include -I."
for i in "$@"; do
  e=${i%_m*}; e=${e#e}; m=${i#*_m}
  ( /usr/local/cuda/bin/nvcc $F "${defs[@]}" -DBPQ_INST_ENGINE=$e -DBPQ_INST_M=$m -c search_inst.cu \
      -o build/search_$i.o > build/search_$i.ptxas.log 2>&1 || (cat build/search_$i.ptxas.log; exit 1) ) &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libbpq_b200.so build/*.o -lcudart
for i in "$@"; do
  grep -A2 "Compiling entry function '_ZN3bpq.*search_kernel" build/search_$i.ptxas.log | grep -E "Used|spill" | \
    sed "s/^/$i: /" | head -4
done
