#!/bin/bash
# phase profile + ncu --set full of cell_flow_kernel at c4 and c1
tag=${1:-flowncu}
o=gpurun_out
mkdir -p $o
for cfg in c4 c1; do
  B="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
  BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 $B --phase-profile > $o/${tag}_${cfg}_prof.json 2> $o/${tag}_${cfg}_prof.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cell_flow -s 3 -c 1 -o $o/${tag}_${cfg}_flow \
      $B > $o/${tag}_${cfg}_ncu.log 2>&1
  echo "ncu rc=$?" >> $o/${tag}_${cfg}_ncu.log
done
