#!/bin/bash
# ncu --set full of the large-cell stream kernel at c4 and c1 (each command first exits 0 without ncu)
tag=$1
mkdir -p gpurun_out
for cfg in c4 c1; do
  timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_${cfg}_plain.json 2>&1 &&
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:big_scan -s 2 -c 1 \
      -o gpurun_out/${tag}_${cfg} python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline --recall-queries 0 \
      > gpurun_out/${tag}_${cfg}_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/${tag}_${cfg}_ncu.log
done
