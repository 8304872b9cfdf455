#!/bin/bash
# GPU tests, then ncu --set full captures of the large-cell stream kernel and the traversal kernel at c1 and
# c4 (each command first exits 0 without ncu).
tag=${1:-prof}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for cfg in c1 c4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_${cfg}.json 2> gpurun_out/${tag}_${cfg}.err &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'big_scan_kernel|search_kernel' -s 2 -c 2 \
      -o gpurun_out/${tag}_${cfg} python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/${tag}_${cfg}_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/${tag}_${cfg}_ncu.log
done
