#!/bin/bash
# c4 bench line (with recall) and one ncu --set full capture (source-level) of the large-cell stream kernel
tag=$1
mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:big_scan -s 1 -c 1 \
    -o gpurun_out/${tag}_c4 python bench.py --config c4 --steps 1 --warmup 1 --no-cpu-baseline --recall-queries 0 \
    > gpurun_out/${tag}_c4_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_c4_ncu.log
