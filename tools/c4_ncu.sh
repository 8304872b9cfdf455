#!/bin/bash
# c4 (N=1e9, T=16384, M=8) bench line, launch list and one ncu --set full capture of the fused search kernel.
tag=${1:-c4}
mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 2 -c 1 \
    -o gpurun_out/${tag}_search python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
