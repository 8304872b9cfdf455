#!/bin/bash
# c4 (N=1e9, T=16384, M=8) bench line, then one ncu --set full capture of the large-cell stream kernel.
tag=${1:-c4}
mkdir -p gpurun_out
timeout 1200 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 1200 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_plain.json 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"big_scan|big_stream|cell_stream" -s 3 -c 1 \
    -o gpurun_out/${tag}_stream python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --recall-queries 0 \
    > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
