#!/bin/bash
# ncu --set full of one kernel (regex $2) at config $3 -> gpurun_out/$1.ncu-rep
tag=$1; kn=$2; cfg=${3:-c4}
o=gpurun_out; mkdir -p $o
B="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 $B > $o/${tag}_plain.json 2> $o/${tag}_plain.err &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kn -s 3 -c 1 -o $o/${tag} $B > $o/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> $o/${tag}_ncu.log
