#!/bin/bash
# Round-2 sweep: every BASELINE config on one GPU with the C-oracle parity block (cpu_baseline) and
# Recall@{1,10,100}; config 1 over L x k.  One JSON line per run into gpurun_out/${tag}.jsonl.
tag=${1:-sweep_r2}
out=gpurun_out/${tag}.jsonl
mkdir -p gpurun_out
: > $out
run() { timeout 1500 python bench.py --steps 5 --warmup 3 "$@" 2>>gpurun_out/${tag}.err | tail -1 >> $out; }
run --config c0
run --config c0 --engine baseline
for L in 1000 10000 100000; do for k in 1 10 100; do run --config c1 --L $L --k $k --recall-queries 0 --no-cpu-baseline; done; done
run --config c1
run --config c1 --engine baseline
run --config c1 --exact
run --config c2
run --config c3
run --config c4
run --config c4m16
