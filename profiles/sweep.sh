#!/bin/bash
# Parameter sweep over BASELINE configs[1] (L x k, engines) and configs[0]/[2];
# one JSON line per run into gpurun_out/sweep.jsonl (run on the GPU box).
cd "$(dirname "$0")/.."
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" 2>>gpurun_out/sweep.err | tail -1 >> $out; }
run --config c0
run --config c0 --engine baseline
for L in 1000 10000 100000; do for k in 1 10 100; do run --config c1 --L $L --k $k; done; done
run --config c1 --engine baseline
run --config c2
run --config c3
run --config c4
