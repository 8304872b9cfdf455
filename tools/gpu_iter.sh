#!/bin/bash
# Development iteration on the GPU box: GPU tests, then bench lines for the configs given.
# usage: tools/gpu_iter.sh TAG "bench args 1" "bench args 2" ...
tag=$1; shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
i=0
for a in "$@"; do
  timeout 900 python bench.py $a > gpurun_out/${tag}_b$i.json 2> gpurun_out/${tag}_b$i.err; echo "rc=$? args=$a" >> gpurun_out/${tag}_b$i.err
  i=$((i+1))
done
tail -3 gpurun_out/${tag}_tests.log
