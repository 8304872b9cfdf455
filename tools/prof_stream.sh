#!/bin/bash
# GPU tests, then ncu --set full captures of the large-cell stream kernel and the traversal kernel at c1 and
# c4 (each command first exits 0 without ncu).
tag=${1:-prof}
mkdir -p gpurun_out
#timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for cfg in c1 c4; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_${cfg}.json 2> gpurun_out/${tag}_${cfg}.err &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:big_scan -s 1 -c 1 \
      -o gpurun_out/${tag}_${cfg} python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/${tag}_${cfg}_ncu.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/${tag}_${cfg}_ncu.log
done
# nb0 (first sparse-traversal batch) A/B at c4 and c1
timeout 600 python tools/ab_env.py --config c4 --var BPQ_NB0 --values 128 64 32 16 > gpurun_out/${tag}_nb0_c4.jsonl 2> gpurun_out/${tag}_nb0_c4.err
timeout 600 python tools/ab_env.py --config c1 --var BPQ_NB0 --values 128 64 32 16 > gpurun_out/${tag}_nb0_c1.jsonl 2> gpurun_out/${tag}_nb0_c1.err
