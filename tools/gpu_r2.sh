#!/bin/bash
# tests, c1 + c4 bench lines, nb0 A/B
tag=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
timeout 900 python bench.py --steps 10 > gpurun_out/${tag}_c1.json 2> gpurun_out/${tag}_c1.err
timeout 900 python bench.py --config c4 --steps 5 --no-cpu-baseline > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err
timeout 600 python tools/ab_env.py --config c4 --var BPQ_NB0 --values 128 64 32 16 > gpurun_out/${tag}_nb0_c4.jsonl 2> gpurun_out/${tag}_nb0_c4.err
timeout 600 python tools/ab_env.py --config c1 --var BPQ_NB0 --values 128 64 32 16 > gpurun_out/${tag}_nb0_c1.jsonl 2> gpurun_out/${tag}_nb0_c1.err
