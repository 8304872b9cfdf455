#!/bin/bash
tag=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 python bench.py --config c4 --steps 2 --no-cpu-baseline --recall-queries 0 --phase-profile > gpurun_out/${tag}_c4prof.json 2> gpurun_out/${tag}_c4prof.err
timeout 900 python bench.py --steps 10 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_c1.json 2> gpurun_out/${tag}_c1.err
timeout 900 python bench.py --config c4 --steps 5 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_c4.json 2> gpurun_out/${tag}_c4.err
