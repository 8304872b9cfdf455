#!/bin/bash
# Round-2 baseline session: GPU tests, smoke, c1 bench (parity + CPU baseline), reference arm, c1 launch list.
tag=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_c1.json 2> gpurun_out/${tag}_c1.err; echo "bench rc=$?" >> gpurun_out/${tag}_c1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc=$?" >> gpurun_out/${tag}_ref.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_c1short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_c1_launches.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --recall-queries 0 > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${tag}_ncu.log
tail -3 gpurun_out/${tag}_tests.log
