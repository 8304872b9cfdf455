#!/bin/bash
# Round-2 final evidence: compute-sanitizer logs, the all-config sweep (parity block + recall per line), ncu
# launch list and --set full captures of the stream kernel (c1, c4), c2 phase profile (residual-table bytes).
tag=${1:-r2n}
o=gpurun_out; mkdir -p $o
bash tools/gpu_sanitize.sh ${tag}_san
bash tools/sweep_r2.sh ${tag}_sweep
BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 python bench.py --config c2 --steps 3 --no-cpu-baseline --recall-queries 0 --phase-profile > $o/${tag}_c2prof.json 2> $o/${tag}_c2prof.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 $B > $o/${tag}_c1_plain.json 2> $o/${tag}_c1_plain.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_c1_launches.csv $B > $o/${tag}_c1_launches.log 2>&1
timeout 600 $B --config c4 > $o/${tag}_c4_plain.json 2> $o/${tag}_c4_plain.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_c4_launches.csv $B --config c4 > $o/${tag}_c4_launches.log 2>&1
for cfg in c1 c4; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cell_flow -s 3 -c 1 -o $o/${tag}_${cfg}_flow $B --config $cfg > $o/${tag}_${cfg}_flow_ncu.log 2>&1
done
