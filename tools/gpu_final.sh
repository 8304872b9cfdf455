#!/bin/bash
# Final round-2 pass: GPU tests, smoke, default bench (both arms), c4 bench, launch lists filtered to the
# search-step kernels, the row_cut A/B.
tag=${1:-fin}
o=gpurun_out; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $o/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $o/${tag}_tests.log
tail -4 $o/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> $o/${tag}_smoke.log
timeout 900 python bench.py > $o/${tag}_c1.json 2> $o/${tag}_c1.err; echo "bench rc=$?" >> $o/${tag}_c1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/${tag}_ref.json 2> $o/${tag}_ref.err; echo "ref rc=$?" >> $o/${tag}_ref.err
timeout 1500 python bench.py --config c4 --steps 10 > $o/${tag}_c4.json 2> $o/${tag}_c4.err
KN='regex:coarse_dots|row_topk|row_cut|row_sort|fold_kernel|search_kernel|cell_flow|big_scan'
for cfg in c1 c4; do
  B="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
  timeout 900 $B > $o/${tag}_${cfg}_plain.json 2> $o/${tag}_${cfg}_plain.err &&
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KN" -c 80 --csv --log-file $o/${tag}_${cfg}_launches.csv $B > $o/${tag}_${cfg}_launches.log 2>&1
done
for cfg in c1 c4; do
  B="python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:cell_flow -s 3 -c 1 -o $o/${tag}_${cfg}_flow $B > $o/${tag}_${cfg}_flow_ncu.log 2>&1
done
BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0 --phase-profile > $o/${tag}_c4_prof.json 2> $o/${tag}_c4_prof.err
BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0 --phase-profile > $o/${tag}_c1_prof.json 2> $o/${tag}_c1_prof.err
for f in c1 c4; do python - <<PY
import json
d=json.loads(open("$o/${tag}_$f.json").read().strip().splitlines()[-1])
print("$f", round(d["value"]), round(d["e2e"]["value"]), {k:round(v,3) for k,v in d["stage_ms"].items()}, round(d["roofline"]["frac"],3), d.get("parity",{}).get("unclassified"))
PY
done
