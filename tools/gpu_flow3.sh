#!/bin/bash
tag=${1:-flow3}
o=gpurun_out
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $o/${tag}_tests.log
tail -4 $o/${tag}_tests.log
for cfg in c1 c4; do
  timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 > $o/${tag}_$cfg.json 2> $o/${tag}_$cfg.err; echo "rc=$?" >> $o/${tag}_$cfg.err
  BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0 --phase-profile > $o/${tag}_${cfg}_prof.json 2> $o/${tag}_${cfg}_prof.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/${tag}_$cfg.json").read().strip().splitlines()[-1])
    print("$cfg", d["value"], d["stage_ms"], d["roofline"]["frac"], {k:d["parity"][k] for k in ("exact_lists","near_tie_distance","near_tie_boundary","unclassified")} if "parity" in d else None)
    d=json.loads(open("$o/${tag}_${cfg}_prof.json").read().strip().splitlines()[-1])
    print("   prof", d["phase_profile"]["stream_kernel_share"], d["phase_profile"]["traversal_kernel_share"])
except Exception as e:
    print("$cfg ERR", e)
PY
done
