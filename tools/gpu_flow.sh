#!/bin/bash
# A/B of the large-cell stream kernels: GPU tests, then c1 / c4 / c4m16 bench lines (parity block included)
# with the default (cell_flow_kernel) and with BPQ_STREAM_TMA=1 (TMA-ring big_scan_kernel).
tag=${1:-flow}
o=gpurun_out
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $o/${tag}_tests.log
tail -5 $o/${tag}_tests.log
for cfg in c1 c4 c4m16 c3; do
  timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 > $o/${tag}_$cfg.json 2> $o/${tag}_$cfg.err; echo "rc=$?" >> $o/${tag}_$cfg.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/${tag}_$cfg.json").read().strip().splitlines()[-1])
    print("$cfg", d["value"], d["stage_ms"], d["roofline"]["frac"], {k:d["parity"][k] for k in ("exact_lists","near_tie_distance","near_tie_boundary","unclassified")} if "parity" in d else None)
except Exception as e:
    print("$cfg ERR", e)
PY
done
for cfg in c1 c4; do
  BPQ_STREAM_TMA=1 timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 --no-cpu-baseline > $o/${tag}_${cfg}_tma.json 2> $o/${tag}_${cfg}_tma.err
done
