#!/bin/bash
# row_cut_kernel validation: full GPU test suite, then c1 / c4 / c3 bench lines with the parity block, and
# the A/B against the round-1 histogram kernel (BPQ_ROW_TOPK_OLD=1)
tag=${1:-rowcut}
o=gpurun_out; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $o/${tag}_tests.log
tail -4 $o/${tag}_tests.log
for cfg in c1 c4 c3; do
  timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 > $o/${tag}_$cfg.json 2> $o/${tag}_$cfg.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/${tag}_$cfg.json").read().strip().splitlines()[-1])
    print("$cfg", round(d["value"]), {k:round(v,3) for k,v in d["stage_ms"].items()}, round(d["roofline"]["frac"],3), {k:d["parity"][k] for k in ("exact_lists","near_tie_distance","near_tie_boundary","unclassified")} if "parity" in d else None)
except Exception as e:
    print("$cfg ERR", e, open("$o/${tag}_$cfg.err").read()[-600:])
PY
done
bash tools/gpu_ab.sh ${tag}_ab BPQ_ROW_TOPK_OLD "1" "c1 c4"
