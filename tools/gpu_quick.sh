#!/bin/bash
# quick A/B: large-cell tests + c4 / c1 bench lines (no CPU baseline)
tag=${1:-quick}
o=gpurun_out
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "large_cells or adversarial or scale_sparse or c0_vs_reference" > $o/${tag}_tests.log 2>&1; tail -2 $o/${tag}_tests.log
for cfg in ${CFGS:-c4 c1}; do
  timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 --no-cpu-baseline > $o/${tag}_$cfg.json 2> $o/${tag}_$cfg.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/${tag}_$cfg.json").read().strip().splitlines()[-1])
    print("$cfg", round(d["value"]), {k:round(v,3) for k,v in d["stage_ms"].items()}, round(d["roofline"]["frac"],3))
except Exception as e:
    print("$cfg ERR", e, open("$o/${tag}_$cfg.err").read()[-400:])
PY
done
