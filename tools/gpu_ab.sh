#!/bin/bash
# A/B one environment variable over values: tools/gpu_ab.sh TAG VAR "v1 v2 ..." "cfg1 cfg2"
tag=$1; var=$2; vals=$3; cfgs=${4:-"c4 c1"}
o=gpurun_out; mkdir -p $o
for cfg in $cfgs; do for v in $vals; do
  env $var=$v timeout 900 python bench.py --config $cfg --steps 10 --recall-queries 0 --no-cpu-baseline > $o/${tag}_${cfg}_$v.json 2> $o/${tag}_${cfg}_$v.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/${tag}_${cfg}_$v.json").read().strip().splitlines()[-1])
    print("$cfg $var=$v", round(d["value"]), {k:round(x,3) for k,x in d["stage_ms"].items()}, round(d["roofline"]["frac"],3))
except Exception as e:
    print("$cfg $v ERR", e)
PY
done; done
