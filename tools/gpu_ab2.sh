#!/bin/bash
# A/B of the stream kernel's CTA variants over configs, with the roll-back count of one batch
o=gpurun_out; mkdir -p $o
run() { # cfg extra-args var val
  env $3=$4 timeout 900 python bench.py --config $1 $2 --steps 8 --recall-queries 0 --no-cpu-baseline > $o/ab2.json 2> $o/ab2.err
  python - <<PY
import json,re
try:
    d=json.loads(open("$o/ab2.json").read().strip().splitlines()[-1])
    m=re.search(r"roll-backs (\d+)", open("$o/ab2.err").read())
    print("$1 $2 $3=$4", round(d["value"]), {k:round(x,3) for k,x in d["stage_ms"].items()}, round(d["roofline"]["frac"],3), "rollbacks", m.group(1) if m else None)
except Exception as e:
    print("$1 $2 $4 ERR", e)
PY
}
for c in "c1|" "c1|--L 100000" "c1|--L 1000" "c4|" "c3|" "c4m16|"; do
  cfg=${c%%|*}; ex=${c#*|}
  for v in 2 3; do run $cfg "$ex" BPQ_FLOW_CTAS $v; done
done
