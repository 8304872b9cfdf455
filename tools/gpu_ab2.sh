#!/bin/bash
o=gpurun_out; mkdir -p $o
run() { # cfg extra-args var val
  env $3=$4 timeout 900 python bench.py --config $1 $2 --steps 8 --recall-queries 0 --no-cpu-baseline > $o/ab2.json 2> $o/ab2.err
  python - <<PY
import json
try:
    d=json.loads(open("$o/ab2.json").read().strip().splitlines()[-1])
    print("$1 $2 $3=$4", round(d["value"]), {k:round(x,3) for k,x in d["stage_ms"].items()}, round(d["roofline"]["frac"],3))
except Exception as e:
    print("$1 $2 $4 ERR", e)
PY
}
for v in 2 3; do run c1 "--L 100000" BPQ_FLOW_CTAS $v; done
for v in 2 3; do run c1 "--L 1000" BPQ_FLOW_CTAS $v; done
for v in 2 3; do run c4m16 "" BPQ_FLOW_CTAS $v; done
for v in 2 3; do run c4 "--k 10" BPQ_FLOW_CTAS $v; done
