#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_case.py: config-0 searches,
# sparse tables with partial sort / extension / retry, the large-cell stream kernels (register-pipelined default
# and the TMA ring), a tie plateau.  Logs -> gpurun_out/<tag>_<tool>.log
tag=${1:-san}
o=gpurun_out
mkdir -p $o
timeout 600 python tools/sanitize_case.py > $o/${tag}_plain.log 2>&1 || { echo "plain run failed"; tail -5 $o/${tag}_plain.log; exit 1; }
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > $o/${tag}_$tool.log 2>&1
  echo "rc=$?" >> $o/${tag}_$tool.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=" $o/${tag}_$tool.log | tail -3
done
BPQ_STREAM_TMA=1 timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_case.py > $o/${tag}_racecheck_tma.log 2>&1
echo "rc=$?" >> $o/${tag}_racecheck_tma.log
grep -E "RACECHECK SUMMARY|rc=" $o/${tag}_racecheck_tma.log | tail -2
