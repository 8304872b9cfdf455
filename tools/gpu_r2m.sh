#!/bin/bash
# Round-2 evidence pass: GPU tests + smoke, c1 bench (both arms), c1 ncu launch list, ncu --set full captures
# of the stream / traversal / first-layer kernels at c1 and of the stream kernel at c4 (every ncu command
# runs only after the same command exited 0 without ncu), c4 bench with the C-oracle parity sample and the
# phase profile of the stream kernel.
tag=${1:-r2m}
o=gpurun_out
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $o/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $o/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> $o/${tag}_smoke.log
timeout 900 python bench.py > $o/${tag}_c1.json 2> $o/${tag}_c1.err; echo "bench rc=$?" >> $o/${tag}_c1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/${tag}_ref.json 2> $o/${tag}_ref.err; echo "ref rc=$?" >> $o/${tag}_ref.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
timeout 600 $B > $o/${tag}_c1_plain.json 2> $o/${tag}_c1_plain.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_c1_launches.csv \
    $B > $o/${tag}_c1_launches.log 2>&1
for kn in big_scan search_kernel coarse_dots_tc row_topk; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kn -s 3 -c 1 -o $o/${tag}_c1_$kn \
      $B > $o/${tag}_c1_${kn}_ncu.log 2>&1
  echo "ncu rc=$?" >> $o/${tag}_c1_${kn}_ncu.log
done
timeout 1500 python bench.py --config c4 --steps 5 --warmup 3 > $o/${tag}_c4.json 2> $o/${tag}_c4.err; echo "bench rc=$?" >> $o/${tag}_c4.err
B4="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0"
BPQ_LIB=$PWD/paper_1404_1831_b200/libbpq_b200_prof.so timeout 900 $B4 --phase-profile > $o/${tag}_c4prof.json 2> $o/${tag}_c4prof.err
for kn in big_scan search_kernel row_topk; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kn -s 3 -c 1 -o $o/${tag}_c4_$kn \
      $B4 > $o/${tag}_c4_${kn}_ncu.log 2>&1
  echo "ncu rc=$?" >> $o/${tag}_c4_${kn}_ncu.log
done
tail -3 $o/${tag}_tests.log
