#!/bin/bash
# ncu --set full capture of the two-queries-per-thread K8 scan (option scan2q) on config 2.
# usage (under gpurun): bash scripts/ncu_k8_2q.sh TAG [chunk]
set -u
TAG=${1:-k82q}; CH=${2:-512}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --opt scan2q=1 --opt chunk=$CH"
$CMD > $OUT/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:window_lowd_2q -s 2 -c 1 -o $OUT/k82q $CMD > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
r=$OUT/k82q.ncu-rep
python scripts/ncu_summary.py full $r > $OUT/k82q_metrics.txt 2>&1
python scripts/ncu_lines.py $r 30 > $OUT/k82q_lines.txt 2>&1
ncu -i $r --page raw --csv > $OUT/k82q_raw.csv 2>/dev/null; gzip -f $OUT/k82q_raw.csv
rm -f $r
