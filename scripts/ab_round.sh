#!/bin/bash
# One gpurun call: a pytest subset, then alternating A/B bench runs (no rebuild; the in-tree
# .so travels).  usage: bash scripts/ab_round.sh TAG "pytest -k expr" "cfg:steps:opts" ...
set -u
TAG=$1; shift; K=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.txt
fi
NOBUILD=1 bash scripts/ab_run.sh $TAG "$@"
