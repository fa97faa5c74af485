#!/bin/bash
# A/B runs under gpurun: bash scripts/ab_run.sh TAG "cfg:steps:opt1,opt2" ...   (opts as key=value)
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "${NOBUILD:-}" ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -20 $OUT/build.log; exit 1; }
for spec in "$@"; do
  IFS=: read cfg steps opts <<< "$spec"
  args=""; name="${cfg}"
  for o in ${opts//,/ }; do args="$args --opt $o"; name="${name}_${o}"; done
  timeout 300 python bench.py --config $cfg --steps $steps --no-cpu-baseline $args > $OUT/$name.jsonl 2>$OUT/$name.err
  python - "$OUT/$name.jsonl" "$name" <<'PY'
import json, sys
try:
    l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    b = l["breakdown_ms_per_step"]
    print(f"{sys.argv[2]:40s} step {l['ms_per_step']:.3f} ms  " + " ".join(f"{k}={v:.3f}" for k, v in b.items() if v) + f"  e2e {l['e2e']['ms_per_step']:.2f}  clk {l['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
done
