set -u
OUT=gpurun_out/ab1; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -k "finalize or row_staging or everything or partition or symmetric or concurrent" > $OUT/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.txt
for i in 1 2 3; do for fp in 0 -1; do
  timeout 300 python bench.py --config c2 --steps 30 --no-cpu-baseline --opt finalize_pipe=$fp > $OUT/c2_fp${fp}_$i.jsonl 2>/dev/null
  python -c "
import json; l=json.loads(open('$OUT/c2_fp${fp}_$i.jsonl').read().strip().splitlines()[-1]); b=l['breakdown_ms_per_step']
print('fp=$fp', round(l['ms_per_step'],3), 'write', round(b['window_write'],3), 'scan', round(b['window_count'],3))"
done; done
