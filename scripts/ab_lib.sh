# A/B of two in-tree builds on config 2: lib/libsnn_base.so vs lib/libsnn.so (SNN_LIB), extra bench args in "$@"
for i in 1 2; do
for L in libsnn_base.so libsnn.so; do
SNN_LIB=paper_2212_07679_b200/lib/$L timeout 300 python bench.py --config c2 --steps 20 --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=l['breakdown_ms_per_step']
print('$L', round(l['ms_per_step'],3), 'K8', round(b['window_count'],3), 'write', round(b['window_write'],3))"
done; done
