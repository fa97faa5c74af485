for v in "" "SNN_BENCH_EXT_STREAMS=1" "SNN_BENCH_NOFLUSH=1" "SNN_BENCH_EXT_STREAMS=1 SNN_BENCH_NOFLUSH=1"; do
  env $v SNN_BENCH_TIMELINE=1 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/r2n.json 2> gpurun_out/r2n.err
  python -c "
import json; l=json.loads(open('gpurun_out/r2n.json').read().strip().splitlines()[-1]); print('$v', l['e2e']['ms_per_step'], l['e2e']['serial_ms_per_step'])"
  grep "^step" gpurun_out/r2n.err | tail -5
done
