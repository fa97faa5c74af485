SNN_BENCH_TIMELINE=1 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/r2m.json 2> gpurun_out/r2m.err; tail -16 gpurun_out/r2m.err
