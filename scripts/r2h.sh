python scripts/pipe_probe2.py > gpurun_out/r2h_probe.txt 2>&1; cat gpurun_out/r2h_probe.txt
