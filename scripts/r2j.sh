python scripts/pipe_probe3.py > gpurun_out/r2j_probe.txt 2>&1; cat gpurun_out/r2j_probe.txt
