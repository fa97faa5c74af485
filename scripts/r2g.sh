python scripts/pipe_probe.py > gpurun_out/r2g_probe.txt 2>&1; cat gpurun_out/r2g_probe.txt
bash scripts/ab_run.sh r2g "c4:8:" "c4:8:" "c4:8:gram_rows=-1"
