python scripts/pipe_probe3.py > gpurun_out/r2k_probe.txt 2>&1; cat gpurun_out/r2k_probe.txt
python scripts/pipe_probe2.py > gpurun_out/r2k_probe2.txt 2>&1; tail -9 gpurun_out/r2k_probe2.txt
bash scripts/ab_run.sh r2k "c2:20:" "c3:10:" "c4:8:" "c1:20:"
