python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:window_lowd -s 6 -c 1 -o gpurun_out/k8 $CMD > gpurun_out/ncu_k8.log 2>&1; echo ncu rc=$?
python scripts/ncu_lines.py gpurun_out/k8.ncu-rep 30 > gpurun_out/k8_lines.txt 2>&1
python scripts/ncu_source.py gpurun_out/k8.ncu-rep 40 > gpurun_out/k8_source.txt 2>&1

