python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python scripts/union_check.py union_snap=-1 union_snap=1 union_snap=3 union_snap=1 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:union_snap -s 1 -c 1 -o gpurun_out/union_snap python scripts/union_check.py union_snap=1 > gpurun_out/ncu_union.log 2>&1; echo ncu rc=$?
python scripts/ncu_summary.py full gpurun_out/union_snap.ncu-rep > gpurun_out/union_snap_metrics.txt 2>&1
python scripts/ncu_source.py gpurun_out/union_snap.ncu-rep 40 > gpurun_out/union_snap_source.txt 2>&1
ncu -i gpurun_out/union_snap.ncu-rep --page raw --csv > gpurun_out/union_snap_raw.csv 2>/dev/null; gzip -f gpurun_out/union_snap_raw.csv; rm -f gpurun_out/union_snap.ncu-rep
