python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k9_build.log 2>&1 || { tail -20 gpurun_out/k9_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tc or c3 or c4 or tensor or random_parity" > gpurun_out/k9_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/k9_pytest.txt
SNN_PARITY_RECORD=gpurun_out/k9_parity.jsonl timeout 900 python -m pytest tests/test_full_parity.py -m gpu -q -k "c3 or c4" > gpurun_out/k9_parity.txt 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/k9_parity.txt
bash scripts/ab_run.sh k9 "c3:10:" "c4:8:" "c3:10:tc_tiles=16"
