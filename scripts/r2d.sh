set -u
OUT=gpurun_out/r2d; mkdir -p $OUT
bash scripts/ab_run.sh r2d "c4:8:" "c4:8:gram_rows=-1" "c3:10:" "c2:20:" 
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.txt
