bash scripts/ab_run.sh r2c "c2:20:finalize_order=-1" "c2:20:finalize_order=1" "c2:20:finalize_order=-1" "c2:20:finalize_order=1" "c5:8:union_load=0" "c5:8:union_load=1"
OUT=gpurun_out/r2c
SNN_PARITY_RECORD=$OUT/full_parity.jsonl timeout 1200 python -m pytest tests/test_full_parity.py -m gpu -v > $OUT/pytest_full_parity.txt 2>&1; echo "parity_full rc=$?"; grep -E "PASS|FAIL" $OUT/pytest_full_parity.txt
CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"compact_lowd_bal|rows_finalize" -s 8 -c 2 -o $OUT/write_c2 $CMD > $OUT/ncu_write_c2.log 2>&1; echo "ncu write c2 rc=$?"
