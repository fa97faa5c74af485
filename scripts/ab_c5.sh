set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -20 $OUT/build.log; exit 1; }
for u in 0 1 2; do timeout 300 python bench.py --config c5 --steps 8 --no-cpu-baseline --opt union_load=$u > $OUT/c5_u$u.jsonl 2>$OUT/c5_u$u.err; echo "c5 u$u rc=$?"; done
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_full_parity.py::test_full_size_every_row_matches_oracle > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu.txt
