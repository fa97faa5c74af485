#!/bin/bash
# One gpurun call: GPU parity tests, benches per config, ncu launch lists + full captures.
# usage (under gpurun): bash scripts/gpu_round.sh TAG [stages...]
#   stages: build tests smoke bench benchfast ncu_launch ncu_full_c2 ncu_full_c3 ncu_full_c4 ncu_full_c5 ncu_gram_c4
set -u
TAG=${1:-run}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
STAGES=${@:-build tests bench}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> $OUT/nproc.txt
for s in $STAGES; do
  case $s in
    build) python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -20 $OUT/build.log; exit 1; } ;;
    tests) timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.txt ;;
    bench) timeout 600 python bench.py > $OUT/bench_c2.jsonl 2> $OUT/bench_c2.err; echo "bench c2 rc=$?"
           for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 10 > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; echo "bench $c rc=$?"; done ;;
    parity_full) rm -f $OUT/full_parity.jsonl; SNN_PARITY_RECORD=$OUT/full_parity.jsonl timeout 1200 python -m pytest tests/test_full_parity.py -m gpu -v > $OUT/pytest_full_parity.txt 2>&1; echo "parity_full rc=$?"; tail -8 $OUT/pytest_full_parity.txt ;;
    benchfast) for c in c2 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 10 --no-cpu-baseline > $OUT/bench_$c.jsonl 2> $OUT/bench_$c.err; echo "bench $c rc=$?"; done ;;
    reference) timeout 600 python bench.py --impl reference --steps 3 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err; echo "reference rc=$?" ;;
    ablation) timeout 900 python scripts/ablation_pruning.py c2 c3 c4 > $OUT/ablation_pruning.jsonl 2> $OUT/ablation.err; echo "ablation rc=$?"; cat $OUT/ablation_pruning.jsonl ;;
    ncu_launch) for c in c2 c3 c4 c5; do
        CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
        $CMD > $OUT/plain_$c.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1; echo "ncu launch $c rc=$?"; done ;;
    ncu_full_*) c=${s#ncu_full_}
        case $c in c2) K='regex:window_lowd';; c5) K='regex:union_snap';; *) K='regex:tc_window';; esac
        CMD="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline"
        $CMD > $OUT/plainf_$c.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k $K -s 6 -c 2 -o $OUT/full_$c $CMD > $OUT/ncu_full_$c.log 2>&1; echo "ncu full $c rc=$?" ;;
    ncu_dbscan_c5)
        CMD="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline"
        $CMD > $OUT/plaind_c5.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:core_count -s 3 -c 1 -o $OUT/core_c5 $CMD > $OUT/ncu_core_c5.log 2>&1; echo "ncu core c5 rc=$?"
        timeout 1200 ncu --set full --clock-control none --import-source on -k regex:union_snap -s 3 -c 1 -o $OUT/union_c5 $CMD > $OUT/ncu_union_c5.log 2>&1; echo "ncu union c5 rc=$?"
        timeout 1200 ncu --set full --clock-control none --import-source on -k regex:union_seed -s 3 -c 1 -o $OUT/seed_c5 $CMD > $OUT/ncu_seed_c5.log 2>&1; echo "ncu seed c5 rc=$?" ;;
    ncu_write_c2)
        CMD="python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline"
        $CMD > $OUT/plainw_c2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"compact_lowd_bal|rows_finalize" -s 8 -c 2 -o $OUT/write_c2 $CMD > $OUT/ncu_write_c2.log 2>&1; echo "ncu write c2 rc=$?" ;;
    ncu_gram_c4)
        CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline"
        $CMD > $OUT/plaing_c4.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gram_tc -s 3 -c 1 -o $OUT/gram_c4 $CMD > $OUT/ncu_gram_c4.log 2>&1; echo "ncu gram c4 rc=$?" ;;
    summarize)   # text summaries of every capture, then drop the .ncu-rep files (gpurun_out <= 64 MiB)
        for r in $OUT/*.ncu-rep; do [ -f "$r" ] || continue; b=${r%.ncu-rep}
            python scripts/ncu_summary.py full $r > ${b}_metrics.txt 2>&1
            python scripts/ncu_source.py $r 40 > ${b}_source_top40.txt 2>&1
            python scripts/ncu_lines.py $r 30 > ${b}_lines.txt 2>&1
            ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null; gzip -f ${b}_raw.csv
            rm -f $r; done
        for c in $OUT/launches_*.csv; do [ -f "$c" ] || continue; python scripts/ncu_summary.py launches $c > ${c%.csv}_summary.txt 2>&1; done
        du -sh $OUT ;;
  esac
done
