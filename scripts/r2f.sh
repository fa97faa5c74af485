bash scripts/ab_run.sh r2f "c2:20:" "c5:8:union_load=3" "c5:8:union_load=1" "c1:20:" "c3:10:" "c4:8:"
