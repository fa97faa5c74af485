bash scripts/ab_run.sh r2l "c2:20:" "c3:10:" "c4:8:" "c1:20:"
