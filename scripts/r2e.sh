bash scripts/ab_run.sh r2e "c2:20:" "c3:10:tc_tiles=4" "c3:10:tc_tiles=16" "c3:10:tc_tiles=32" "c3:10:tc_group=32" "c5:8:union_load=1" "c5:8:union_load=0"
