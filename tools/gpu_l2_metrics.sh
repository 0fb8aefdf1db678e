#!/bin/bash
# for the L2-resident configs (c1-c4) report L2 traffic and DRAM bytes per launch of the
# iteration kernels (ncu metrics pass, --clock-control none, cold-cache serialised launches).
OUT=gpurun_out/${1:-l2m}; mkdir -p $OUT
for c in c1 c2 c3 c4 c5; do
  timeout 300 python tools/prof_run.py $c 6 > /dev/null 2>&1 || { echo "$c plain run failed"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "regex:k_apply_s3|k_elem_pass_lanes|k_node_pass_lanes|k_cg_general_persistent" -c 12 --csv \
    python tools/prof_run.py $c 6 > $OUT/$c.csv 2>&1
done
python tools/l2_summary.py $OUT/c1.csv $OUT/c2.csv $OUT/c3.csv $OUT/c4.csv $OUT/c5.csv | tee $OUT/summary.txt
