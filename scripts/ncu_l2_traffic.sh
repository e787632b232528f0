#!/bin/bash
# DRAM bytes and L2 write requests per SRHT launch at a config's full size, largest and smallest m of its solve
# (application replay: the matrix is regenerated per pass, no save/restore of the 8-64 GB problem)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CFG=${CFG:-c3}; MS=${MS:-65536,2048}
python scripts/sketch_bench.py --config $CFG --ms $MS --reps 2 > gpurun_out/sketch_${CFG}_plain.log 2>&1; echo "plain rc=$?"
timeout -s KILL 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_requests_srcunit_tex_op_write.sum \
  --replay-mode application --clock-control none -k "regex:srht_" --csv --log-file gpurun_out/ncu_l2_${CFG}full.csv \
  python scripts/sketch_bench.py --config $CFG --ms $MS --reps 0 > gpurun_out/ncu_l2_${CFG}full.log 2>&1; echo "ncu rc=$?"
