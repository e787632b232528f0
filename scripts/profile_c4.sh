#!/bin/bash
# C4 evidence: per-launch device times of one solve (ncu launch list, cold cache, serialised) and one
# `ncu --set full` capture of each dominant kernel (SRHT phase 1, the two-round emitting pass, the gradient pass).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --no-delta"
timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4.csv $CMD > gpurun_out/ncu_c4l.log 2>&1; echo "launches rc=$?"
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on \
  -k "regex:srht_phase1_tma|srht_phase2_r2|grad_rr_kernel" -s 30 -c 3 \
  -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4f.log 2>&1; echo "full rc=$?"
