#!/bin/bash
# ncu --set full of the L2-resident SRHT launch on C4's rows with d = 256 (the full 64 GiB problem does not fit the
# replay buffer), m = 8192; then the same under IHS_SRHT_L2_DBG=4 (phase 1 without transform/store: emitting side)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for dbg in ${DBGS:-0 4}; do
IHS_SRHT_L2_DBG=$dbg timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:srht_l2_kernel" \
  -s 1 -c 1 -o gpurun_out/prof_l2_dbg$dbg python scripts/sketch_bench.py --config c4 --d 256 --ms 8192 --reps 1 \
  > gpurun_out/ncu_l2_dbg$dbg.log 2>&1; echo "dbg $dbg rc=$?"
done
