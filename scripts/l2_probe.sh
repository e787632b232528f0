#!/bin/bash
# Timing probes of the L2-resident SRHT launch at the C4 shape (d reduced): IHS_SRHT_L2_DBG 0 normal, 1 emitting
# side idle, 2 no phase-1 transform, 3 no phase-1 store, 4 neither (wrong results; timing only)
for dbg in ${DBGS:-0 1 2 3 4 5}; do
  echo "dbg=$dbg"
  IHS_SRHT_L2_DBG=$dbg timeout -s KILL 300 python scripts/sketch_bench.py --config c4 --d ${D:-512} --ms 8192,131072 --reps 3
done
