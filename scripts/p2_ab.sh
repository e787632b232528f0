#!/bin/bash
# phase-2 tile width A/B: launch lists of the SRHT sketch harness per IHS_SRHT_P2T
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for t in ${P2TS:-256 512}; do
  IHS_SRHT_P2T=$t python scripts/time_sketch.py --ms ${MS:-64,2048} --reps 2 > gpurun_out/p2_$t.log 2>&1 && \
  IHS_SRHT_P2T=$t ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_p2_$t.csv \
      python scripts/time_sketch.py --ms ${MS:-64,2048} --reps 2 > /dev/null 2>&1
  echo "p2t $t exit $?"
done
