#!/bin/bash
# per-kernel device times of the streamed SRHT kernel under the timing-experiment modes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/time_sketch.py --ms ${MS:-2,2048} --reps 2"
for dbg in ${MODES:-0 1 3}; do
  IHS_SRHT_FUSED=${FUSED:-1} IHS_SRHT_STREAM_DBG=$dbg $CMD > gpurun_out/ts_dbg$dbg.log 2>&1 && \
  IHS_SRHT_FUSED=${FUSED:-1} IHS_SRHT_STREAM_DBG=$dbg ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_dbg$dbg.csv $CMD > /dev/null 2>&1
  echo "mode $dbg exit $?"; tail -4 gpurun_out/ts_dbg$dbg.log
done
