#!/bin/bash
# per-launch device times (cold-cache, serialised) for one config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${CFG:-c2}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-0} -c ${COUNT:-3000} --csv \
    --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_$CFG.log 2>&1
echo "exit $?"
