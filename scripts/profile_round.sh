#!/bin/bash
# Evidence for one config: full bench line (cpu baseline + e2e), the ncu launch
# list of the same bench command, and one `ncu --set full` capture of the
# kernels matching KREGEX (each ncu pass only after the plain run exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${CFG:-c2}
timeout 900 python bench.py --config $CFG --steps ${STEPS:-5} --warmup 3 ${BENCH_FLAGS} > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
echo "bench exit $?"; tail -c 400 gpurun_out/bench_$CFG.json
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD \
    > gpurun_out/ncu_$CFG.log 2>&1
echo "launch list exit $?"
if [ -n "$KREGEX" ]; then
  ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s ${SKIP:-0} -c ${COUNT:-3} \
      -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
  echo "full capture exit $?"
fi
