#!/bin/bash
# Round-2 evidence refresh: C4 and C2 launch lists (ncu gpu__time_duration, cold cache, serialised) and one
# `ncu --set full` capture of C2's S*A DMMA GEMM (scripts/sketch_bench.py at the C2 shape).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in c4 c2; do
  timeout -s KILL 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline \
    --no-e2e --no-clocks --no-delta > gpurun_out/ncu_${c}l.log 2>&1; echo "launches $c rc=$?"
done
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:dgemm_big" -c 1 \
  -o gpurun_out/prof_sa_c2 python scripts/sketch_bench.py --config c2 --kind gaussian --ms 1024 --reps 0 \
  > gpurun_out/ncu_sa.log 2>&1; echo "sa rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('__SMOKE_OK__')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
