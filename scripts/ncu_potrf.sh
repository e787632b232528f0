#!/bin/bash
# ncu --set full of the diagonal-block Cholesky kernel inside C1 (warm cache), with source
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --cache-control none --clock-control none --import-source on -k "regex:potrf_diag" \
  -s 40 -c 2 -o gpurun_out/prof_potrf python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_potrf.log 2>&1; echo "rc=$?"
