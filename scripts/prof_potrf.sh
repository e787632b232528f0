#!/bin/bash
# One ncu --set full capture of the diagonal-block Cholesky kernel on C1 (the factor-bound config).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CMD="python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
$CMD > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:potrf_diag|tri_inv64" -s 40 -c 4 \
    -o gpurun_out/prof_potrf $CMD > gpurun_out/ncu_potrf.log 2>&1
echo "exit $?"
