#!/bin/bash
# Round-end evidence in one GPU call: every config's bench line + the reference arm (scripts/bench_all.sh), then the
# C2 / C1 launch lists (ncu, cold cache, serialised) and the GPU test suite.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TESTS=0 bash scripts/bench_all.sh
for c in c2 c1; do CFG=$c COUNT=2000 bash scripts/ncu_launches.sh; done
timeout -s KILL 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputest_final.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
