#!/bin/bash
# ncu --set full of the C4 sketch kernels (SRHT phase 1 + two-round emitting pass at n = 2^22, m = 131072) and of
# the gradient pass, on C4's row count with fewer columns (the full 64 GiB problem does not fit ncu's
# save/restore replay); per-launch behaviour is per column, so throughput and traffic per byte carry over.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k "regex:srht_phase1_tma|srht_phase2_r2" \
  -c 2 -o gpurun_out/prof_c4_srht python scripts/sketch_bench.py --config c4 --d 128 --ms 131072 --reps 0 \
  > gpurun_out/ncu_c4s.log 2>&1; echo "srht rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k "regex:grad_rr_kernel" -s 2 -c 1 \
  -o gpurun_out/prof_c4_grad python scripts/grad_bench.py --n 524288 --d 2048 --reps 4 > gpurun_out/ncu_c4g.log 2>&1; echo "grad rc=$?"
