#!/bin/bash
# Round-end evidence for the three single-GPU configs (bench line + launch list + one ncu --set full
# capture of the dominant kernels each), then the CG/PCG comparator lines. See profiles/README.md.
cd $GRAFT_REPO_ROOT
CFG=c2 KREGEX="grad_rr|dgemm_nn_big" COUNT=2 SKIP=10 bash scripts/profile_round.sh
CFG=c3 KREGEX="grad_rr|srht_phase" COUNT=3 SKIP=20 bash scripts/profile_round.sh
CFG=c1 KREGEX="grad_rr|srht_phase|potrf" COUNT=3 SKIP=20 bash scripts/profile_round.sh
RUNS="${BASELINE_RUNS:-pcg c2|pcg c3}" 
IFS='|' read -ra R <<< "$RUNS"
for sc in "${R[@]}"; do
  set -- $sc
  timeout 900 python bench.py --solver $1 --config $2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bb_$1_$2.json 2> gpurun_out/bb_$1_$2.err
  echo "bench $1 $2 exit $?"
done
