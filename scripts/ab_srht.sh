#!/bin/bash
# A/B of the SRHT paths: parity tests and c1/c3 benches with the two-kernel
# path (default) and a single-launch variant selected by $VAR (default
# IHS_SRHT_FUSED; IHS_SRHT_COOP selects the cooperative kernel).
VAR=${VAR:-IHS_SRHT_FUSED}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/gpu_tests.log
env $VAR=1 timeout 600 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests_fused.log 2>&1
echo "pytest fused exit $?"; tail -2 gpurun_out/gpu_tests_fused.log
for c in ${CONFIGS:-c1 c3}; do
  for f in 0 1; do
    env $VAR=$f timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$f.json 2> gpurun_out/ab_${c}_$f.err
    echo "bench $c fused=$f exit $?"
    python - "$c" "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(d["ms_per_step"], d["roofline"]["phase_ms"])
except Exception as e:
    print("no result", e)
PY
  done
done
