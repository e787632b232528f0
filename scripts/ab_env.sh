#!/bin/bash
# Generic A/B: bench configs $CONFIGS with env $VAR set to each of $VALS (empty = unset), device step only.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${CONFIGS:-c1 c2}; do
  for v in ${VALS:-x}; do
    if [ "$v" = "x" ]; then E=""; else E="$VAR=$v"; fi
    env $E timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    python - "$c" "$v" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d["ms_per_step"], 3), {k: round(v, 3) for k, v in d["roofline"]["phase_ms"].items()})
except Exception as e:
    print("no result", e)
PY
  done
done
