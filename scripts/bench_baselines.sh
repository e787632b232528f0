#!/bin/bash
# CG / PCG comparators (bench.py --solver) on the BASELINE configs' data, plus their GPU parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_baselines.py -q -p no:cacheprovider > gpurun_out/gb.log 2>&1
echo "baselines pytest exit $?"; tail -1 gpurun_out/gb.log
for sc in ${RUNS:-"pcg c1" "pcg c2" "pcg c3" "cg c1" "cg c2" "cg c3"}; do
  set -- $sc
  timeout 900 python bench.py --solver $1 --config $2 --steps 3 --warmup 3 --no-e2e > gpurun_out/bb_$1_$2.json 2> gpurun_out/bb_$1_$2.err
  echo "bench $1 $2 exit $?"
  python - "$1" "$2" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/bb_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(" ms/step %.3f" % d["ms_per_step"], "solve", {k: v for k, v in d["solve"].items() if k != "step_ms"})
    print(" phases", r.get("phase_ms"), "dominant", r.get("dominant"), "frac %.3f" % (r.get("frac") or 0))
    print(" cpu", d["cpu_baseline"])
except Exception as e:
    print("no result", e)
PY
done
