#!/bin/bash
# One B200 pass over every BASELINE config: bench line per config (recording the solve counters the reference arm
# extrapolates with), the reference arm on the default config, then the GPU test suite. Output in gpurun_out/.
set -u
mkdir -p gpurun_out
for c in ${CONFIGS:-c4 c3 c5 c1 c2 c4g}; do
  steps=5; [ "$c" = c4g ] && steps=2
  timeout 1200 python bench.py --config $c --record-counters --steps $steps --warmup 3 --out gpurun_out/b_$c.json \
    > gpurun_out/b_$c.log 2>&1
  echo "$c rc=$?"
done
cp profiles/ref_counters.json gpurun_out/ref_counters.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err
echo "ref rc=$?"
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest.log
fi
