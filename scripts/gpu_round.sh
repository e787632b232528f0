#!/bin/bash
# One GPU call: parity tests, smoke, then short benches of several configs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
for c in ${CONFIGS:-c1 c2 c3}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 ${BENCH_FLAGS} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c exit $?"; tail -c 600 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
