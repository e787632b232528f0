#!/bin/bash
# the doublings sketched behind the chunked upload: tests, then C4 / C3 / C5 e2e with and without them
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_path.py -q -x -p no:cacheprovider -k "upload" > gpurun_out/spec_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/spec_tests.log
for c in ${CONFIGS:-c4 c3 c5}; do
  for dep in 5 0; do
    IHS_UPLOAD_SPEC_DEPTH=$dep timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/spec_${c}_d$dep.json 2> gpurun_out/spec_${c}_d$dep.err
    echo "$c depth $dep rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/spec_${c}_d$dep.json'));print(d['ms_per_step'],d['e2e'],d['solve']['delta_rel_vs_direct'])"
  done
done
