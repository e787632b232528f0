#!/bin/bash
# one ncu --set full capture of the top kernels of a config (single GPU)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${CFG:-c3}
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks"
$CMD > gpurun_out/plain_full_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-grad_smem|srht_phase}" -s ${SKIP:-20} -c ${COUNT:-4} \
    -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "exit $?"
