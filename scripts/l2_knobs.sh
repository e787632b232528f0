#!/bin/bash
# A/B of the L2-resident SRHT launch's knobs at C4's row count (d = $D, default 512): each argument is one env
# setting, e.g.  bash scripts/l2_knobs.sh "" "IHS_SRHT_L2_TS=0" "IHS_SRHT_L2_NS=2"
# CHECK=1 first verifies bit-exactness of each setting against the oracle (scripts/l2_check.py).
# Knobs: IHS_SRHT_L2_TS (tensor-store items, default 1), IHS_SRHT_L2_NS (ring depth), IHS_SRHT_L2_PF (prefetch
# distance), IHS_SRHT_L2_TPOL (T store policy), IHS_SRHT_L2_DBG (timing probes: see srht.cu launch_l2_t).
for setting in "$@"; do
  echo "== ${setting:-default}"
  if [ "${CHECK:-0}" = 1 ]; then env $setting timeout -s KILL 400 python scripts/l2_check.py 2>&1 | tail -1; fi
  env $setting timeout -s KILL 300 python scripts/sketch_bench.py --config c4 --d ${D:-512} --ms ${MS:-8192,131072} --reps 3 2>&1 | grep -v Warn
done
