#!/bin/bash
# ring-depth scan of the L2-resident SRHT launch vs the two-kernel path (device sketch times)
for cfg in "c4 8192,131072" "c5 16384,262144" "c3 2048,65536"; do
  set -- $cfg
  echo "== $1 two-kernel"; IHS_SRHT_L2=0 timeout -s KILL 300 python scripts/sketch_bench.py --config $1 --ms $2 --reps 3
  for ns in 2 3 4 6 8 12; do
    echo "== $1 ns=$ns"; IHS_SRHT_L2=1 IHS_SRHT_L2_NS=$ns timeout -s KILL 300 python scripts/sketch_bench.py --config $1 --ms $2 --reps 3
  done
done
