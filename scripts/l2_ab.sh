#!/bin/bash
# A/B of the L2-resident SRHT launch against the two-kernel path: bit-exactness at 9..12 high bits, then
# device sketch times at the C4 / C3 shapes. usage: bash scripts/l2_ab.sh > gpurun_out/l2ab.txt
IHS_SRHT_L2=1 IHS_SRHT_L2_NS=2 timeout -s KILL 400 python scripts/l2_check.py 2>&1 | tail -2
for e in "IHS_SRHT_L2=0" "IHS_SRHT_L2=1" "IHS_SRHT_L2=1 IHS_SRHT_L2_NS=3"; do
  echo "env=$e"
  env $e timeout -s KILL 300 python scripts/sketch_bench.py --config c4 --ms 8192,131072 --reps 3
  env $e timeout -s KILL 300 python scripts/sketch_bench.py --config c3 --ms 2048,65536 --reps 3
done
