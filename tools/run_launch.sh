#!/bin/bash
# launch lists (per-kernel device time) for configs given in $CONFIGS
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-c2 c3}; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e"
  $B > gpurun_out/plain_l_$c.log 2>&1 && \
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $B > /dev/null 2>&1
  echo "launches $c rc=$?"
done
