#!/bin/bash
# A/B of one environment switch on one config: tools/ab_env.sh <config> "<env A>" "<env B>" [steps]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ab
C=$1; A=$2; B=$3; S=${4:-20}
for rep in 1 2; do
  for side in A B; do
    e=$A; [ $side = B ] && e=$B
    env $e timeout 300 python bench.py --config $C --no-cpu --no-e2e --no-sharded --steps $S > gpurun_out/ab/$C.$side.$rep.json 2>/dev/null
    python -c "
import json
l=[x for x in open('gpurun_out/ab/$C.$side.$rep.json') if x.startswith('{')][-1]; d=json.loads(l)
print('$C $side [$e] rep $rep:', round(d['ms_per_step'],4), 'ms/step, hot', round(d['roofline']['kernel_ms'],4), 'ms')"
  done
done
