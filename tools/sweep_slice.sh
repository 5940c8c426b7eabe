#!/bin/bash
# c2 interpolator: record-slice size sweep (ESN_INTERP_SLICE)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
for s in 256 384 512 640 768 1024; do
  ESN_INTERP_SLICE=$s timeout 300 python bench.py --no-cpu --no-e2e --no-sharded --steps 20 > gpurun_out/r2/slice_$s.json 2>/dev/null
  python -c "
import json
l=[x for x in open('gpurun_out/r2/slice_$s.json') if x.startswith('{')][-1]; d=json.loads(l)
print('slice $s', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done
