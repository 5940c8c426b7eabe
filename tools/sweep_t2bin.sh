#!/bin/bash
# c2 interpolation bin shape sweep (ESN_T2_BIN=WxH)
cd "$(dirname "$0")/.."
for b in 32x32 64x16 128x8 64x32 16x64; do
  ESN_T2_BIN=$b timeout 200 python bench.py --no-cpu --no-e2e --no-sharded --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads([x for x in sys.stdin if x.startswith('{')][-1]); print('bin $b', round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done
