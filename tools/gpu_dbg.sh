#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for e in "CUDA_LAUNCH_BLOCKING=1" "ESN_INTERP=tile" "ESN_INTERP_PRODUCER=0" "ESN_INTERP_RING=3" "ESN_INTERP_PITCH=37" "ESN_SORT_AUX=0 ESN_SORT_PRIO=0"; do
echo "== $e"
env $e timeout 300 python bench.py --config c2 --no-cpu --no-e2e --no-sharded --steps 3 2>&1 | tail -2 | cut -c1-300
done
