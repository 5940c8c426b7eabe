#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "interp or type2 or fullsize or transforms" > gpurun_out/pytest_gpu_sub.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_sub.log
bash tools/ab_env.sh c2 "ESN_INTERP_PITCH=37" "ESN_INTERP_PITCH=40" 20
bash tools/ab_env.sh c2 "ESN_INTERP_PITCH=40 ESN_INTERP_SLICE=384" "ESN_INTERP_PITCH=48 ESN_INTERP_SLICE=256" 20
timeout 300 python tools/timeline.py c2 3 0 > gpurun_out/timeline_c2.log 2>&1; echo "timeline rc=$?"
