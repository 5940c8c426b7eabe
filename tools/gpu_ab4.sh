#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x -k "interp or type2" > gpurun_out/pytest_gpu_sub.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_sub.log
ESN_INTERP_RING=4 timeout 300 python -m pytest tests -m gpu -q -x -k "interp or type2 or fullsize" > gpurun_out/pytest_gpu_sub4.log 2>&1; echo "pytest ring4 rc=$?"; tail -2 gpurun_out/pytest_gpu_sub4.log
bash tools/ab_env.sh c2 "ESN_INTERP_RING=2" "ESN_INTERP_RING=3" 20
bash tools/ab_env.sh c2 "ESN_INTERP_RING=4" "ESN_INTERP_RING=4 ESN_INTERP_SLICE=192" 20
bash tools/ab_env.sh c2 "ESN_INTERP_RING=3 ESN_INTERP_SLICE=256" "ESN_INTERP_RING=4 ESN_INTERP_SLICE=160" 20
