#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/ab_env.sh c2 "ESN_SORT_COUNT_LO=0" "ESN_SORT_COUNT_LO=1" 20
timeout 300 python tools/timeline.py c2 4 0 > gpurun_out/timeline_c2.log 2>&1; tail -24 gpurun_out/timeline_c2.txt
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
