#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/ab_env.sh c2 "ESN_SORT_PRIO=0 ESN_SORT_AUX=0" "ESN_SORT_PRIO=1 ESN_SORT_AUX=0" 20
bash tools/ab_env.sh c2 "ESN_SORT_PRIO=0 ESN_SORT_AUX=1" "ESN_SORT_PRIO=1 ESN_SORT_AUX=1" 20
bash tools/ab_env.sh c4 "ESN_SORT_AUX=0" "ESN_SORT_AUX=1" 10
bash tools/ab_env.sh c3f "ESN_SORT_AUX=0" "ESN_SORT_AUX=1" 10
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
