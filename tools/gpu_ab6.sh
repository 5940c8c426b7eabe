#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/ab_env.sh c2 "ESN_SCATTER_CTAS=3" "ESN_SCATTER_CTAS=2" 20
bash tools/ab_env.sh c2 "ESN_SCATTER_CTAS=1" "ESN_SCATTER_CTAS=2 ESN_SORT_PRIO=0" 20
