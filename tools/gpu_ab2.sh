#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c2 c5 c3f; do
bash tools/ab_env.sh $c "ESN_GRAPH_MAX_M=524288" "ESN_GRAPH_MAX_M=100000000" 20
done
