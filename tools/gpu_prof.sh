#!/bin/bash
# GPU call: full ncu capture of the hot kernels of one config.
# usage: tools/gpu_prof.sh <config> <kernel-regex> <tag> [skip] [count]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=$1; K=$2; TAG=$3; S=${4:-6}; N=${5:-3}
B="python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $N -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
