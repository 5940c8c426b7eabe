#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for mb in 24 32 48 64; do
bash tools/ab_env.sh c2 "ESN_OUT_CHUNK_MB=94" "ESN_OUT_CHUNK_MB=$mb" 20 | grep "rep 2"
done
