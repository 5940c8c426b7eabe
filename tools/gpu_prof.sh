#!/bin/bash
# GPU call: full ncu capture of the hot kernels of one config, exported to
# text on the box (raw metrics csv + per-kernel SASS stall table).  The
# .ncu-rep is kept only with KEEP=1 (gpurun_out/ is capped at 64 MiB).
# usage: tools/gpu_prof.sh <config> <kernel-regex> <tag> [skip] [count]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=$1; K=$2; TAG=$3; S=${4:-6}; N=${5:-3}
B="python bench.py --config $C --steps 2 --warmup 3 --no-cpu --no-e2e"
$B > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $N -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu $TAG rc=$?"
if [ -f gpurun_out/prof_$TAG.ncu-rep ]; then
  python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/sum_$TAG.txt 2>&1
  for k in $(echo "$K" | tr '|' ' '); do
    python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep "$k" 2>/dev/null | sed -n '/-- stalls/,$p' >> gpurun_out/sum_$TAG.txt
  done
  [ "$KEEP" = "1" ] || rm -f gpurun_out/prof_$TAG.ncu-rep
fi
