#!/bin/bash
# GPU call: parity tests, per-config timings, launch list + full ncu of the hot kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in c1 c3 c3f c4 c5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"
done
B2="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$B2 > gpurun_out/plain_c2.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B2 > /dev/null 2>&1; echo "ncu launches c2 rc=$?"
$B2 > gpurun_out/plain_c2b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_interp_thread|k_setpts_bin|k_setpts_scatter" -s 3 -c 3 -o gpurun_out/prof_c2 $B2 > gpurun_out/ncu_c2.log 2>&1; echo "ncu full c2 rc=$?"
B3="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu --no-e2e"
$B3 > gpurun_out/plain_c3.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_tile|k_deconv" -s 3 -c 2 -o gpurun_out/prof_c3 $B3 > gpurun_out/ncu_c3.log 2>&1; echo "ncu full c3 rc=$?"
