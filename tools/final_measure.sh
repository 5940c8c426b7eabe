#!/bin/bash
# GPU call: the full evidence set for DESIGN.md / profiles/ -- GPU tests,
# the default bench line, every config's bench line and launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/final/pytest_gpu.log
python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo "ref rc=$?"
for c in c1 c2 c3 c3f c4 c5; do
  B="python bench.py --config $c --steps 5 --warmup 3 --no-cpu"
  timeout 300 $B > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
  echo "$c rc=$?"
done
