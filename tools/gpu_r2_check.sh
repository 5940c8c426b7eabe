#!/bin/bash
# round-2 GPU check: GPU tests + the default bench line (with the sharded configs)
cd "$(dirname "$0")/.."
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
tail -5 $O/bench_default.err
for c in c3 c3f c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
