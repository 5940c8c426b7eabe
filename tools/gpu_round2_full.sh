#!/bin/bash
# round-2 full GPU check: all GPU tests, the default bench line, every config's
# line, the reference arm; then the per-kernel evidence tables.
cd "$(dirname "$0")/.."
O=gpurun_out/full
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
for c in c1 c3 c3f c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu --no-sharded > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
