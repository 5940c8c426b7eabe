#!/bin/bash
# round-2 GPU check: GPU tests + the default bench line (with the sharded configs)
cd "$(dirname "$0")/.."
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
tail -5 $O/bench_default.err
