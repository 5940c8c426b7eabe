#!/bin/bash
# GPU call: parity tests + per-config timings (no profiler).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2 c1 c3 c3f c4 c5}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    l = [x for x in open(f'gpurun_out/bench_{c}.log') if x.startswith('{')]
    d = json.loads(l[-1])
    print(c, '%.3g pts/s' % d['value'], '%.3f ms' % d['ms_per_step'], 'frac=%.3f' % d['roofline']['frac'],
          'kern=%.3f ms' % d['roofline']['kernel_ms'], {k: round(v, 3) for k, v in d['stages_ms'].items()})
except Exception as e:
    print(c, 'FAILED', e); print(open(f'gpurun_out/bench_{c}.log').read()[-1500:])
PY
done
