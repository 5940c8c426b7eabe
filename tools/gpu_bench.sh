#!/bin/bash
# GPU call: per-config timings only (no tests, no profiler).  CONFIGS / ENVS.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for e in ${ENVS:-NONE}; do
for c in ${CONFIGS:-c2 c1 c3 c3f c4 c5}; do
  if [ "$e" = NONE ]; then EV=""; else EV="$e"; fi
  env $EV timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1
  python - "$c" "$e" <<'PY'
import json, sys
c = sys.argv[1]
try:
    l = [x for x in open(f'gpurun_out/bench_{c}.log') if x.startswith('{')]
    d = json.loads(l[-1])
    print(sys.argv[2], c, '%.3g pts/s' % d['value'], '%.3f ms' % d['ms_per_step'], 'frac=%.3f' % d['roofline']['frac'],
          'kern=%.3f ms' % d['roofline']['kernel_ms'], {k: round(v, 3) for k, v in d['stages_ms'].items()})
except Exception as e:
    print(c, 'FAILED', e); print(open(f'gpurun_out/bench_{c}.log').read()[-1500:])
PY
done
done
