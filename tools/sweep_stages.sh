#!/bin/bash
# usage: VAR=NAME VALUES="a b c" CONFIG=c2 tools/sweep_stages.sh -> per-stage ms per value
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in $VALUES; do
  env $VAR=$v timeout 300 python bench.py --config ${CONFIG:-c2} --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweep_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    l = [x for x in open(f'gpurun_out/sweep_{v}.log') if x.startswith('{')]
    d = json.loads(l[-1])
    print(v, '%.3f ms/step' % d['ms_per_step'], {k: round(x, 3) for k, x in d['stages_ms'].items()})
except Exception as e:
    print(v, 'FAILED', e, open(f'gpurun_out/sweep_{v}.log').read()[-800:])
PY
done
