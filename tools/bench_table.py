"""One-line-per-config summary of bench JSON logs."""
import json
import sys

print(f"{'cfg':5s} {'value pts/s':>12s} {'ms/step':>8s} {'e2e pts/s':>11s} {'e2e ms':>7s} {'kernel ms':>9s} {'frac':>6s}  stages(ms)")
for path in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(path) if l.startswith('{')][-1])
    except Exception as exc:
        print(path, 'no result', exc)
        continue
    name = d['config']['workload'].split(':')[0]
    e2e = d.get('e2e', {})
    print(f"{name:5s} {d['value']:12.3e} {d['ms_per_step']:8.3f} {e2e.get('value', 0):11.3e} "
          f"{e2e.get('ms_per_step', 0):7.2f} {d['roofline']['kernel_ms']:9.3f} {d['roofline']['frac']:6.3f}  "
          + ' '.join(f"{k}={v:.3f}" for k, v in d['stages_ms'].items()))
