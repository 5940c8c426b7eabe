"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg, order = {}, []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        n = r[ki].split('(')[0].replace('void ', '').replace('esn::', '')[:60]
        if n not in agg:
            order.append(n)
        agg.setdefault(n, []).append(float(r[vi].replace(',', '')))
    print('==', path)
    tot = 0
    for n in order:
        v = agg[n]
        m = sum(v) / len(v) / 1e3
        tot += m
        print(f'   {n:60s} n={len(v):3d} mean={m:9.1f} us')
    print(f'   {"sum of means":60s}       {tot:9.1f} us')
