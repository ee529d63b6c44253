#!/usr/bin/env python3
"""Top SASS instructions by stall samples from `ncu --page source --csv` output (sm_100a, -lineinfo)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows[:10]) if 'Address' in r)
hdr = rows[h]
ix = {k: i for i, k in enumerate(hdr)}
reasons = [k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
data = []
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    try:
        n = float(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    except ValueError:
        continue
    st = sorted(((k[6:], float(r[ix[k]] or 0)) for k in reasons), key=lambda x: -x[1])[:3]
    data.append((n, r[ix['Address']], r[ix['Source']], st))
tot = sum(d[0] for d in data)
print(f'total samples {tot:.0f}')
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for n, a, s, st in sorted(data, key=lambda x: -x[0])[:top]:
    print(f'{n:7.0f} {100*n/tot:5.1f}% {a:>6} {s[:70]:70s} ' + ' '.join(f'{k}={v:.0f}' for k, v in st if v))
