#!/usr/bin/env python3
"""Executed-instruction mix (by SASS opcode) and stall totals from `ncu --page source --csv`."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows[:10]) if 'Address' in r)
hdr = rows[h]
ix = {k: i for i, k in enumerate(hdr)}
ops, st = Counter(), Counter()
tot = 0
for r in rows[h + 1:]:
    if len(r) < len(hdr):
        continue
    src = r[ix['Source']].split()
    if not src:
        continue
    op = src[1] if src[0].startswith('@') and len(src) > 1 else src[0]
    n = float(r[ix['Instructions Executed']] or 0)
    ops[op.split('.')[0]] += n
    tot += n
    st[op.split('.')[0]] += float(r[ix['Warp Stall Sampling (All Samples)']] or 0)
print(f'total warp-instructions {tot:.3e}')
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f'{op:10s} {n:.3e} {100 * n / tot:5.1f}%  stall-samples {st[op]:.0f}')
