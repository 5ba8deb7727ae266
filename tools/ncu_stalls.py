"""Summarise ncu --page source CSV: stall reasons per kernel and top hot instructions."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) > 5 and r[0].startswith('0x')]
f = lambda x: float(x) if x not in ('', '-') else 0.0
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot = collections.Counter()
for r in data:
    for c in cols:
        tot[c] += f(r[h.index(c)])
s = sum(tot.values())
print('stall breakdown:', ', '.join(f"{k[6:]}={100*v/s:.1f}%" for k, v in tot.most_common(8)))
si = h.index('Warp Stall Sampling (All Samples)')
src = h.index('Source')
top = sorted(data, key=lambda r: -f(r[si]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]
for r in top:
    reasons = sorted(((f(r[h.index(c)]), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{100*f(r[si])/s:5.1f}%  {r[src][:60]:60s} {reasons}")
