"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel launches, total and mean device time, share of the total."""
import csv
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if not l.startswith("==")]
for d in csv.DictReader(lines):
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    name = d["Kernel Name"].split("(")[0]
    rows.append((name, v * scale))
agg = defaultdict(lambda: [0, 0.0])
for n, ms in rows:
    agg[n][0] += 1
    agg[n][1] += ms
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
for n, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:48]:48s} {c:8d} {ms:10.3f} {1e3 * ms / c:10.2f} {100 * ms / tot:6.1f}%")
print(f"{'TOTAL':48s} {sum(a[0] for a in agg.values()):8d} {tot:10.3f}")
