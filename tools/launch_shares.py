"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv):
total device time and share per kernel name."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
while rows and "Kernel Name" not in rows[0]:
    rows.pop(0)
hdr = rows[0]
iN, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iN].split("(")[0][:90]
    tot[name] += float(r[iV].replace(",", ""))
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':92s} {'launches':>8s} {'total_ms':>10s} {'avg_ms':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:92s} {cnt[k]:8d} {v / 1e6:10.3f} {v / 1e6 / cnt[k]:9.3f} {v / T * 100:5.1f}%")
