"""Summarise an ncu --page source --print-source sass CSV: executed
instructions per code region (split at zero/low-count gaps)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iE, iW = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                        "Warp Stall Sampling (All Samples)"))
seen = set()
data = []
for r in rows[2:]:
    try:
        a = int(r[iA], 16)
    except Exception:
        continue
    if a in seen:
        continue
    seen.add(a)
    data.append((a, r[iS].strip(), int(r[iE] or 0), int(r[iW] or 0)))
data.sort()
base = data[0][0]
tot = sum(d[2] for d in data)
totw = sum(d[3] for d in data)
print("total warp-instructions", tot, "stall samples", totw)
# regions: runs of instructions with identical execution count
regions = []
cur = None
for a, s, e, w in data:
    if cur and e == cur[2]:
        cur[1] = a
        cur[3] += e
        cur[4] += w
        cur[5] += 1
    else:
        if cur:
            regions.append(cur)
        cur = [a, a, e, e, w, 1]
regions.append(cur)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for a0, a1, e, tote, w, n in regions:
    if tote > tot * thr:
        print(f"{a0 - base:#07x}-{a1 - base:#07x} n={n:4d} exec_each={e:12d} share={tote / tot * 100:5.1f}% stalls={w / totw * 100:5.1f}%")
