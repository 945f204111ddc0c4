"""Summarise an `ncu --page source --csv` export (development tool): stall-reason totals and the
hottest non-DMMA instructions.  usage: python tools/ncu_source_summary.py source.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
rows = [r for r in rows[2:] if len(r) == len(h)]
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot = collections.Counter()
for r in rows:
    for c in cols:
        tot[c] += int(r[h.index(c)] or 0)
T = sum(tot.values())
print(f"samples {T}")
for c, v in tot.most_common():
    if v:
        print(f"  {c:24s} {v:9d} {100 * v / T:5.1f}%")
hot = []
for r in rows:
    s = int(r[2] or 0)
    if 'DMMA' in r[1] or r[1].strip().startswith('NOP'):
        continue
    top = {c[6:]: int(r[h.index(c)]) for c in cols if int(r[h.index(c)] or 0) > 0.2 * s and s}
    hot.append((s, r[0][-5:], r[1].strip()[:58], int(r[5] or 0), top))
hot.sort(reverse=True)
print("hottest non-DMMA instructions (samples, addr, sass, executed, dominant stalls):")
for x in hot[:top_n]:
    print(f"  {x[0]:7d} {100 * x[0] / T:5.2f}% {x[1]} {x[2]:58s} {x[3]:12d} {x[4]}")
