"""Stall-reason breakdown of an ncu --page source --csv dump over an address range (SASS view)."""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 64
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
src = hdr.index("Source")
tot = Counter()
by_instr = []
for r in data:
    a = int(r[0], 16) & 0xFFFFF
    if not (lo <= a < hi):
        continue
    row = {c: int(r[hdr.index(c)] or 0) for c in cols}
    tot.update(row)
    by_instr.append((sum(row.values()), hex(a), r[src].strip()[:60], {k: v for k, v in row.items() if v}))
s = sum(tot.values())
print("total", s)
for k, v in tot.most_common(12):
    print(f"{v:7d} {100 * v / max(s, 1):5.1f}% {k}")
print()
for t in sorted(by_instr, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    print(t)
