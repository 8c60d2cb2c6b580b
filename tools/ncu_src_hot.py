"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = []
for r in rows[2:]:          # first kernel section only
    if r and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        data.append(r)
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
iS, iX = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
tot = Counter()
items = []
for i, r in enumerate(data):
    st = {c: int(r[hdr.index(c)] or 0) for c in cols}
    tot.update(st)
    items.append((int(r[iX] or 0), i, r[iS].strip()[:70], int(r[iE] or 0), {k[6:]: v for k, v in st.items() if v}))
s = sum(tot.values())
print("total samples", s)
for k, v in tot.most_common(14):
    print(f"{v:8d} {100 * v / max(s, 1):5.1f}% {k}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print()
for smp, i, src, ex, st in sorted(items, reverse=True)[:n]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{smp:7d} #{i:5d} x{ex:9d} {src:70s} {top}")
