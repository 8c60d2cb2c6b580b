"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel time and share."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, out, cmd):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        tot[r[ki][:70]] += v
        cnt[r[ki][:70]] += 1
    s = sum(tot.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none; cmd: {cmd}",
             "# per kernel: total device us, launches, mean us/launch, share of listed launches (cold, serialised)"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{tot[k]:10.1f} us {cnt[k]:4d} {tot[k] / cnt[k]:9.1f} us/launch {100 * tot[k] / s:5.1f}%  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], " ".join(sys.argv[3:]))
