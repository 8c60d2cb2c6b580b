"""Per-CTA K2 timeline on C1 (stream-K segments, combines): where each pair spends its time."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("DZ_LIB_PATH", os.path.join(ROOT, "paper_2602_15922_b200", "libdz_trace.so"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun

w = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "C1")
run = GpuRun(w)
run.fill()
import time
t_end = time.time() + float(os.environ.get("WARM_S", "0"))
while True:   # optional warm phase (clocks under sustained load)
    for _ in range(50):
        run.attend()
    torch.cuda.synchronize()
    if time.time() >= t_end:
        break
dz.debug_trace(True)
run.attend(); torch.cuda.synchronize()
tr = dz.debug_trace(False, read=True).astype(np.int64)
tl = tr[8192:].reshape(160, 64)
n = 148
t0 = min(int(x) for x in tl[:n, 0])
R = lambda x: ((int(x) - t0) & 0xffffffff) / 1000.0
ends = [R(tl[c, 1]) for c in range(n)]
eff = [((int(tl[c, 3]) - int(tl[c, 2])) & 0xffffffff) / max(1, (int(tl[c, 1]) - int(tl[c, 0])) & 0xffffffff) for c in range(n)]
print(f"effective SM clock during the kernel (clock()/globaltimer): median {np.median(eff):.3f} GHz, min {min(eff):.3f}")
print(f"kernel span (first start .. last end): {max(ends):.1f} us; end spread min {min(ends):.1f} median {np.median(ends):.1f}")
for c in list(range(0, n, 2))[:74]:
    segs = int(tl[c, 4])
    c0 = int(tl[c, 2])
    K = lambda x: ((int(x) - c0) & 0xffffffff) / 1000.0   # kilo-cycles since the CTA's start
    parts = " ".join(f"[{K(tl[c, 8 + 4 * i]):6.1f} {K(tl[c, 9 + 4 * i]):6.1f} {K(tl[c, 10 + 4 * i]):6.1f} {K(tl[c, 11 + 4 * i]):6.1f}]"
                     for i in range(min(segs, 14)))
    parts += " | pieces: " + " ".join(f"[{K(tl[c, 50 + 5 * i]):6.1f} {K(tl[c, 51 + 5 * i]):6.1f} {K(tl[c, 52 + 5 * i]):6.1f} {K(tl[c, 53 + 5 * i]):6.1f}]" for i in range(2))
    print(f"cta {c:3d} end {R(tl[c, 1]):6.1f}us {K(tl[c, 3]):6.1f}kclk segs {segs} comb {int(tl[c, 5])} | {parts}")
