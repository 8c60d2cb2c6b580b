"""Run C1 attend with the K2 cycle trace on and print the per-step pipeline timeline of CTA 0."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun

w = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "C1")
run = GpuRun(w)
run.fill()
run.attend(); torch.cuda.synchronize()
dz.debug_trace(True)
run.attend(); torch.cuda.synchronize()
tr = dz.debug_trace(False, read=True).astype(np.int64)
S = 256
steps = min((w.kv_tokens + 127) // 128, S)
base = tr[8 * 1 + 0]
rel = lambda x: int((x - base) & 0xffffffff) if x else -1
print("j | kvwait b/e | mma t0 wait/issue | t1 wait/issue | sm0 S/P (dur) | sm1 S/P (dur) | period | sm0: ld exp st arrive")
prev = None
for j in range(1, steps):
    r = tr[j * 8: j * 8 + 8]
    d = tr[S * 10 + j * 4: S * 10 + j * 4 + 4]
    kb, ke = tr[S * 8 + 2 * j], tr[S * 8 + 2 * j + 1]
    per = (r[1] - prev) & 0xffffffff if prev is not None else 0
    prev = r[1]
    print(f"{j:3d} | {rel(kb):7d} {rel(ke):7d} | {rel(r[0]):7d} {rel(r[1]):7d} | {rel(r[2]):7d} {rel(r[3]):7d} | "
          f"{rel(r[4]):7d} {rel(r[5]):7d} ({(r[5]-r[4]) & 0xffffffff:5d}) | {rel(r[6]):7d} {rel(r[7]):7d} ({(r[7]-r[6]) & 0xffffffff:5d}) | {per}"
          f" | {(d[0]-r[4]) & 0xffffffff:4d} {(d[1]-d[0]) & 0xffffffff:4d} {(d[2]-d[1]) & 0xffffffff:4d} {(r[5]-d[2]) & 0xffffffff:4d}")
