"""Single-issuer timeline: per step, time to issue each MMA group (QK0, PV0, QK1, PV1) and its waits."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun
w = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "C1")
run = GpuRun(w); run.fill(); run.attend(); torch.cuda.synchronize()
dz.debug_trace(True); run.attend(); torch.cuda.synchronize()
tr = dz.debug_trace(False, read=True).astype(np.int64)
S = 256
base = tr[8]
R = lambda x: int((x - base) & 0xffffffff)
print("j | kv-waits-done | QK0 wait->issue->done | PV0 issue->done | QK1 wait->issue->done | PV1 issue->done || S0 ready, P0 done | S1 ready, P1 done")
peer = tr[S * 16:]
print("peer CTA softmax: j | S0 ready P0 done | S1 ready P1 done   (same clock domain only if the SMs share a clock)")
for j in range(1, 6):
    sm = peer[8 * j + 4: 8 * j + 8]
    print(f"  {j:2d} | {R(sm[0]):6d} {R(sm[1]):6d} | {R(sm[2]):6d} {R(sm[3]):6d}")
for j in range(1, 14):
    q = tr[8 * j: 8 * j + 4]; pv = tr[S * 8 + 2 * j: S * 8 + 2 * j + 2]; dn = tr[S * 12 + 4 * j: S * 12 + 4 * j + 4]
    kv = tr[S * 10 + 4 * j + 3]; sm = tr[8 * j + 4: 8 * j + 8]
    print(f"{j:2d} | {R(kv):6d} | {R(q[0]):6d} {R(q[1]):6d} {R(dn[0]):6d} | {R(pv[0]):6d} {R(dn[1]):6d} | "
          f"{R(q[2]):6d} {R(q[3]):6d} {R(dn[2]):6d} | {R(pv[1]):6d} {R(dn[3]):6d} || {R(sm[0]):6d} {R(sm[1]):6d} | {R(sm[2]):6d} {R(sm[3]):6d}")
