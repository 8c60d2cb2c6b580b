"""Design-C timeline (one tile per CTA, 256-key steps): QK / PV issue and softmax events per step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("DZ_LIB_PATH", os.path.join(ROOT, "paper_2602_15922_b200", "libdz_trace.so"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun
w = synth.workload(sys.argv[1] if len(sys.argv) > 1 else "C1")
run = GpuRun(w, flags=int(os.environ.get("DZ_FLAGS", "0"))); run.fill(); run.attend(); torch.cuda.synchronize()
dz.debug_trace(True); run.attend(); torch.cuda.synchronize()
tr = dz.debug_trace(False, read=True).astype(np.int64)
base = tr[0]
R = lambda x: int((x - base) & 0xffffffff)
print(" j | QK wait issue | PV wait issue | SM S-ready S-loaded exp-done P-done | QK->S  S->P | TMA K V issued")
for j in range(0, int(os.environ.get("NSTEPS", "16"))):
    r = tr[8 * j: 8 * j + 8]
    print(f"{j:2d} | {R(r[0]):6d} {R(r[1]):6d} | {R(r[2]):6d} {R(r[3]):6d} | {R(r[4]):6d} {R(r[6]):6d} {R(r[7]):6d} {R(r[5]):6d} |"
          f" {R(r[4]) - R(r[1]):5d} {R(r[5]) - R(r[4]):5d} | {R(tr[2560 + 2 * j]):6d} {R(tr[2561 + 2 * j]):6d}")
q = tr[256 * 8: 256 * 8 + 32]
print("QK(9) per-MMA issue times:", [R(x) for x in q[:16]])
print("PV(9) per-MMA issue times:", [R(x) for x in q[16:32]])
