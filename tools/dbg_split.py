import os, sys, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun
w = synth.Workload("R", 7, batch=1, heads=int(sys.argv[1]), head_dim=128, rope_dims=(44,42,42), frames=1, grid_h=1, grid_w=int(sys.argv[2]), views=1, actions=0, cached_chunks=1)
run = GpuRun(w)
run.fill()
out = run.attend()
torch.cuda.synchronize()
print("watchdog", dz.watchdog(reset=True))
o = out.cpu().double().numpy()[0]
want = run.oracle_out()
print("maxerr", np.abs(o - want).max(), "rel", np.linalg.norm(o-want)/np.linalg.norm(want))
