import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
from helpers import GpuRun, errors
w = synth.scaled(synth.workload("C1"), heads=2)
for flags in (dz.FLAG_ONLINE_SOFTMAX, 0):
    run = GpuRun(w, flags=flags | dz.FLAG_WRITE_LSE)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    lse = run.cache.lse(w.chunk_tokens).cpu().numpy()[0]
    want, wl = None, None
    import oracle
    s = run.streams[0]
    want, wlse = oracle.attend_chunk(run.gq, run.gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0], s.cur_v[0], s.cur_pos, w.rope_dims, with_lse=True)
    e = np.abs(out - want)
    print("flags", flags, "err", errors(out, want), "lse err", np.abs(lse.T - wlse).max())
    rows = e.max(axis=(1, 2))
    print(" worst rows", np.argsort(rows)[-8:], rows[np.argsort(rows)[-8:]])
    cols = e.max(axis=(0, 1))
    print(" err by dim block of 16", [f"{cols[i:i+16].max():.2e}" for i in range(0, 128, 16)])
    print(" err by row block of 128", [f"{rows[i:i+128].max():.2e}" for i in range(0, 1344, 128)])
