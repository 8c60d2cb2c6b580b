import os, sys, time
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch, numpy as np, synth
import paper_2602_15922_b200 as dz
M, n, heads = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
w = synth.scaled(synth.workload("C1"), heads=heads, cached_chunks=0)
spans = synth.teacher_forcing_spans(M, n); sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
q, k, v, pos = synth.span_inputs(w, spans); ntot = q.shape[0]
gq, gk = synth.draw_gains(w)
dev = torch.device("cuda")
cache = dz.ChunkKVCache(1, heads, 128, 0, ntot, w.rope_dims, gq.to(dev), gk.to(dev), flags=dz.FLAG_WRITE_LSE | dz.FLAG_BACKWARD, device=dev)
Q, K, V, P = (x.to(dev) for x in (q[None], k[None], v[None], pos))
DO = torch.randn_like(Q, dtype=torch.float32).to(torch.bfloat16)
if os.environ.get("NOFWD"):
    out = torch.randn_like(Q, dtype=torch.float32).to(torch.bfloat16); lse = torch.full((1, heads, ntot), 5.0, device=dev)
else:
    t = time.time(); out = cache.attend_spans(Q, K, V, P, sl); torch.cuda.synchronize(); print("fwd", time.time() - t, flush=True)
    lse = cache.lse(ntot); torch.cuda.synchronize(); print("lse", flush=True)
t = time.time(); r = cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO); torch.cuda.synchronize(); print("bwd", time.time() - t, flush=True)
print([float(x.float().abs().max()) for x in r])
