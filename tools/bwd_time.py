import os, sys, time
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, ROOT)
import torch, synth
import paper_2602_15922_b200 as dz
M, n, heads = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
w = synth.scaled(synth.workload("C1"), heads=heads, cached_chunks=0)
spans = synth.teacher_forcing_spans(M, n); sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
ntot = sum(s.n_tokens for s in spans)
gq, gk = synth.draw_gains(w)
dev = torch.device("cuda")
cache = dz.ChunkKVCache(1, heads, 128, 0, ntot, w.rope_dims, gq.to(dev), gk.to(dev), flags=dz.FLAG_WRITE_LSE | dz.FLAG_BACKWARD, device=dev)
g = torch.Generator(device=dev); g.manual_seed(0)
Q, K, V, DO = (torch.randn(1, ntot, heads, 128, generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
P = torch.cat([synth.chunk_positions(w, s.chunk) for s in spans]).to(dev)
out = cache.attend_spans(Q, K, V, P, sl); lse = cache.lse(ntot)
for _ in range(3): cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO)
e1.record(); torch.cuda.synchronize()
print(f"{os.environ.get('DZ_LIB_PATH', 'libdz.so').split('/')[-1]}: bwd {e0.elapsed_time(e1) / 10:.3f} ms")
