"""Backward kernel per-step timeline (clock() of one CTA) from the DZ_BWD_TRACE diagnostics build."""
import ctypes, os, sys
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo"); sys.path.insert(0, ROOT)
os.environ.setdefault("DZ_LIB_PATH", os.path.join(ROOT, "paper_2602_15922_b200", "libdz_bwdtrace.so"))
import numpy as np, torch, synth
import paper_2602_15922_b200 as dz
M, n, heads, cta = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
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
cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO); torch.cuda.synchronize()
L = dz.lib(); L.dz_debug_bwd_trace.argtypes = [ctypes.c_int, ctypes.c_void_p]
assert L.dz_debug_bwd_trace(cta, None) == 0
cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO); torch.cuda.synchronize()
tr = np.zeros(128 * 24, np.uint32)
assert L.dz_debug_bwd_trace(-1, tr.ctypes.data) == 0
tr = tr.reshape(128, 24).astype(np.int64)
t0 = tr[0, 0]
R = lambda x: int((x - t0) & 0xffffffff) if x else -1
names = {0: "iss:sdp", 11: "q_full", 1: "s_read", 16: "sdp_iss", 12: "p_wait", 2: "MMA345", 17: "345_iss", 3: "s_full", 4: "ldS", 5: "math",
         6: "p_ready", 8: "drainB", 7: "dq_free", 10: "prodQ"}
cols = [10, 0, 11, 1, 16, 3, 4, 5, 6, 12, 2, 17, 8, 7]
print("  i | " + " ".join(f"{names[c]:>8s}" for c in cols) + " | period")
print(f"kernel entry {R(tr[0, 15])}, after setup {R(tr[0, 13])}, compute loop done {R(tr[1, 13])}, end {R(tr[0, 14])}")
prev = None
for i in range(int(os.environ.get("NSTEPS", "30"))):
    r = tr[i]
    if not r.any(): break
    per = R(r[2]) - prev if prev is not None else 0
    prev = R(r[2])
    print(f"{i:3d} | " + " ".join(f"{R(r[c]):8d}" for c in cols) + f" | {per}")
for r_, nm in ((100, "S/dP(5)"), (101, "MMA345(5)"), (102, "S/dP(6)"), (103, "MMA345(6)")):
    print(f"{nm:10s} per-MMA issue stamps:", [R(x) for x in tr[r_, :16]])
# per-CTA start / end / steps / SM over the whole launch
ct = np.zeros(4096 * 4, np.uint32)
assert L.dz_debug_bwd_trace(-2, ct.ctypes.data) == 0
ncta = (ntot + 127) // 128 * heads
ct = ct.reshape(4096, 4)[:ncta].astype(np.int64)
g0 = ct[:, 0].min()
st_, en_ = (ct[:, 0] - g0) & 0xffffffff, (ct[:, 1] - g0) & 0xffffffff
dur = en_ - st_
steps = ct[:, 2]
print(f"launch span {en_.max() / 1e3:.1f} us; CTAs {ncta}; sum(dur)/148 {dur.sum() / 148 / 1e3:.1f} us")
for s_ in sorted(set(steps.tolist())):
    m = steps == s_
    print(f"  steps {s_:3d}: {m.sum():5d} CTAs, dur mean {dur[m].mean() / 1e3:7.1f} us  min {dur[m].min() / 1e3:7.1f}"
          f"  max {dur[m].max() / 1e3:7.1f}  ns/step {dur[m].mean() / max(s_, 1):7.0f}")
last = np.argsort(en_)[-10:]
print("last CTAs to finish (id, steps, start us, end us):", [(int(i), int(steps[i]), round(st_[i] / 1e3, 1), round(en_[i] / 1e3, 1)) for i in last])
# SM busy fraction over time
T = en_.max()
busy = np.zeros(148)
for i in range(ncta):
    busy[ct[i, 3] % 148] += dur[i]
print(f"SM busy: mean {busy.mean() / T:.3f} min {busy.min() / T:.3f}")
