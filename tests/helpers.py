"""Shared test plumbing: build a ChunkKVCache for a synth workload, run the
GPU path, and compute the fp64 oracle for the same seeded inputs."""
from __future__ import annotations

import numpy as np
import torch

import synth

TOL_MAX_ABS = 2e-2     # BASELINE.json north_star: max |err| <= 2e-2
TOL_REL_FRO = 5e-3     # ... and relative Frobenius error <= 5e-3


def errors(got: np.ndarray, want: np.ndarray):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    max_abs = float(np.abs(got - want).max())
    rel_fro = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
    return max_abs, rel_fro


def assert_parity(got, want, what=""):
    max_abs, rel_fro = errors(got, want)
    assert np.isfinite(got).all(), f"{what}: non-finite output"
    assert max_abs <= TOL_MAX_ABS and rel_fro <= TOL_REL_FRO, f"{what}: max|err|={max_abs:.3e} rel_fro={rel_fro:.3e}"
    return max_abs, rel_fro


class GpuRun:
    """Cache of workload w on cuda: committed chunks 0..C-1 appended via the library."""

    def __init__(self, w: synth.Workload, dev="cuda", capacity=None, slack=0, flags=0, steps=None):
        import paper_2602_15922_b200 as dz
        self.w, self.dev = w, torch.device(dev)
        self.gq, self.gk = synth.draw_gains(w)
        self.streams = [synth.draw_stream(w, b, steps=steps) for b in range(w.batch)]
        cap = w.cache_tokens if capacity is None else capacity
        self.cache = dz.ChunkKVCache(w.batch, w.heads, w.head_dim, cap, w.chunk_tokens, w.rope_dims,
                                     self.gq.to(self.dev), self.gk.to(self.dev), rope_theta=w.rope_theta,
                                     rms_eps=w.rms_eps, window_slack=slack, flags=flags, device=self.dev)

    def stack(self, key, c):
        return torch.stack([getattr(s, key)[c] for s in self.streams]).to(self.dev).contiguous()

    def fill(self):
        for c in range(self.w.cached_chunks):
            pos = self.streams[0].cache_pos[c].to(self.dev)
            self.cache.append(self.stack("cache_k", c), self.stack("cache_v", c), pos, c)

    def attend(self, step=0, chunk_id=None):
        C = self.w.cached_chunks
        pos = self.streams[0].cur_pos.to(self.dev)
        return self.cache.attend(self.stack("cur_q", step), self.stack("cur_k", step), self.stack("cur_v", step),
                                 pos, C if chunk_id is None else chunk_id)

    def oracle_out(self, b=0, step=0, heads=None, rows=None):
        """fp64 oracle for batch element b; heads (h0, h1) and query rows subsets."""
        import oracle  # test infrastructure: loaded only where a test compares against it
        s = self.streams[b]
        h0, h1 = heads if heads is not None else (0, self.w.heads)
        sl = lambda x: x[:, h0:h1]
        q, pos = sl(s.cur_q[step]), s.cur_pos
        if rows is not None:
            q, pos = q[rows], pos[rows]
        kq = sl(s.cur_k[step])
        # the current chunk's keys keep all rows; only the queries are sampled
        o = oracle.attend_chunk(self.gq[h0:h1], self.gk[h0:h1], [sl(k) for k in s.cache_k],
                                [sl(v) for v in s.cache_v], s.cache_pos, q, kq, sl(s.cur_v[step]),
                                s.cur_pos, self.w.rope_dims, self.w.rope_theta, self.w.rms_eps) \
            if rows is None else _oracle_rows(self, s, step, h0, h1, rows)
        return o


def _oracle_rows(run: GpuRun, s, step, h0, h1, rows):
    import oracle
    w = run.w
    sl = lambda x: x[:, h0:h1]
    C = len(s.cache_k)
    ks, vs, sizes = [], [], []
    for c in range(C):
        ks.append(oracle.prologue(sl(s.cache_k[c]), run.gk[h0:h1], s.cache_pos[c], w.rope_dims, w.rope_theta,
                                  w.rms_eps))
        vs.append(sl(s.cache_v[c]).double().numpy())
        sizes.append(ks[-1].shape[0])
    ks.append(oracle.prologue(sl(s.cur_k[step]), run.gk[h0:h1], s.cur_pos, w.rope_dims, w.rope_theta, w.rms_eps))
    vs.append(sl(s.cur_v[step]).double().numpy())
    sizes.append(ks[-1].shape[0])
    qn = oracle.prologue(sl(s.cur_q[step])[rows], run.gq[h0:h1], s.cur_pos[rows], w.rope_dims, w.rope_theta,
                         w.rms_eps)
    n = qn.shape[0]
    kt = oracle.chunk_tags(list(range(C)) + [C], [oracle.CLEAN] * C + [oracle.NOISY], sizes)
    qt = (np.full(n, C, np.int32), np.full(n, oracle.NOISY, np.int32), np.full(n, C, np.int32))
    return oracle.attention(qn, np.concatenate(ks), np.concatenate(vs), qt, kt)
