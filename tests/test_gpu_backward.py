"""NEXT-1 backward on the GPU (dz_attend_spans_backward) against the fp64 backward oracle
(oracle/backward.py, pinned by finite differences): teacher-forced span layouts (Fig. 10(a), PAPER.md
l.502-507) with an empty cache.  Tolerance: per gradient (dq, dk, dv, dg_q, dg_k)
rel-Fro <= 5e-3 and max|err| <= 2e-2 * max(1, max|grad|): BASELINE's bf16 figures, with the absolute
bound scaled because gradients (the gain gradients sum over every token) are not bounded by 1 like
O.  Measured: rel-Fro 0.5-2.4e-3 (P is rounded to bf16 and dS to fp16 before their products)."""
import numpy as np
import pytest
import torch

import synth
from helpers import errors
from oracle import backward as ob

pytestmark = pytest.mark.gpu
TOL_REL = 5e-3
TOL_ABS = 2e-2


def _case(M, n, heads, seed=0, spans=None):
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=heads, cached_chunks=0)
    spans = synth.teacher_forcing_spans(M, n) if spans is None else spans
    sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
    q, k, v, pos = synth.span_inputs(w, spans)
    ntot = q.shape[0]
    gq, gk = synth.draw_gains(w)
    g = torch.Generator().manual_seed(1234 + seed)
    dout = torch.randn(ntot, heads, 128, generator=g).to(torch.bfloat16)
    dev = torch.device("cuda")
    cache = dz.ChunkKVCache(1, heads, 128, 0, ntot, w.rope_dims, gq.to(dev), gk.to(dev),
                            flags=dz.FLAG_WRITE_LSE | dz.FLAG_BACKWARD, device=dev)
    Q, K, V, P, DO = (x.to(dev) for x in (q[None], k[None], v[None], pos, dout[None]))
    out = cache.attend_spans(Q, K, V, P, sl)
    lse = cache.lse(ntot)
    dq, dk, dv, dgq, dgk = cache.attend_spans_backward(Q, K, V, P, sl, out, lse, DO)
    torch.cuda.synchronize()
    return w, sl, (q, k, v, pos, dout, gq, gk), (dq, dk, dv, dgq, dgk), out


def _check(name, got, want):
    got = np.asarray(got, np.float64)
    max_abs, rel = errors(got, want)
    scale = max(1.0, float(np.abs(want).max()))
    print(f"{name}: max|err|={max_abs:.3e} (max|want| {np.abs(want).max():.3e}) rel_fro={rel:.3e}")
    assert np.isfinite(got).all(), name
    assert rel <= TOL_REL and max_abs <= TOL_ABS * scale, (name, max_abs, rel)


@pytest.mark.parametrize("M,n,heads", [(2, 96, 4), (3, 200, 2), (2, 37, 3), (1, 1, 2)])
def test_backward_small_all_heads(M, n, heads):
    w, sl, (q, k, v, pos, dout, gq, gk), (dq, dk, dv, dgq, dgk), _ = _case(M, n, heads)
    want = ob.spans_backward(gq, gk, q, k, v, pos, sl, dout, w.rope_dims)
    _check("dq", dq[0].cpu().double().numpy(), want["dq"])
    _check("dk", dk[0].cpu().double().numpy(), want["dk"])
    _check("dv", dv[0].cpu().double().numpy(), want["dv"])
    _check("dgq", dgq.cpu().double().numpy(), want["dgq"])
    _check("dgk", dgk.cpu().double().numpy(), want["dgk"])


def test_backward_wan_shape_two_heads():
    # the Wan-14B shape of Fig. 10(a) training, [C0 C1; Z1 Z2] x 1344 tokens, 40 heads; oracle on heads 0, 39
    w, sl, (q, k, v, pos, dout, gq, gk), (dq, dk, dv, dgq, dgk), _ = _case(2, 1344, 40)
    for h in (0, 39):
        g = lambda x: x[:, h:h + 1]
        want = ob.spans_backward(gq[h:h + 1], gk[h:h + 1], g(q), g(k), g(v), pos, sl, g(dout), w.rope_dims)
        _check(f"dq h{h}", dq[0, :, h:h + 1].cpu().double().numpy(), want["dq"])
        _check(f"dk h{h}", dk[0, :, h:h + 1].cpu().double().numpy(), want["dk"])
        _check(f"dv h{h}", dv[0, :, h:h + 1].cpu().double().numpy(), want["dv"])
        _check(f"dgq h{h}", dgq[h:h + 1].cpu().double().numpy(), want["dgq"])
        _check(f"dgk h{h}", dgk[h:h + 1].cpu().double().numpy(), want["dgk"])


def test_backward_deterministic_dv_dk():
    # dV and dK' come from one CTA per key tile in a fixed order: bitwise repeatable
    _, _, _, g1, _ = _case(2, 96, 4)
    _, _, _, g2, _ = _case(2, 96, 4)
    assert torch.equal(g1[2], g2[2])


def test_backward_many_visible_ranges():
    # 26 clean spans of 64 tokens in interleaved chunk order 25, 0, 24, 1, ..., 13, 12: a key of chunk c
    # sees the spans of chunks >= c (every other step), so key tiles near the middle have more separate
    # visible step ranges than the kernel keeps in shared memory (12) and take the span-walk path
    order = [c for pair in zip(range(25, 12, -1), range(0, 13)) for c in pair]
    spans = [synth.Span(c, synth.CLEAN, 64) for c in order]
    w, sl, (q, k, v, pos, dout, gq, gk), (dq, dk, dv, dgq, dgk), _ = _case(0, 0, 1, spans=spans)
    want = ob.spans_backward(gq, gk, q, k, v, pos, sl, dout, w.rope_dims)
    _check("dq", dq[0].cpu().double().numpy(), want["dq"])
    _check("dk", dk[0].cpu().double().numpy(), want["dk"])
    _check("dv", dv[0].cpu().double().numpy(), want["dv"])
    _check("dgq", dgq.cpu().double().numpy(), want["dgq"])
    _check("dgk", dgk.cpu().double().numpy(), want["dgk"])


def test_backward_batch_two():
    # two batch elements with their own inputs in one call: per-element gradients, gain gradients summed
    import paper_2602_15922_b200 as dz
    heads, M, n = 2, 2, 160
    w = synth.scaled(synth.workload("C1"), heads=heads, cached_chunks=0)
    spans = synth.teacher_forcing_spans(M, n)
    sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
    ins = [synth.span_inputs(w, spans, b=b) for b in (0, 1)]
    ntot = ins[0][0].shape[0]
    gq, gk = synth.draw_gains(w)
    g = torch.Generator().manual_seed(99)
    dout = torch.randn(2, ntot, heads, 128, generator=g).to(torch.bfloat16)
    dev = torch.device("cuda")
    cache = dz.ChunkKVCache(2, heads, 128, 0, ntot, w.rope_dims, gq.to(dev), gk.to(dev),
                            flags=dz.FLAG_WRITE_LSE | dz.FLAG_BACKWARD, device=dev)
    Q, K, V = (torch.stack([x[i] for x in ins]).to(dev) for i in range(3))
    P = ins[0][3].to(dev)
    out = cache.attend_spans(Q, K, V, P, sl)
    lse = cache.lse(ntot)
    dq, dk, dv, dgq, dgk = cache.attend_spans_backward(Q, K, V, P, sl, out, lse, dout.to(dev))
    torch.cuda.synchronize()
    wants = [ob.spans_backward(gq, gk, q, k, v, pos, sl, dout[b], w.rope_dims)
             for b, (q, k, v, pos) in enumerate(ins)]
    for b in (0, 1):
        _check(f"dq b{b}", dq[b].cpu().double().numpy(), wants[b]["dq"])
        _check(f"dk b{b}", dk[b].cpu().double().numpy(), wants[b]["dk"])
        _check(f"dv b{b}", dv[b].cpu().double().numpy(), wants[b]["dv"])
    _check("dgq", dgq.cpu().double().numpy(), wants[0]["dgq"] + wants[1]["dgq"])
    _check("dgk", dgk.cpu().double().numpy(), wants[0]["dgk"] + wants[1]["dgk"])
