"""GPU parity of the general Fig. 10 form (dz_attend_spans) against the fp64 oracle.

PAPER.md Fig. 10 (l.505): a NOISY query of chunk k sees the CLEAN keys of
chunks < k and its own span; a CLEAN query of chunk j sees CLEAN keys of
chunks <= j.  The kernel skips (256-row x 256-key) tiles with no visible pair
and masks partial ones; its tile decisions must equal the oracle's pair
enumeration bit-exactly, and its output must meet the BJ:5 tolerance.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import assert_parity

pytestmark = pytest.mark.gpu
CLEAN, NOISY = synth.CLEAN, synth.NOISY


def _cache(w, capacity, max_chunk, flags=8, gq=None, gk=None):   # 8 = FLAG_TILE_MAP
    import paper_2602_15922_b200 as dz
    dev = torch.device("cuda")
    if gq is None:
        gq, gk = synth.draw_gains(w)
    c = dz.ChunkKVCache(w.batch, w.heads, w.head_dim, capacity, max_chunk, w.rope_dims, gq.to(dev), gk.to(dev),
                        rope_theta=w.rope_theta, rms_eps=w.rms_eps, flags=flags, device=dev)
    return c, gq, gk


def _oracle_spans(w, gq, gk, spans, q, k, v, pos, committed=None):
    """Oracle output for the span layout; committed = (k_raw list, v_raw list, pos list) of clean chunks."""
    qn = oracle.prologue(q, gq, pos, w.rope_dims, w.rope_theta, w.rms_eps)
    kn = oracle.prologue(k, gk, pos, w.rope_dims, w.rope_theta, w.rms_eps)
    ids = [s.chunk for s in spans]
    kinds = [s.kind for s in spans]
    sizes = [s.n_tokens for s in spans]
    q_tags = oracle.chunk_tags(ids, kinds, sizes)
    ks, vs, kids, kkinds, ksizes = [], [], [], [], []
    if committed is not None:
        for c, (kc, vc, pc) in enumerate(zip(*committed)):
            ks.append(oracle.prologue(kc, gk, pc, w.rope_dims, w.rope_theta, w.rms_eps))
            vs.append(vc.double().numpy())
            kids.append(c)
            kkinds.append(CLEAN)
            ksizes.append(kc.shape[0])
    ks.append(kn)
    vs.append(v.double().numpy())
    k_tags = oracle.chunk_tags(kids + ids, kkinds + kinds, ksizes + sizes)
    # span indices: committed chunks are spans 0..C-1 of the key sequence, so shift the query spans
    C = len(kids)
    q_tags = (q_tags[0], q_tags[1], q_tags[2] + C)
    out = oracle.attention(qn, np.concatenate(ks), np.concatenate(vs), q_tags, k_tags)
    return out, q_tags, k_tags


def _run(cache, spans, q, k, v, pos):
    dev = torch.device("cuda")
    out = cache.attend_spans(q[None].to(dev), k[None].to(dev), v[None].to(dev), pos.to(dev),
                             [(s.chunk, s.kind, s.n_tokens) for s in spans])
    torch.cuda.synchronize()
    return out[0]


@pytest.mark.parametrize("M", [2, 3])
def test_teacher_forcing_c0(M):
    # Fig. 10(a) training layout [C0 .. C_{M-1}; Z1 .. Z_M] at the C0 shape (64-token chunks)
    w = synth.workload("C0")
    spans = synth.teacher_forcing_spans(M, w.chunk_tokens)
    q, k, v, pos = synth.span_inputs(w, spans)
    n = q.shape[0]
    cache, gq, gk = _cache(w, 0, n)
    out = _run(cache, spans, q, k, v, pos).cpu().double().numpy()
    want, qt, kt = _oracle_spans(w, gq, gk, spans, q, k, v, pos)
    assert_parity(out, want, f"teacher forcing M={M}")
    got_map, bm, bn = cache.tile_map(with_tiles=True)
    assert np.array_equal(got_map, oracle.tile_map(qt, kt, bm, bn)), oracle.tile_map_str(got_map)


def test_teacher_forcing_wan_shape_skips_tiles():
    # M = 4 chunks of 1344 tokens (C1 chunk shape), 2 heads: ~42% visible pairs, many SKIP tiles
    w = synth.scaled(synth.workload("C1"), heads=2)
    spans = synth.teacher_forcing_spans(4, w.chunk_tokens)
    q, k, v, pos = synth.span_inputs(w, spans)
    n = q.shape[0]
    cache, gq, gk = _cache(w, 0, n)
    out = _run(cache, spans, q, k, v, pos).cpu().double().numpy()
    want, qt, kt = _oracle_spans(w, gq, gk, spans, q, k, v, pos)
    assert_parity(out, want, "teacher forcing M=4 x 1344")
    got_map, bm, bn = cache.tile_map(with_tiles=True)
    want_map = oracle.tile_map(qt, kt, bm, bn)
    assert np.array_equal(got_map, want_map)
    assert (want_map == 0).sum() > 0.3 * want_map.size, "layout must exercise tile skipping"


def test_ragged_spans_over_committed_cache():
    # committed clean chunks 0, 1 plus new spans of uneven sizes (not tile aligned), mixed kinds
    w = synth.scaled(synth.workload("C1"), heads=3)
    dev = torch.device("cuda")
    spans = [synth.Span(2, CLEAN, 300), synth.Span(3, CLEAN, 77), synth.Span(3, NOISY, 500),
             synth.Span(4, NOISY, 129), synth.Span(5, CLEAN, 64)]
    q, k, v, pos = synth.span_inputs(w, spans)
    n = q.shape[0]
    cache, gq, gk = _cache(w, 2 * w.chunk_tokens, max(n, w.chunk_tokens))
    comm_k, comm_v, comm_p = [], [], []
    for c in range(2):
        _, kc, vc = synth.draw_qkv(w, 0, c)
        pc = synth.chunk_positions(w, c)
        cache.append(kc[None].to(dev), vc[None].to(dev), pc.to(dev), c)
        comm_k.append(kc)
        comm_v.append(vc)
        comm_p.append(pc)
    out = _run(cache, spans, q, k, v, pos).cpu().double().numpy()
    want, qt, kt = _oracle_spans(w, gq, gk, spans, q, k, v, pos, (comm_k, comm_v, comm_p))
    assert_parity(out, want, "ragged spans + cache")
    got_map, bm, bn = cache.tile_map(with_tiles=True)
    assert np.array_equal(got_map, oracle.tile_map(qt, kt, bm, bn))
    # the committed cache is untouched and still usable for a plain attend
    assert cache.state() == (2 * w.chunk_tokens, 2, 1)


def test_kv_cache_equals_teacher_forcing_rows():
    # attend_chunk(current | committed) == attend_spans([C0..C_{C-1} clean; current noisy]) on its rows
    w = synth.scaled(synth.workload("C1"), heads=2, cached_chunks=3)
    dev = torch.device("cuda")
    C, n = w.cached_chunks, w.chunk_tokens
    s = synth.draw_stream(w, 0)
    cache, gq, gk = _cache(w, C * n, n)
    for c in range(C):
        cache.append(s.cache_k[c][None].to(dev), s.cache_v[c][None].to(dev), s.cache_pos[c].to(dev), c)
    a = cache.attend(s.cur_q[0][None].to(dev), s.cur_k[0][None].to(dev), s.cur_v[0][None].to(dev),
                     s.cur_pos.to(dev), C)[0]
    spans = [synth.Span(c, CLEAN, n) for c in range(C)] + [synth.Span(C, NOISY, n)]
    q = torch.cat([s.cur_q[0]] * C + [s.cur_q[0]])   # clean rows' queries are irrelevant here
    k = torch.cat(s.cache_k + [s.cur_k[0]])
    v = torch.cat(s.cache_v + [s.cur_v[0]])
    pos = torch.cat(s.cache_pos + [s.cur_pos])
    tf, _, _ = _cache(w, 0, (C + 1) * n, gq=gq, gk=gk)
    b = _run(tf, spans, q, k, v, pos)[C * n:]
    torch.cuda.synchronize()
    ga, gb = a.cpu().double().numpy(), b.cpu().double().numpy()
    want = oracle.attend_chunk(gq, gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0], s.cur_v[0],
                               s.cur_pos, w.rope_dims)
    assert_parity(ga, want, "attend_chunk")
    assert_parity(gb, want, "attend_spans rows")
    rel = np.linalg.norm(ga - gb) / np.linalg.norm(want)
    assert rel <= 5e-3, rel


def test_masked_span_perturbation_is_bitwise_invariant():
    # rows that cannot see span C2 (Z1, Z2 of the teacher-forcing layout) must not change when
    # C2's K/V change (finite values: masked keys contribute exactly 0)
    w = synth.scaled(synth.workload("C1"), heads=2)
    spans = synth.teacher_forcing_spans(3, 512)
    q, k, v, pos = synth.span_inputs(w, spans)
    cache, _, _ = _cache(w, 0, q.shape[0])
    ref = _run(cache, spans, q, k, v, pos).clone()
    k2, v2 = k.clone(), v.clone()
    k2[2 * 512:3 * 512] = 3.0   # span C2
    v2[2 * 512:3 * 512] = -7.0
    out = _run(cache, spans, q, k2, v2, pos)
    z1z2 = slice(3 * 512, 5 * 512)
    assert torch.equal(out[z1z2], ref[z1z2])
    assert torch.equal(out[:2 * 512], ref[:2 * 512])        # C0, C1 rows cannot see C2 either
    assert not torch.equal(out[5 * 512:], ref[5 * 512:])    # Z3 sees C2


def test_online_softmax_spans():
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=2)
    spans = synth.teacher_forcing_spans(3, 640)
    q, k, v, pos = synth.span_inputs(w, spans)
    cache, gq, gk = _cache(w, 0, q.shape[0], flags=dz.FLAG_ONLINE_SOFTMAX | dz.FLAG_TILE_MAP)
    out = _run(cache, spans, q, k, v, pos).cpu().double().numpy()
    want, _, _ = _oracle_spans(w, gq, gk, spans, q, k, v, pos)
    assert_parity(out, want, "online spans")


def test_spans_validation():
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=2)
    cache, _, _ = _cache(w, w.chunk_tokens, w.chunk_tokens)
    dev = torch.device("cuda")
    _, kc, vc = synth.draw_qkv(w, 0, 0)
    cache.append(kc[None].to(dev), vc[None].to(dev), synth.chunk_positions(w, 0).to(dev), 0)
    q = torch.zeros(1, 256, 2, 128, dtype=torch.bfloat16, device=dev)
    pos = torch.zeros(256, 3, dtype=torch.int32, device=dev)
    with pytest.raises(dz.DzError, match="DZ_ESTATE"):      # span id must exceed the committed id 0
        cache.attend_spans(q, q, q, pos, [(0, NOISY, 256)])
    big = w.chunk_tokens + 64
    with pytest.raises(dz.DzError, match="DZ_ECAPACITY"):   # more tokens than max_chunk
        q2 = torch.zeros(1, big, 2, 128, dtype=torch.bfloat16, device=dev)
        cache.attend_spans(q2, q2, q2, torch.zeros(big, 3, dtype=torch.int32, device=dev), [(1, NOISY, big)])
    with pytest.raises(dz.DzError, match="DZ_ESTATE"):      # nothing staged by attend_spans
        cache.attend_spans(q, q, q, pos, [(1, CLEAN, 128), (2, NOISY, 128)])
        cache.commit_staged(1)


def test_spans_tile_table_limit():
    # several spans: ceil(n/256) query groups x 128-key steps must fit the kernel's 65536-tile table
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C0"), heads=1)
    n = 2 * 40000                                   # 313 groups x 625 steps > 65536
    cache, _, _ = _cache(w, 0, n, flags=0)
    dev = torch.device("cuda")
    q = torch.zeros(1, n, 1, w.head_dim, dtype=torch.bfloat16, device=dev)
    pos = torch.zeros(n, 3, dtype=torch.int32, device=dev)
    with pytest.raises(dz.DzError, match="DZ_ESHAPE"):
        cache.attend_spans(q, q, q, pos, [(0, CLEAN, n // 2), (1, NOISY, n // 2)])
    # one span of the same size has no table: it runs
    out = cache.attend_spans(q, q, q, pos, [(1, NOISY, n)])
    torch.cuda.synchronize()
    assert out.shape == q.shape


def test_teacher_forcing_wan_shape_all_heads_hybrid_schedule():
    # all 40 heads: 1680 units, so the hybrid schedule deals whole units of unequal executed
    # length round-robin and stream-K splits the rest; heads 0 and 39 against the oracle
    w = synth.workload("C1")
    spans = synth.teacher_forcing_spans(4, w.chunk_tokens)
    q, k, v, pos = synth.span_inputs(w, spans)
    n = q.shape[0]
    cache, gq, gk = _cache(w, 0, n, flags=0)
    out = _run(cache, spans, q, k, v, pos)
    again = _run(cache, spans, q, k, v, pos)
    assert torch.equal(out, again), "the schedule must be deterministic"
    for h in (0, 39):
        sl = lambda x: x[:, h:h + 1].contiguous()
        w1 = synth.scaled(w, heads=1)
        want, _, _ = _oracle_spans(w1, gq[h:h + 1], gk[h:h + 1], spans, sl(q), sl(k), sl(v), pos)
        assert_parity(out[:, h:h + 1].cpu().double().numpy(), want, f"teacher forcing 40 heads, head {h}")
