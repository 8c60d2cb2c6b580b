"""Ulysses sequence parallelism (§8(e); BASELINE.json C4)
and the CFG batch split (C3, PAPER.md l.141 / l.617), with N ranks emulated on
one B200 (tests/sp_emul.py: the library's own exchange plan delivered with one
device copy per transfer; everything else is the N-GPU code path).

Checks (SURVEY §8(c) "SP" pin, reading A21):
  * N-rank output == 1-GPU output bitwise when every unit is computed whole
    (FLAG_WHOLE_UNITS: a unit's bits depend only on its rows and keys);
  * with the default stream-K schedule: rel-Fro <= 1e-3 against the 1-GPU run
    and the BASELINE tolerance against the fp64 oracle;
  * C4 at N = 2, 4, 8: heads {0, 39} (ranks 0 and N-1) against the oracle;
  * the appended (phase-1 exchanged) K' / V of every rank equal the 1-GPU
    cache's head slice bitwise, and rank 0's against the oracle per element.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import GpuRun, assert_parity, errors
from sp_emul import SpRanks

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _stack(run, key, c):
    return torch.stack([getattr(s, key)[c] for s in run.streams]).contiguous()


def _fill_both(w, single: GpuRun, sp: SpRanks):
    single.fill()
    for c in range(w.cached_chunks):
        sp.append(_stack(single, "cache_k", c), _stack(single, "cache_v", c), single.streams[0].cache_pos[c], c)


def _attend_both(w, single: GpuRun, sp: SpRanks, step=0):
    a = single.attend(step=step)
    q, k, v = (_stack(single, x, step) for x in ("cur_q", "cur_k", "cur_v"))
    b = sp.attend(q, k, v, single.streams[0].cur_pos, w.cached_chunks)
    torch.cuda.synchronize()
    return a, b


def _check_caches(w, single: GpuRun, sp: SpRanks):
    Hl = w.heads // sp.N
    for b in range(w.batch):
        k1, v1 = single.cache.cache_view(b)
        for r, (kr, vr) in enumerate(sp.cache_views(b)):
            assert torch.equal(kr, k1[:, r * Hl:(r + 1) * Hl]), f"rank {r} b {b}: K' differs from the 1-GPU cache"
            assert torch.equal(vr, v1[:, r * Hl:(r + 1) * Hl]), f"rank {r} b {b}: V differs from the 1-GPU cache"


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("N", [2, 4, 8])
def test_sp_bitwise_equals_single_gpu_c1(N, peer):
    import paper_2602_15922_b200 as dz
    w = synth.workload("C1")
    single = GpuRun(w, flags=dz.FLAG_WHOLE_UNITS)
    sp = SpRanks(w, N, single.gq, single.gk, DEV, flags=dz.FLAG_WHOLE_UNITS, peer=peer)
    _fill_both(w, single, sp)
    _check_caches(w, single, sp)
    a, b = _attend_both(w, single, sp)
    assert sp.phases[-2:] == [0, 2], sp.phases   # attend: pre-exchange then post-exchange
    assert torch.equal(a, b), f"N={N}: SP output differs from the 1-GPU output"
    if peer:
        assert sp.transfers == 0, "peer stores: the exchanges must move no bytes"
    got = b[0].cpu().double().numpy()
    for h in (0, w.heads - 1):
        assert_parity(got[:, h:h + 1], single.oracle_out(heads=(h, h + 1)), f"SP N={N} head {h}")
    sp.close()


@pytest.mark.parametrize("N", [2, 8])
def test_sp_default_schedule_c1(N):
    # stream-K splits differ with the unit count, so the bits may differ: rel-Fro <= 1e-3 (A21)
    w = synth.workload("C1")
    single = GpuRun(w)
    sp = SpRanks(w, N, single.gq, single.gk, DEV)
    _fill_both(w, single, sp)
    a, b = _attend_both(w, single, sp)
    _, rel = errors(b.cpu().double().numpy(), a.cpu().double().numpy())
    assert rel <= 1e-3, rel
    got = b[0].cpu().double().numpy()
    for h in (0, w.heads - 1):
        assert_parity(got[:, h:h + 1], single.oracle_out(heads=(h, h + 1)), f"SP N={N} head {h}")
    sp.close()


@pytest.mark.parametrize("peer", [False, True])
def test_sp_append_against_oracle(peer):
    # phase-1 exchange: rank r's cache holds K' / V of heads [r*Hl, (r+1)*Hl) of every token
    w = synth.scaled(synth.workload("C1"), cached_chunks=2)
    N = 4
    gq, gk = synth.draw_gains(w)
    sp = SpRanks(w, N, gq, gk, DEV, peer=peer)
    s = synth.draw_stream(w, 0)
    for c in range(w.cached_chunks):
        sp.append(s.cache_k[c][None], s.cache_v[c][None], s.cache_pos[c], c)
    torch.cuda.synchronize()
    assert all(c.state() == (w.cache_tokens, w.cached_chunks, w.cached_chunks - 1) for c in sp.caches)
    Hl = w.heads // N
    want_k = np.concatenate([oracle.prologue(k, gk, p, w.rope_dims) for k, p in zip(s.cache_k, s.cache_pos)])
    want_v = torch.cat(s.cache_v)
    for r, (kr, vr) in enumerate(sp.cache_views(0)):
        assert torch.equal(vr.cpu(), want_v[:, r * Hl:(r + 1) * Hl]), f"rank {r}: V"
        wk = want_k[:, r * Hl:(r + 1) * Hl]
        got = kr.cpu().double().numpy()
        ulp = np.spacing(np.abs(wk).astype(np.float16)).astype(np.float64)
        pair = np.repeat(np.hypot(wk[..., 0::2], wk[..., 1::2]), 2, axis=-1)
        assert np.all(np.abs(got - wk) <= ulp + 2.0 ** -20 * pair), f"rank {r}: K'"
    sp.close()


@pytest.mark.parametrize("N,peer", [(2, False), (4, False), (8, False), (8, True)])
def test_sp_c4_against_oracle_and_single_gpu(N, peer):
    # BASELINE C4: 32 cached chunks of 2688 tokens, 40/N heads per rank; oracle on heads 0 and 39
    # (ranks 0 and N-1) at sampled query rows; the N-rank output against the 1-GPU run
    import paper_2602_15922_b200 as dz
    w = synth.workload("C4")
    single = GpuRun(w, flags=dz.FLAG_WHOLE_UNITS)
    sp = SpRanks(w, N, single.gq, single.gk, DEV, flags=dz.FLAG_WHOLE_UNITS, peer=peer)
    _fill_both(w, single, sp)
    a, b = _attend_both(w, single, sp)
    assert torch.equal(a, b), f"C4 N={N}: SP output differs from the 1-GPU output"
    got = b[0].cpu().double().numpy()
    rows = np.unique(np.concatenate([np.arange(0, w.chunk_tokens, 53), [w.chunk_tokens - 1, 2639, 2640],
                                     [r * (w.chunk_tokens // N) for r in range(N)]]))
    for h in (0, w.heads - 1):
        want = single.oracle_out(heads=(h, h + 1), rows=rows)
        assert_parity(got[rows, h:h + 1], want, f"C4 N={N} head {h}")
    sp.close()


@pytest.mark.parametrize("peer", [False, True])
def test_sp_gt_injection_and_window(peer):
    # under SP: attend a clean chunk then commit its staged (exchanged) K'/V; evict the oldest
    # chunk (compaction with no slack); the next attention equals the 1-GPU one bitwise
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=8, cached_chunks=2)
    N, C, n = 4, 2, w.chunk_tokens
    single = GpuRun(w, capacity=3 * n, flags=dz.FLAG_WHOLE_UNITS, steps=2)
    sp = SpRanks(w, N, single.gq, single.gk, DEV, capacity=3 * n, flags=dz.FLAG_WHOLE_UNITS, peer=peer)
    _fill_both(w, single, sp)
    s0 = single.streams[0]
    q, k, v = (_stack(single, x, 0) for x in ("cur_q", "cur_k", "cur_v"))
    a = single.cache.attend(q.to(DEV), k.to(DEV), v.to(DEV), s0.cur_pos.to(DEV), C, kind=dz.CLEAN)
    single.cache.commit_staged(C)
    b = sp.attend(q, k, v, s0.cur_pos, C, kind=dz.CLEAN)
    sp.commit_staged(C)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    _check_caches(w, single, sp)
    single.cache.evict_front(1)
    sp.evict_front(1)
    pos = synth.chunk_positions(w, C + 1)
    q2, k2, v2 = (_stack(single, x, 1) for x in ("cur_q", "cur_k", "cur_v"))
    a2 = single.cache.attend(q2.to(DEV), k2.to(DEV), v2.to(DEV), pos.to(DEV), C + 1)
    b2 = sp.attend(q2, k2, v2, pos, C + 1)
    torch.cuda.synchronize()
    assert torch.equal(a2, b2)
    sp.close()


@pytest.mark.parametrize("peer", [False, True])
def test_sp_teacher_forcing_spans(peer):
    # Fig. 10(a) layout under SP: [C0 C1; Z1 Z2], sequence-sharded; equals the 1-GPU call bitwise
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=8, cached_chunks=0)
    N, n = 2, 320
    spans = synth.teacher_forcing_spans(2, n)
    q, k, v, pos = synth.span_inputs(w, spans)
    q, k, v = q[None], k[None], v[None]
    gq, gk = synth.draw_gains(w)
    sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
    one = dz.ChunkKVCache(1, w.heads, w.head_dim, 0, 4 * n, w.rope_dims, gq.to(DEV), gk.to(DEV),
                          flags=dz.FLAG_WHOLE_UNITS, device=DEV)
    a = one.attend_spans(q.to(DEV), k.to(DEV), v.to(DEV), pos.to(DEV), sl)
    sp = SpRanks(w, N, gq, gk, DEV, capacity=0, max_chunk=4 * n, flags=dz.FLAG_WHOLE_UNITS, peer=peer)
    b = sp.attend_spans(q, k, v, pos, sl)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    sp.close()


def test_cfg_split_two_contexts_equal_batch2():
    # C3 on "2 GPUs": cond and uncond each in their own batch-1 context, no
    # collective; bitwise equal to the batch-2 context with whole units, and oracle parity
    import paper_2602_15922_b200 as dz
    w = synth.workload("C3")
    both = GpuRun(w, flags=dz.FLAG_WHOLE_UNITS)
    both.fill()
    outs = [both.attend(step=st).clone() for st in (0, 3)]
    w1 = synth.scaled(w, batch=1)
    for b in range(2):
        one = GpuRun(w1, flags=dz.FLAG_WHOLE_UNITS)
        one.streams = [both.streams[b]]
        one.fill()
        for i, st in enumerate((0, 3)):
            got = one.attend(step=st)
            torch.cuda.synchronize()
            assert torch.equal(got[0], outs[i][b]), f"CFG element {b} step {st}"
            g = got[0].cpu().double().numpy()
            for h in (0, 39):
                assert_parity(g[:, h:h + 1], both.oracle_out(b=b, step=st, heads=(h, h + 1)), f"cfg b{b} s{st} h{h}")
        one.cache.close()
