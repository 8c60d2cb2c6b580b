"""the denoising steps of one chunk captured as one CUDA graph.

PAPER.md Alg. 2 (l.584-585): during the N denoising steps of a chunk the KV cache
is only read (update=False); the paper runs the DiT under CUDA graphs with a
functional cache (l.627-628).  dz_attend_chunk is capture-safe (no host
synchronisation, every launch on the caller's stream), so the C3 workload --
CFG batch of 2, 8 cached chunks, 4 denoise steps (BJ:10) -- can be captured once
and replayed.  A replay must reproduce the eager calls bit for bit, leave the
committed cache untouched, and follow new inputs copied into the captured
buffers.
"""
import pytest
import torch

import synth
from helpers import GpuRun, assert_parity

pytestmark = pytest.mark.gpu


def _graph_run(w):
    run = GpuRun(w)
    run.fill()
    C = w.cached_chunks
    pos = run.streams[0].cur_pos.to(run.dev)
    ins = [[run.stack(k, s).clone() for k in ("cur_q", "cur_k", "cur_v")] for s in range(w.steps)]
    outs = [torch.empty_like(ins[s][0]) for s in range(w.steps)]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):   # warm-up on the capture stream (first-call attribute setup)
        run.cache.attend(*ins[0], pos, C, out=outs[0])
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for s in range(w.steps):
            run.cache.attend(*ins[s], pos, C, out=outs[s])
    return run, g, ins, outs, pos


def test_graph_denoise_steps_c3_bitwise_and_cache_untouched():
    w = synth.workload("C3")
    run, g, ins, outs, pos = _graph_run(w)
    C = w.cached_chunks
    before = [t.clone() for b in range(w.batch) for t in run.cache.cache_view(b)]
    eager = [run.cache.attend(*ins[s], pos, C).clone() for s in range(w.steps)]
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for s in range(w.steps):
        assert torch.equal(outs[s], eager[s]), f"graph replay differs from the eager call at step {s}"
    after = [t for b in range(w.batch) for t in run.cache.cache_view(b)]
    assert all(torch.equal(a, b) for a, b in zip(before, after)), "denoise steps changed the committed cache"
    assert run.cache.state()[0] == C * w.chunk_tokens
    # parity of a replayed step against the fp64 oracle (two heads, both CFG branches)
    for b in (0, 1):
        got = outs[3][b, :, 0:2].cpu().double().numpy()
        assert_parity(got, run.oracle_out(b=b, step=3, heads=(0, 2)), f"graph C3 b{b} step3")


def test_graph_replay_follows_new_inputs():
    w = synth.scaled(synth.workload("C3"), heads=4)
    run, g, ins, outs, pos = _graph_run(w)
    C = w.cached_chunks
    # rotate the step inputs inside the captured buffers: replay must compute the new steps
    saved = [[t.clone() for t in step] for step in ins]
    for s in range(w.steps):
        for t, src in zip(ins[s], saved[(s + 1) % w.steps]):
            t.copy_(src)
    g.replay()
    torch.cuda.synchronize()
    for s in range(w.steps):
        want = run.cache.attend(*saved[(s + 1) % w.steps], pos, C)
        assert torch.equal(outs[s], want), f"replay with new inputs differs at step {s}"


def test_graph_capture_as_the_first_call():
    # capture before any eager call: the context's one-time device setup (piece counters, RoPE
    # table) is recorded into the graph, so an eager call before the first replay must still
    # set it up itself, and the replay must reproduce that call
    w = synth.scaled(synth.workload("C1"), heads=4, cached_chunks=0)
    run = GpuRun(w, capacity=w.chunk_tokens)
    pos = run.streams[0].cur_pos.to(run.dev)
    q, k, v = [run.stack(key, 0).clone() for key in ("cur_q", "cur_k", "cur_v")]
    out = torch.empty_like(q)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="thread_local"):
        run.cache.attend(q, k, v, pos, 0, out=out)
    eager = run.cache.attend(q, k, v, pos, 0).clone()
    torch.cuda.synchronize()
    assert_parity(eager[0].cpu().double().numpy(), run.oracle_out(), "eager after capture")
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager), "first-call graph replay differs from the eager call"
