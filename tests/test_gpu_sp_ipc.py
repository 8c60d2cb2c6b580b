"""Ulysses with peer stores across PROCESSES (rows a3 / a6): two rank processes on
one B200, each with its own context (world 2, rank r, FLAG_PEER_STORE | FLAG_EXTERNAL_EXCHANGE).  Every
rank's cache storage reaches the other process through CUDA IPC (torch.multiprocessing shares the
allocation), so K1 stores Q' / K' / V rows and K2 stores O rows straight into the other process's memory
through IPC-mapped pointers -- the node-level path, minus NVLink.  The exchanges are barriers: each
process synchronises its stream and meets the other at a multiprocessing barrier, then resumes.

Check: the two ranks' outputs, concatenated, equal the one-GPU output bitwise (FLAG_WHOLE_UNITS), for the
phase-1 appends of the cached chunks and the attend of the current chunk."""
import pytest
import torch
import torch.multiprocessing as mp

import synth

pytestmark = pytest.mark.gpu
N = 2


def _workload():
    return synth.scaled(synth.workload("C1"), heads=8, cached_chunks=2)


def _drive(cache, barrier):
    """Meet the other rank at every exchange the last call stopped at (peer stores: no transfers)."""
    while True:
        torch.cuda.synchronize()
        phase, xs = cache.sp_pending()
        assert xs == [], "peer stores move no bytes"
        barrier.wait()
        if phase < 0:
            return
        cache.sp_resume()


def _rank(r, queues, barrier, results):
    torch.cuda.set_device(0)
    import paper_2602_15922_b200 as dz
    w = _workload()
    gq, gk = synth.draw_gains(w)
    s = synth.draw_stream(w, 0)
    dev = torch.device("cuda")
    flags = dz.FLAG_WHOLE_UNITS | dz.FLAG_EXTERNAL_EXCHANGE | dz.FLAG_PEER_STORE
    cache = dz.ChunkKVCache(1, w.heads, w.head_dim, w.cache_tokens, w.chunk_tokens, w.rope_dims, gq.to(dev),
                            gk.to(dev), rope_theta=w.rope_theta, rms_eps=w.rms_eps, world_size=N, rank=r,
                            flags=flags, device=dev)
    for p in range(N):  # share this rank's storage with the other process (CUDA IPC)
        if p != r:
            queues[p].put((r, cache.storage))
    storages = [None] * N
    storages[r] = cache.storage
    for _ in range(N - 1):
        p, t = queues[r].get()
        storages[p] = t
    cache.set_peers([t.data_ptr() for t in storages])
    barrier.wait()
    nl = w.chunk_tokens // N
    sh = lambda x: x[None, r * nl:(r + 1) * nl].to(dev).contiguous()
    for c in range(w.cached_chunks):
        cache.append(sh(s.cache_k[c]), sh(s.cache_v[c]), s.cache_pos[c][r * nl:(r + 1) * nl].to(dev).contiguous(), c)
        _drive(cache, barrier)
    out = cache.attend(sh(s.cur_q[0]), sh(s.cur_k[0]), sh(s.cur_v[0]),
                       s.cur_pos[r * nl:(r + 1) * nl].to(dev).contiguous(), w.cached_chunks)
    _drive(cache, barrier)
    k_view, v_view = cache.cache_view(0)
    # (raw 16-bit patterns as numpy arrays: plain pickles, no shared-memory tensors to outlive the process)
    bits = lambda t: t.cpu().contiguous().view(torch.int16).numpy()
    results.put((r, bits(out), bits(k_view), bits(v_view)))
    barrier.wait()  # keep the storage alive until the other rank is done with it
    cache.close()


def test_sp_peer_stores_across_processes():
    import paper_2602_15922_b200 as dz
    from helpers import GpuRun
    w = _workload()
    single = GpuRun(w, flags=dz.FLAG_WHOLE_UNITS)
    single.fill()
    bits = lambda t: t.cpu().contiguous().view(torch.int16)
    want = bits(single.attend())
    k1, v1 = (bits(x) for x in single.cache.cache_view(0))
    ctx = mp.get_context("spawn")
    queues = [ctx.Queue() for _ in range(N)]
    barrier = ctx.Barrier(N)
    results = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, queues, barrier, results)) for r in range(N)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(N):
        r, out, kr, vr = results.get(timeout=600)
        got[r] = (out, kr, vr)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
    got = {r: tuple(torch.from_numpy(x) for x in v) for r, v in got.items()}
    out = torch.cat([got[r][0] for r in range(N)], dim=1)
    assert torch.equal(out, want), "2-process peer-store output differs from the 1-GPU output"
    Hl = w.heads // N
    for r in range(N):
        assert torch.equal(got[r][1], k1[:, r * Hl:(r + 1) * Hl]), f"rank {r}: K' differs from the 1-GPU cache"
        assert torch.equal(got[r][2], v1[:, r * Hl:(r + 1) * Hl]), f"rank {r}: V differs from the 1-GPU cache"
