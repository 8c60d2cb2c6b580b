"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances from BASELINE.json north_star: max |err| <=
2e-2 and relative Frobenius <= 5e-3 on bf16 inputs; bit-exact for integer /
mask / tile decisions and for V (a copy)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from helpers import GpuRun, assert_parity, errors

pytestmark = pytest.mark.gpu


def _small(name="C1", **kw):
    return synth.scaled(synth.workload(name), **kw)


# ---------------------------------------------------------------- append --
@pytest.mark.parametrize("wname", ["C0", "C1"])
def test_append_parity(wname):
    _append_parity(synth.workload(wname))


def test_append_parity_many_heads_ring_prologue():
    # 56 heads at D = 128 exceed one pass of the token-loop prologue (48 heads): the
    # persistent TMA-ring prologue runs instead; same checks
    _append_parity(synth.scaled(synth.workload("C1"), heads=56, cached_chunks=2))


def test_positions_beyond_rope_table():
    # the prologue takes (cos, sin) from a table of positions 0..4095 and computes the others in
    # place: t straddles the table's end inside the cache (4094..4097), h and w lie far beyond it
    w = synth.workload("C0")
    run = GpuRun(w)
    for s in run.streams:
        for p in list(s.cache_pos) + [s.cur_pos]:
            p[:, 0] += 4094
            p[:, 1] += 70000
            p[:, 2] += 123456
    _append_parity(w, run)
    out = run.attend().cpu().double().numpy()[0]
    assert_parity(out, run.oracle_out(), "positions beyond the table")


def _append_parity(w, run=None):
    run = run or GpuRun(w)
    run.fill()
    torch.cuda.synchronize()
    valid, nch, last = run.cache.state()
    assert (valid, nch, last) == (w.cache_tokens, w.cached_chunks, w.cached_chunks - 1)
    kc, vc = run.cache.cache_view(0)
    s = run.streams[0]
    want_k = np.concatenate([oracle.prologue(k, run.gk, p, w.rope_dims) for k, p in zip(s.cache_k, s.cache_pos)])
    want_v = torch.cat(s.cache_v)
    assert torch.equal(vc.cpu(), want_v), "V must be copied bit-exactly"
    got = kc.cpu().double().numpy()
    # K' within 1 ulp of fp16 of the oracle's exact value, plus the fp32
    # rounding of the rotation u*c - w*s (cancellation: relative to the pair norm)
    ulp = np.spacing(np.abs(want_k).astype(np.float16)).astype(np.float64)
    pair = np.repeat(np.hypot(want_k[..., 0::2], want_k[..., 1::2]), 2, axis=-1)
    bound = ulp + 2.0 ** -20 * pair
    assert np.all(np.abs(got - want_k) <= bound), float((np.abs(got - want_k) / bound).max())
    assert np.mean(np.abs(got - want_k) <= 0.5 * ulp + 2.0 ** -20 * pair) > 0.99


# ---------------------------------------------------------------- attend --
def test_attend_parity_c0():
    w = synth.workload("C0")
    run = GpuRun(w)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    assert_parity(out, run.oracle_out(), "C0")


def test_attend_parity_c1_all_heads():
    w = synth.workload("C1")
    run = GpuRun(w)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    m, r = assert_parity(out, run.oracle_out(), "C1")
    print(f"C1 max|err|={m:.3e} rel_fro={r:.3e}")


@pytest.mark.parametrize("D,rd", [(128, (44, 42, 42)), (64, (16, 24, 24))])
@pytest.mark.parametrize("n,cached", [(1, 0), (64, 0), (130, 1), (200, 2), (256, 3), (300, 2), (320, 1), (383, 2), (1344, 1)])
def test_attend_parity_ragged(D, rd, n, cached):
    # chunk sizes spanning several tiles with ragged tails; cache of `cached` chunks
    w = synth.Workload(f"R{n}", 7, batch=1, heads=3, head_dim=D, rope_dims=rd, frames=1, grid_h=1, grid_w=n,
                       views=1, actions=0, cached_chunks=cached)
    run = GpuRun(w)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    assert_parity(out, run.oracle_out(), f"D{D} n{n} c{cached}")


def test_empty_cache_first_chunk():
    w = _small(cached_chunks=0)
    run = GpuRun(w, capacity=w.chunk_tokens)
    out = run.attend().cpu().double().numpy()[0]
    assert_parity(out, run.oracle_out(heads=(0, 40)), "empty cache")


def test_determinism_and_cache_unchanged():
    w = synth.workload("C1")
    run = GpuRun(w)
    run.fill()
    k0, v0 = [t.clone() for t in run.cache.cache_view(0)]
    a = run.attend()
    b = run.attend()
    torch.cuda.synchronize()
    assert torch.equal(a, b), "same call twice must be bitwise identical"
    k1, v1 = run.cache.cache_view(0)
    assert torch.equal(k0, k1) and torch.equal(v0, v1), "attend must not modify committed chunks"


def test_tile_map_matches_oracle_classifier():
    import paper_2602_15922_b200 as dz
    w = synth.workload("C1")
    run = GpuRun(w, flags=dz.FLAG_TILE_MAP)
    run.fill()
    run.attend()
    torch.cuda.synchronize()
    got, bm, bn = run.cache.tile_map(with_tiles=True)
    C, n = w.cached_chunks, w.chunk_tokens
    kt = oracle.chunk_tags(list(range(C)) + [C], [oracle.CLEAN] * C + [oracle.NOISY], [n] * (C + 1))
    qt = (np.full(n, C, np.int32), np.full(n, oracle.NOISY, np.int32), np.full(n, C, np.int32))
    want = oracle.tile_map(qt, kt, bm, bn)   # the kernel's (query group, key step) tiles
    assert got.shape == want.shape
    assert np.array_equal(got, want), oracle.tile_map_str(got) + " vs " + oracle.tile_map_str(want)


def test_masked_beyond_valid_is_bitwise_invariant():
    # slots past the visible range hold garbage (finite or NaN): the output must not change
    w = _small(heads=4, cached_chunks=2)
    run = GpuRun(w, slack=4 * w.chunk_tokens)
    run.fill()
    ref = run.attend().clone()
    n_total = (w.cached_chunks + 1) * w.chunk_tokens
    for fill in (float("nan"), 1e4, -3.0):
        k, v = run.cache.cache_view(0, tokens=n_total + 3 * w.chunk_tokens)
        k[n_total:] = fill
        v[n_total:] = fill
        out = run.attend()
        torch.cuda.synchronize()
        assert torch.equal(out, ref), f"fill={fill}"


def test_cfg_batch_steps_c3():
    # C3: batch 2 (cond/uncond caches drawn independently), 4 denoise steps over one cache
    w = synth.workload("C3")
    run = GpuRun(w)
    run.fill()
    k0 = [t.clone() for t in run.cache.cache_view(0)] + [t.clone() for t in run.cache.cache_view(1)]
    outs = []
    for st in range(w.steps):
        outs.append(run.attend(step=st).clone())
    torch.cuda.synchronize()
    k1 = list(run.cache.cache_view(0)) + list(run.cache.cache_view(1))
    assert all(torch.equal(a, b) for a, b in zip(k0, k1)), "committed cache changed across denoise steps"
    assert torch.equal(run.attend(step=0), outs[0]), "replaying step 0 must reproduce it bitwise"
    for b in (0, 1):
        for st in (0, 3):
            for h in (0, 39):
                got = outs[st][b, :, h:h + 1].cpu().double().numpy()
                assert_parity(got, run.oracle_out(b=b, step=st, heads=(h, h + 1)), f"C3 b{b} step{st} h{h}")


def test_long_cache_outliers_c2():
    w = synth.workload("C2")
    run = GpuRun(w)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    for h in (0, 39):
        assert_parity(out[:, h:h + 1], run.oracle_out(heads=(h, h + 1)), f"C2 head {h}")


def test_sp_shape_c4_single_gpu_sampled_rows():
    # full C4 size on one GPU (32 cached chunks of 2688 tokens); oracle on heads {0, 39}, sampled queries
    w = synth.workload("C4")
    run = GpuRun(w)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    rows = np.arange(0, w.chunk_tokens, 37)
    rows = np.unique(np.concatenate([rows, [w.chunk_tokens - 1, 2639, 2640]]))
    for h in (0, 39):
        want = run.oracle_out(heads=(h, h + 1), rows=rows)
        assert_parity(out[rows, h:h + 1], want, f"C4 head {h}")


def test_gt_injection_attend_then_commit():
    # Alg. 2 l.601-602 as a model runs it: attend the clean chunk, then commit its staged K'/V
    w = _small(heads=4, cached_chunks=2)
    run = GpuRun(w, capacity=3 * w.chunk_tokens)
    run.fill()
    C = w.cached_chunks
    s = run.streams[0]
    pos = s.cur_pos.to(run.dev)
    q, k, v = (run.stack(x, 0) for x in ("cur_q", "cur_k", "cur_v"))
    run.cache.attend(q, k, v, pos, C, kind=0)
    run.cache.commit_staged(C)
    torch.cuda.synchronize()
    assert run.cache.state() == (3 * w.chunk_tokens, 3, C)
    kc, vc = run.cache.cache_view(0)
    want_k = oracle.prologue(s.cur_k[0], run.gk, s.cur_pos, w.rope_dims)
    got = kc[C * w.chunk_tokens:].cpu().double().numpy()
    assert errors(got, want_k)[0] < 1e-2
    assert torch.equal(vc[C * w.chunk_tokens:].cpu(), s.cur_v[0])


def test_sliding_window_evict_equals_fresh_cache():
    # evicting the oldest chunk (P:510 context budget) == a cache built without it
    w = _small(heads=4, cached_chunks=3)
    run = GpuRun(w, slack=w.chunk_tokens)
    run.fill()
    run.cache.evict_front(1)
    a = run.attend(chunk_id=w.cached_chunks).cpu()
    fresh = GpuRun(w)
    for c in range(1, w.cached_chunks):
        fresh.cache.append(fresh.stack("cache_k", c), fresh.stack("cache_v", c),
                           fresh.streams[0].cache_pos[c].to(fresh.dev), c)
    b = fresh.attend().cpu()
    assert torch.equal(a, b)


def test_pipelined_bench_steps_match_fresh_caches():
    # the bench's step, back to back without host syncs: attend(noisy c) -> evict -> append(clean c)
    # -> attend(noisy c + 1) ...  The append kernel starts before the attention completes (it
    # writes slots the attention does not read) and the kernels overlap programmatically; every
    # attention must equal, bit for bit, the same attention on a cache built from scratch
    w = _small(heads=4, cached_chunks=3)
    steps = 4
    run = GpuRun(w, slack=8 * w.chunk_tokens, steps=steps)
    run.fill()
    C, n = w.cached_chunks, w.chunk_tokens
    s0 = run.streams[0]
    extra = [synth.draw_qkv(w, 0, C + i) for i in range(steps + 1)]          # (q, k, v) of chunks C..
    outs = []
    for i in range(steps):
        c = C + i
        q, k, v = extra[i]
        pos = synth.chunk_positions(w, c).to(run.dev)
        outs.append(run.cache.attend(q[None].to(run.dev), k[None].to(run.dev), v[None].to(run.dev), pos, c))
        run.cache.evict_front(1)
        run.cache.append(k[None].to(run.dev), v[None].to(run.dev), pos, c)   # the chunk enters, clean
    torch.cuda.synchronize()
    for i in range(steps):
        c = C + i
        fresh = GpuRun(w, capacity=C * n)
        for j in range(c - C, c):   # the window of C chunks the i-th attention saw
            if j < C:
                kk, vv = s0.cache_k[j], s0.cache_v[j]
            else:
                _, kk, vv = extra[j - C]
            fresh.cache.append(kk[None].to(fresh.dev), vv[None].to(fresh.dev),
                               synth.chunk_positions(w, j).to(fresh.dev), j)
        q, k, v = extra[i]
        want = fresh.cache.attend(q[None].to(fresh.dev), k[None].to(fresh.dev), v[None].to(fresh.dev),
                                  synth.chunk_positions(w, c).to(fresh.dev), c)
        torch.cuda.synchronize()
        assert torch.equal(outs[i], want), f"step {i}"


def test_online_softmax_path_c1():
    # the running-max (lazy rescale) path, forced on C1, must meet the same bar
    import paper_2602_15922_b200 as dz
    w = synth.workload("C1")
    run = GpuRun(w, flags=dz.FLAG_ONLINE_SOFTMAX)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    for h in (0, 17, 39):
        assert_parity(out[:, h:h + 1], run.oracle_out(heads=(h, h + 1)), f"online C1 head {h}")


def test_fixed_base_near_its_limit():
    # gains x1.25 (max|g| ~ 1.87): QK-norm bound ~57.7 log2 units, still the fixed softmax base
    # (p = 2^s in [2^-58, 2^58]); must meet the BASELINE tolerance like the online path
    w = synth.scaled(synth.workload("C1"), heads=4, cached_chunks=2)
    run = GpuRun(w)
    run.gq, run.gk = run.gq * 1.25, run.gk * 1.25
    import paper_2602_15922_b200 as dz
    run.cache = dz.ChunkKVCache(w.batch, w.heads, w.head_dim, w.cache_tokens, w.chunk_tokens, w.rope_dims,
                                run.gq.to(run.dev), run.gk.to(run.dev), flags=8, device=run.dev)  # tile map
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    _, bm, bn = run.cache.tile_map(with_tiles=True)
    assert bn == 128, "expected the fixed-base (ping-pong, 128-key step) kernel"
    max_abs, rel_fro = errors(out, run.oracle_out())
    scale = max(1.0, float(np.abs(run.oracle_out()).max()))
    assert np.isfinite(out).all()
    assert rel_fro <= 5e-3 and max_abs <= 2e-2 * scale, (max_abs, rel_fro, scale)


def test_large_gains_stress_online_path():
    # gains x3 (scores up to ~50, reading A19's stress case): the QK-norm bound exceeds
    # the fixed-base limit, so the kernel tracks the running max and rescales
    w = synth.scaled(synth.workload("C2"), heads=4, cached_chunks=3)
    run = GpuRun(w)
    run.gq, run.gk = run.gq * 3, run.gk * 3
    import paper_2602_15922_b200 as dz
    run.cache = dz.ChunkKVCache(w.batch, w.heads, w.head_dim, w.cache_tokens, w.chunk_tokens, w.rope_dims,
                                run.gq.to(run.dev), run.gk.to(run.dev), device=run.dev)
    run.fill()
    out = run.attend().cpu().double().numpy()[0]
    want = run.oracle_out()
    # outside BASELINE's configs: outputs reach |O| ~ 3 here, so the absolute bound is
    # scaled by max(1, max|O|) (bf16 output rounding alone is 2^-9 |O|); rel-Fro unchanged
    max_abs, rel_fro = errors(out, want)
    scale = max(1.0, float(np.abs(want).max()))
    assert np.isfinite(out).all()
    assert rel_fro <= 5e-3 and max_abs <= 2e-2 * scale, (max_abs, rel_fro, scale)


@pytest.mark.parametrize("N,B,nl,Hl,D", [(2, 1, 1344, 20, 128), (8, 2, 336, 5, 128), (4, 1, 37, 3, 64)])
def test_sp_unpack_kernel(N, B, nl, Hl, D):
    # K5: receive blocks [N][B][n_loc][Hl][D] -> [B][n_loc][N*Hl][D] (the post-exchange layout of SP)
    import paper_2602_15922_b200 as dz
    g = torch.Generator().manual_seed(N * 1000 + nl)
    recv = torch.randn(N, B, nl, Hl, D, generator=g).to(torch.bfloat16).cuda()
    out = torch.empty(B, nl, N * Hl, D, dtype=torch.bfloat16, device="cuda")
    s = dz.lib().dz_debug_sp_unpack(recv.data_ptr(), out.data_ptr(), N, B, nl, Hl, D,
                                    torch.cuda.current_stream().cuda_stream)
    assert s == 0
    torch.cuda.synchronize()
    want = recv.permute(1, 2, 0, 3, 4).reshape(B, nl, N * Hl, D)
    assert torch.equal(out, want)


# ------------------------------------------------------------- boundary hardening --
def _raw_create(gq, gk, max_abs_gain, flags=0):
    import ctypes
    import paper_2602_15922_b200 as dz
    L = dz.lib()
    c = dz.DzConfig()
    c.batch, c.heads, c.head_dim = 1, gq.shape[0], gq.shape[1]
    for i, d in enumerate((44, 42, 42)):
        c.rope_dims[i] = d
    c.cache_capacity_tokens, c.max_chunk_tokens = 256, 256
    c.q_gain, c.k_gain = gq.data_ptr(), gk.data_ptr()
    c.max_abs_gain = max_abs_gain
    c.world_size, c.rank, c.flags = 1, 0, flags
    nbytes = L.dz_cache_bytes(ctypes.byref(c))
    store = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    c.cache_storage, c.cache_bytes = store.data_ptr(), nbytes
    ctx = ctypes.c_void_p()
    s = L.dz_create(ctypes.byref(c), ctypes.byref(ctx))
    if s == 0:
        L.dz_destroy(ctx)
    return s


def test_create_reads_gains_and_rejects_underreported_bound():
    # dz_create takes max|g| from the device gains (the fixed softmax base depends on it);
    # a caller bound below it, or a non-finite gain, is rejected with DZ_ERANGE
    gq = (torch.rand(4, 128) + 0.5).cuda()
    gk = (torch.rand(4, 128) + 0.5).cuda()
    true_max = float(max(gq.abs().max(), gk.abs().max()))
    assert _raw_create(gq, gk, 0.0) == 0
    assert _raw_create(gq, gk, true_max) == 0
    assert _raw_create(gq, gk, 0.5 * true_max) == -7
    bad = gk.clone()
    bad[2, 5] = float("nan")
    assert _raw_create(gq, bad, 0.0) == -7
    big = gk.clone()
    big[0, 0] = 1e4            # sqrt(128) * 1e4 overflows fp16 Q'/K'
    assert _raw_create(gq, big, 0.0) == -7


def test_lse_against_oracle():
    # DZ_FLAG_WRITE_LSE: the per-row natural-log LSE of the last attend vs the oracle's.  |dLSE| <=
    # max_j |ds_j| (dLSE = sum_j p_j ds_j); the fp16 rounding of Q' and K' bounds |ds| by
    # 2^-10 * ||q'|| ||k'|| * scale <= 2^-10 * D * max|g_q| max|g_k| * scale (+ fp32 sums, exp2 error)
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=4, cached_chunks=2)
    run = GpuRun(w, flags=dz.FLAG_WRITE_LSE)
    run.fill()
    run.attend()
    got = run.cache.lse(w.chunk_tokens)[0].cpu().double().numpy()      # [H][n]
    s = run.streams[0]
    _, want = oracle.attend_chunk(run.gq, run.gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0],
                                  s.cur_v[0], s.cur_pos, w.rope_dims, with_lse=True)   # [n][H]
    bound = 2.0 ** -10 * w.head_dim * float(run.gq.abs().max() * run.gk.abs().max()) * w.head_dim ** -0.5 + 1e-4
    err = np.abs(got.T - want)
    assert np.all(np.isfinite(got)) and err.max() <= bound, (err.max(), bound)
    assert err.mean() < 0.1 * bound


def test_lse_online_path_against_oracle():
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload("C1"), heads=2, cached_chunks=1)
    run = GpuRun(w, flags=dz.FLAG_WRITE_LSE | dz.FLAG_ONLINE_SOFTMAX)
    run.fill()
    run.attend()
    got = run.cache.lse(w.chunk_tokens)[0].cpu().double().numpy()
    s = run.streams[0]
    _, want = oracle.attend_chunk(run.gq, run.gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0],
                                  s.cur_v[0], s.cur_pos, w.rope_dims, with_lse=True)
    bound = 2.0 ** -10 * w.head_dim * float(run.gq.abs().max() * run.gk.abs().max()) * w.head_dim ** -0.5 + 1e-4
    assert np.abs(got.T - want).max() <= bound


def test_compaction_without_slack_equals_fresh_cache():
    # slack 0: the append after an eviction runs past the slot range, so the committed window is
    # compacted to slot 0 (device copies in pieces); the next attention equals a fresh cache's
    w = _small(heads=4, cached_chunks=2)
    n = w.chunk_tokens
    run = GpuRun(w, capacity=2 * n, slack=0)
    run.fill()
    C = w.cached_chunks
    q, k, v = synth.draw_qkv(w, 0, C)
    pos = synth.chunk_positions(w, C).to(run.dev)
    run.cache.attend(q[None].to(run.dev), k[None].to(run.dev), v[None].to(run.dev), pos, C)
    run.cache.evict_front(1)
    run.cache.append(k[None].to(run.dev), v[None].to(run.dev), pos, C)       # -> compaction
    q2, k2, v2 = synth.draw_qkv(w, 0, C + 1)
    pos2 = synth.chunk_positions(w, C + 1).to(run.dev)
    got = run.cache.attend(q2[None].to(run.dev), k2[None].to(run.dev), v2[None].to(run.dev), pos2, C + 1)
    fresh = GpuRun(w, capacity=2 * n)
    s0 = fresh.streams[0]
    fresh.cache.append(s0.cache_k[1][None].to(fresh.dev), s0.cache_v[1][None].to(fresh.dev),
                       s0.cache_pos[1].to(fresh.dev), 1)
    fresh.cache.append(k[None].to(fresh.dev), v[None].to(fresh.dev), pos, C)
    want = fresh.cache.attend(q2[None].to(fresh.dev), k2[None].to(fresh.dev), v2[None].to(fresh.dev), pos2, C + 1)
    torch.cuda.synchronize()
    kc, vc = run.cache.cache_view(0)
    kf, vf = fresh.cache.cache_view(0)
    assert torch.equal(kc, kf) and torch.equal(vc, vf), "compacted cache differs"
    assert torch.equal(got, want)


def test_append_reads_inputs_after_their_producer():
    # the append kernel may be scheduled while the previous kernel drains (PDL), but must read its
    # inputs only after that kernel completes.  Here the producer of the appended k is the
    # attention kernel itself (it triggers its dependents at its start and writes `out`):
    # append(out) right behind attend(...) -> out must commit exactly what a synchronised append
    # of the finished `out` commits.
    w = _small(heads=4, cached_chunks=2)
    n, C = w.chunk_tokens, w.cached_chunks
    run = GpuRun(w, capacity=3 * n)
    run.fill()
    s0 = run.streams[0]
    pos = s0.cur_pos.to(run.dev)
    v = run.stack("cur_v", 0)
    out = run.attend()
    run.cache.append(out, v, pos, C)
    torch.cuda.synchronize()
    ref = GpuRun(w, capacity=3 * n)
    ref.fill()
    torch.cuda.synchronize()
    ref.cache.append(out.clone(), v, pos, C)
    torch.cuda.synchronize()
    kc, vc = run.cache.cache_view(0)
    kr, vr = ref.cache.cache_view(0)
    assert torch.equal(kc, kr) and torch.equal(vc, vr)


# ------------------------------------------------------- fused append + attend --
@pytest.mark.parametrize("wname,heads,cached,kind", [("C1", 40, 3, 1), ("C1", 4, 2, 0), ("C0", 2, 1, 1)])
def test_append_attend_equals_append_then_attend(wname, heads, cached, kind):
    # dz_append_attend(gt, chunk) == dz_append_kv(gt); dz_attend_chunk(chunk): output, cache contents and
    # state bitwise (one prologue launch instead of two); kind 0 (CLEAN) also stages for a commit
    import paper_2602_15922_b200 as dz
    w = synth.scaled(synth.workload(wname), heads=heads, cached_chunks=cached)
    n, C = w.chunk_tokens, w.cached_chunks
    runs = [GpuRun(w, capacity=(C + 2) * n, steps=2) for _ in range(2)]
    for r in runs:
        r.fill()
    s0 = runs[0].streams[0]
    kg, vg = (runs[0].stack(x, 1) for x in ("cur_k", "cur_v"))           # the ground-truth chunk C
    pg = synth.chunk_positions(w, C).to(runs[0].dev)
    q, k, v = synth.draw_qkv(w, 0, C + 1)
    q, k, v = (x[None].to(runs[0].dev) for x in (q, k, v))
    pq = synth.chunk_positions(w, C + 1).to(runs[0].dev)
    runs[0].cache.append(kg, vg, pg, C)
    a = runs[0].cache.attend(q, k, v, pq, C + 1, kind=kind)
    b = runs[1].cache.append_attend(kg, vg, pg, C, q, k, v, pq, C + 1, kind=kind)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert runs[0].cache.state() == runs[1].cache.state() == ((C + 1) * n, C + 1, C)
    for x, y in zip(runs[0].cache.cache_view(0), runs[1].cache.cache_view(0)):
        assert torch.equal(x, y)
    if kind == dz.CLEAN:   # the attended clean chunk was staged after the appended one: commit both ways
        for r in runs:
            r.cache.commit_staged(C + 1)
        torch.cuda.synchronize()
        for x, y in zip(runs[0].cache.cache_view(0), runs[1].cache.cache_view(0)):
            assert torch.equal(x, y)
    got = b[0].cpu().double().numpy()
    gq, gk = runs[0].gq, runs[0].gk
    want = oracle.attend_chunk(gq, gk, list(s0.cache_k) + [s0.cur_k[1]], list(s0.cache_v) + [s0.cur_v[1]],
                               list(s0.cache_pos) + [pg.cpu()], q[0].cpu(), k[0].cpu(), v[0].cpu(), pq.cpu(),
                               w.rope_dims)
    assert_parity(got, want, "append_attend")


def test_append_attend_sliding_window_with_compaction():
    # the bench's step (append_attend + evict) with no slack: compactions happen inside the fused call;
    # every attention equals the same attention on a cache built from scratch
    w = _small(heads=4, cached_chunks=3)
    n, C = w.chunk_tokens, w.cached_chunks
    run = GpuRun(w, capacity=C * n, slack=0)
    run.fill()
    s0 = run.streams[0]
    run.cache.evict_front(1)                         # cache: chunks 1 .. C-1
    extra = [synth.draw_qkv(w, 0, C + i) for i in range(5)]
    chunks = {c: (s0.cache_k[c], s0.cache_v[c]) for c in range(C)}
    for i in range(5):
        chunks[C + i] = tuple(extra[i][1:])
    outs = []
    for i in range(4):
        gt_id, cid = C + i, C + i + 1                # inject chunk C+i, denoise chunk C+i+1
        kg, vg = chunks[gt_id]
        q, k, v = extra[i + 1]
        outs.append(run.cache.append_attend(kg[None].to(run.dev), vg[None].to(run.dev),
                                            synth.chunk_positions(w, gt_id).to(run.dev), gt_id,
                                            q[None].to(run.dev), k[None].to(run.dev), v[None].to(run.dev),
                                            synth.chunk_positions(w, cid).to(run.dev), cid))
        run.cache.evict_front(1)
    torch.cuda.synchronize()
    for i in range(4):
        cid = C + i + 1
        fresh = GpuRun(w, capacity=C * n)
        for j in range(cid - C, cid):                # the window of C chunks the i-th attention saw
            kk, vv = chunks[j]
            fresh.cache.append(kk[None].to(fresh.dev), vv[None].to(fresh.dev),
                               synth.chunk_positions(w, j).to(fresh.dev), j)
        q, k, v = extra[i + 1]
        want = fresh.cache.attend(q[None].to(fresh.dev), k[None].to(fresh.dev), v[None].to(fresh.dev),
                                  synth.chunk_positions(w, cid).to(fresh.dev), cid)
        torch.cuda.synchronize()
        assert torch.equal(outs[i], want), f"step {i}"


def test_append_attend_validation():
    import paper_2602_15922_b200 as dz
    w = _small(heads=4, cached_chunks=1)
    run = GpuRun(w, capacity=2 * w.chunk_tokens)
    run.fill()
    q, k, v = (run.stack(x, 0) for x in ("cur_q", "cur_k", "cur_v"))
    pos = run.streams[0].cur_pos.to(run.dev)
    with pytest.raises(dz.DzError) as e:        # the attended chunk must come after the appended one
        run.cache.append_attend(k, v, pos, 2, q, k, v, pos, 2)
    assert e.value.status == -4
    with pytest.raises(dz.DzError) as e:        # capacity: 1 committed + 2 more would exceed 2 chunks
        run.cache.append(k, v, pos, 1)
        run.cache.append_attend(k, v, pos, 2, q, k, v, pos, 3)
    assert e.value.status == -3
    assert run.cache.state()[1] == 2            # the failed call changed nothing


def test_l2_discard_helper_leaves_no_launch_count_and_validates():
    # bench helper (dz_debug_l2_discard): enqueues without error on a buffer larger than L2, is not
    # counted as a path kernel, and rejects sizes that are not whole 128-byte lines
    import ctypes
    import paper_2602_15922_b200 as dz
    buf = torch.ones(160 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    n0 = dz.kernel_launches()
    dz.l2_discard(buf)
    torch.cuda.synchronize()
    assert dz.kernel_launches() == n0
    s = dz.lib().dz_debug_l2_discard(ctypes.c_void_p(buf.data_ptr()), 100, None)
    assert s != 0
    assert dz.lib().dz_debug_l2_discard(None, 128, None) != 0


def test_k2_clock_counters():
    # dz_debug_k2_clock: every attention launch adds its CTAs' SM cycles and globaltimer ns; the
    # ratio is a plausible SM clock (B200: at most 1.965 GHz) and a reset zeroes both sums
    import paper_2602_15922_b200 as dz
    run = GpuRun(_small("C1", heads=4, cached_chunks=2))
    run.fill()
    torch.cuda.synchronize()
    dz.k2_clock(reset=True)
    run.attend()
    torch.cuda.synchronize()
    cyc, ns = dz.k2_clock(reset=True)
    assert cyc > 0 and ns > 0
    assert 0.3 < cyc / ns < 2.2, cyc / ns
    assert dz.k2_clock() == (0, 0)
