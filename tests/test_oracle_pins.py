"""Pins for the fp64 oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: a closed
form, an invariant the mathematics fixes, an independent pure-Python (fsum)
or mpmath brute force, torch's float64 SDPA as a library reduction, or the
Fig. 10 worked example in tests/golden/.  Chosen so that a plausible slip
(dropped term, wrong sign, wrong pairing, swapped operands, off-by-one chunk
rule) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


# ---------------------------------------------------------------- RMSNorm --
def test_rmsnorm_constant_closed_form():
    # x = c*1  ->  x^ = g * c / sqrt(c^2 + eps)
    H, D, eps = 3, 64, 1e-6
    g = RNG.uniform(0.5, 1.5, (H, D))
    for c in (0.0, 1e-4, 0.37, -2.5, 300.0):
        x = np.full((2, H, D), c)
        got = oracle.rmsnorm(x, g, eps)
        want = g[None] * c / math.sqrt(c * c + eps)
        np.testing.assert_allclose(got, np.broadcast_to(want, got.shape), rtol=1e-15, atol=0)


def test_rmsnorm_unit_rms_and_scale_invariance():
    H, D = 4, 128
    x = RNG.standard_normal((5, H, D))
    g = RNG.uniform(0.5, 1.5, (H, D))
    y = oracle.rmsnorm(x, g, eps=0.0)
    np.testing.assert_allclose(((y / g[None]) ** 2).mean(-1), 1.0, rtol=1e-14)
    for a in (1e-3, 7.0, 1e5):
        np.testing.assert_allclose(oracle.rmsnorm(a * x, g, eps=0.0), y, rtol=1e-13, atol=1e-15)
    # the per-head scope (A1): scaling one head leaves the others untouched
    x2 = x.copy()
    x2[:, 1] *= 10
    y2 = oracle.rmsnorm(x2, g, eps=1e-6)
    y1 = oracle.rmsnorm(x, g, eps=1e-6)
    np.testing.assert_array_equal(y2[:, 0], y1[:, 0])
    np.testing.assert_array_equal(y2[:, 2:], y1[:, 2:])


def test_rmsnorm_gain_is_per_channel_per_head():
    H, D = 2, 64
    x = np.ones((1, H, D))
    g = np.arange(H * D, dtype=np.float64).reshape(H, D) / 100 + 0.5
    y = oracle.rmsnorm(x, g, eps=0.0)
    np.testing.assert_allclose(y[0], g, rtol=1e-15)


# ------------------------------------------------------------------- RoPE --
RD128 = (44, 42, 42)
RD64 = (16, 24, 24)


def test_rope_zero_position_is_identity_exactly():
    x = RNG.standard_normal((6, 3, 128))
    pos = np.zeros((6, 3), np.int32)
    np.testing.assert_array_equal(oracle.rope3d(x, pos, RD128), x)


def test_rope_preserves_pair_norms():
    x = RNG.standard_normal((7, 2, 128))
    pos = RNG.integers(0, 130, (7, 3)).astype(np.int32)
    y = oracle.rope3d(x, pos, RD128)
    nx = np.hypot(x[..., 0::2], x[..., 1::2])
    ny = np.hypot(y[..., 0::2], y[..., 1::2])
    np.testing.assert_allclose(ny, nx, rtol=1e-14)


def test_rope_group_property():
    # R(p1) R(p2) = R(p1 + p2)
    x = RNG.standard_normal((5, 2, 64))
    p1 = RNG.integers(0, 40, (5, 3)).astype(np.int32)
    p2 = RNG.integers(0, 40, (5, 3)).astype(np.int32)
    a = oracle.rope3d(oracle.rope3d(x, p1, RD64), p2, RD64)
    b = oracle.rope3d(x, p1 + p2, RD64)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


@pytest.mark.parametrize("rd", [RD64, RD128])
def test_rope_interleaved_pairs_axis_slices_and_frequencies(rd):
    """A6/A7: pair (o_a+2i, o_a+2i+1) of axis a rotates by p_a * 1e4^(-2i/d_a).

    Measured with atan2 on unit vectors, one basis vector at a time; pair 0
    of each axis rotates by exactly p_a radians (omega_0 = 1)."""
    D = sum(rd)
    offs = [0, rd[0], rd[0] + rd[1]]
    for a in range(3):
        for i in range(rd[a] // 2):
            e = np.zeros((1, 1, D))
            e[0, 0, offs[a] + 2 * i] = 1.0
            pos = np.zeros((1, 3), np.int32)
            pos[0, a] = 1
            y = oracle.rope3d(e, pos, rd)[0, 0]
            # only this pair may move
            mask = np.ones(D, bool)
            mask[offs[a] + 2 * i: offs[a] + 2 * i + 2] = False
            assert np.all(y[mask] == 0.0)
            ang = math.atan2(y[offs[a] + 2 * i + 1], y[offs[a] + 2 * i])
            assert ang == pytest.approx(10000.0 ** (-2.0 * i / rd[a]), rel=1e-13)
            # the other axes' positions do not rotate this pair
            pos2 = np.array([[5, 9, 11]], np.int32)
            pos2[0, a] = 0
            np.testing.assert_array_equal(oracle.rope3d(e, pos2, rd)[0, 0], e[0, 0])


def test_rope_equals_complex_multiplication():
    # library reduction: numpy complex128 rotation x * e^{i phi}
    rd = RD128
    x = RNG.standard_normal((4, 2, 128))
    pos = RNG.integers(0, 120, (4, 3)).astype(np.int32)
    y = oracle.rope3d(x, pos, rd)
    offs = [0, rd[0], rd[0] + rd[1]]
    for a in range(3):
        sl = slice(offs[a], offs[a] + rd[a])
        z = x[..., sl][..., 0::2] + 1j * x[..., sl][..., 1::2]
        om = 10000.0 ** (-np.arange(rd[a] // 2) * 2.0 / rd[a])
        zr = z * np.exp(1j * pos[:, a, None, None] * om[None, None, :])
        np.testing.assert_allclose(y[..., sl][..., 0::2], zr.real, atol=1e-13)
        np.testing.assert_allclose(y[..., sl][..., 1::2], zr.imag, atol=1e-13)


def test_rope_relative_scores_shift_invariant():
    # adding delta to every t (or h or w) of queries and keys leaves all scores unchanged
    q = RNG.standard_normal((6, 1, 128))
    k = RNG.standard_normal((9, 1, 128))
    pq = RNG.integers(0, 60, (6, 3)).astype(np.int32)
    pk = RNG.integers(0, 60, (9, 3)).astype(np.int32)
    s0 = np.einsum("qd,kd->qk", oracle.rope3d(q, pq, RD128)[:, 0], oracle.rope3d(k, pk, RD128)[:, 0])
    for ax in range(3):
        d = np.zeros(3, np.int32)
        d[ax] = 17
        s1 = np.einsum("qd,kd->qk", oracle.rope3d(q, pq + d, RD128)[:, 0],
                       oracle.rope3d(k, pk + d, RD128)[:, 0])
        np.testing.assert_allclose(s1, s0, atol=1e-12)


def test_prologue_is_norm_then_rope():
    # A4: RMSNorm first (order matters only through eps and gains: RoPE does not
    # commute with a per-channel gain)
    x = RNG.standard_normal((3, 2, 64))
    g = RNG.uniform(0.5, 1.5, (2, 64))
    pos = RNG.integers(0, 9, (3, 3)).astype(np.int32)
    want = oracle.rope3d(oracle.rmsnorm(x, g, 1e-6), pos, RD64)
    np.testing.assert_array_equal(oracle.prologue(x, g, pos, RD64), want)
    other = oracle.rmsnorm(oracle.rope3d(x, pos, RD64), g, 1e-6)
    assert np.abs(other - want).max() > 1e-3


# -------------------------------------------------------------- attention --
def _all_visible_tags(nq, nk):
    q = (np.ones(nq, np.int32), np.full(nq, oracle.NOISY, np.int32), np.ones(nq, np.int32))
    k = (np.zeros(nk, np.int32), np.zeros(nk, np.int32), np.zeros(nk, np.int32))
    return q, k


def test_attention_zero_query_gives_mean_of_v():
    k = RNG.standard_normal((37, 2, 64))
    v = RNG.standard_normal((37, 2, 64))
    q = np.zeros((3, 2, 64))
    qt, kt = _all_visible_tags(3, 37)
    o = oracle.attention(q, k, v, qt, kt)
    np.testing.assert_allclose(o, np.broadcast_to(v.mean(0), o.shape), rtol=1e-13, atol=1e-15)


def test_attention_one_and_two_keys_closed_forms():
    q = RNG.standard_normal((4, 1, 64))
    k = RNG.standard_normal((2, 1, 64))
    v = RNG.standard_normal((2, 1, 64))
    qt, kt = _all_visible_tags(4, 1)
    np.testing.assert_allclose(oracle.attention(q, k[:1], v[:1], qt, kt),
                               np.broadcast_to(v[:1], (4, 1, 64)), rtol=1e-15)
    qt, kt = _all_visible_tags(4, 2)
    o = oracle.attention(q, k, v, qt, kt)
    s = np.einsum("qd,kd->qk", q[:, 0], k[:, 0]) / 8.0
    sig = lambda z: 1.0 / (1.0 + np.exp(-z))
    want = sig(s[:, 0] - s[:, 1])[:, None] * v[0, 0] + sig(s[:, 1] - s[:, 0])[:, None] * v[1, 0]
    np.testing.assert_allclose(o[:, 0], want, rtol=1e-13)


def test_attention_weights_sum_to_one_and_are_nonnegative():
    # V = one-hot basis over keys -> O row = the weight vector p
    nk = 24
    q = RNG.standard_normal((5, 1, nk)) * 3
    k = RNG.standard_normal((nk, 1, nk)) * 3
    v = np.eye(nk).reshape(nk, 1, nk)
    qt, kt = _all_visible_tags(5, nk)
    p = oracle.attention(q, k, v, qt, kt)[:, 0]
    assert np.all(p >= 0)
    np.testing.assert_allclose(p.sum(-1), 1.0, rtol=1e-14)


def test_attention_permutation_linearity_and_shift():
    q = RNG.standard_normal((6, 2, 64))
    k = RNG.standard_normal((30, 2, 64))
    v = RNG.standard_normal((30, 2, 64))
    qt, kt = _all_visible_tags(6, 30)
    o = oracle.attention(q, k, v, qt, kt)
    perm = RNG.permutation(30)
    np.testing.assert_allclose(oracle.attention(q, k[perm], v[perm], qt, kt), o, rtol=1e-12, atol=1e-14)
    v2 = RNG.standard_normal((30, 2, 64))
    o2 = oracle.attention(q, k, v2, qt, kt)
    np.testing.assert_allclose(oracle.attention(q, k, 2 * v - 3 * v2, qt, kt), 2 * o - 3 * o2,
                               rtol=1e-12, atol=1e-13)
    c = RNG.standard_normal(64)
    np.testing.assert_allclose(oracle.attention(q, k, v + c, qt, kt), o + c, rtol=1e-12, atol=1e-13)


def test_attention_lse_matches_definition():
    q = RNG.standard_normal((3, 1, 64))
    k = RNG.standard_normal((11, 1, 64))
    v = RNG.standard_normal((11, 1, 64))
    qt, kt = _all_visible_tags(3, 11)
    _, lse = oracle.attention(q, k, v, qt, kt, with_lse=True)
    s = np.einsum("qd,kd->qk", q[:, 0], k[:, 0]) / 8.0
    np.testing.assert_allclose(lse[:, 0], np.log(np.exp(s).sum(-1)), rtol=1e-14)


def test_attention_empty_visible_set_is_zero():
    q = RNG.standard_normal((2, 1, 64))
    k = RNG.standard_normal((4, 1, 64))
    qt = (np.zeros(2, np.int32), np.full(2, oracle.NOISY, np.int32), np.full(2, 7, np.int32))
    kt = (np.zeros(4, np.int32), np.full(4, oracle.NOISY, np.int32), np.zeros(4, np.int32))
    o, lse = oracle.attention(q, k, k, qt, kt, with_lse=True)
    assert np.all(o == 0) and np.all(np.isneginf(lse))


# ---------------------------------------------------------- mask / tiles --
def _fig10_tags(tokens=64, M=3):
    spans = synth.teacher_forcing_spans(M, tokens)
    ch, kd, sp = synth.span_tags(spans)
    return (ch.numpy(), kd.numpy(), sp.numpy()), spans


def test_mask_fig10_caption_example():
    # "Y3 (action) is able to attend to C0, C1, and C2"; Y3 is
    # part of noisy group Z3 and also sees its own group, nothing else.
    tags, spans = _fig10_tags(4)
    names = [f"C{s.chunk}" if s.kind == oracle.CLEAN else f"Z{s.chunk}" for s in spans]
    z3 = names.index("Z3")
    seen = {names[j] for j in range(len(spans))
            if oracle.visible(spans[z3].chunk, spans[z3].kind, z3, spans[j].chunk, spans[j].kind, j)}
    assert seen == {"C0", "C1", "C2", "Z3"}


def test_mask_rule_table_exhaustive():
    # rules (b)-(e) of S:208 with the text span removed (no text tokens in this path)
    for M in range(1, 5):
        spans = synth.teacher_forcing_spans(M, 1)
        for i, a in enumerate(spans):
            for j, b in enumerate(spans):
                vis = oracle.visible(a.chunk, a.kind, i, b.chunk, b.kind, j)
                if a.kind == oracle.CLEAN:
                    want = b.kind == oracle.CLEAN and b.chunk <= a.chunk
                else:
                    want = (b.kind == oracle.CLEAN and b.chunk < a.chunk) or i == j
                assert vis == want, (a, b)


def test_tile_map_fig10_golden():
    gold = {}
    for line in open(os.path.join(GOLD, "fig10_tilemap.txt")):
        if line.strip() and not line.startswith("#"):
            key, val = line.split()
            gold[key] = val
    tags, _ = _fig10_tags(64)
    vis = sum(oracle.visible(tags[0][s], tags[1][s], tags[2][s], tags[0][j], tags[1][j], tags[2][j])
              for s in range(0, 384, 1) for j in range(0, 384, 64)) * 64
    assert vis == int(gold["visible_pairs"])
    assert oracle.tile_map_str(oracle.tile_map(tags, tags, 64, 64)) == gold["BM64"]
    assert oracle.tile_map_str(oracle.tile_map(tags, tags, 128, 128)) == gold["BM128"]


def test_tile_map_bounds_are_not_visible():
    # a 100 x 70 all-visible layout with 64-tiles: last row/col tiles are PARTIAL
    qt, kt = _all_visible_tags(100, 70)
    assert oracle.tile_map_str(oracle.tile_map(qt, kt, 64, 64)) == "FP/PP"


def test_masked_keys_do_not_change_output_bitwise():
    # perturbing K/V of keys the rule hides leaves O bitwise identical
    tags, spans = _fig10_tags(8)
    n = len(tags[0])
    q = RNG.standard_normal((n, 1, 64))
    k = RNG.standard_normal((n, 1, 64))
    v = RNG.standard_normal((n, 1, 64))
    o = oracle.attention(q, k, v, tags, tags)
    z2 = [i for i, s in enumerate(spans) if s.kind == oracle.NOISY and s.chunk == 2][0]
    rows = tags[2] == z2
    hidden = np.array([not oracle.visible(2, oracle.NOISY, z2, tags[0][j], tags[1][j], tags[2][j])
                       for j in range(n)])
    k2, v2 = k.copy(), v.copy()
    k2[hidden] += 100 * RNG.standard_normal(k2[hidden].shape)
    v2[hidden] = 1e30
    o2 = oracle.attention(q, k2, v2, tags, tags)
    np.testing.assert_array_equal(o2[rows], o[rows])


def test_kv_cache_equals_teacher_forcing_rows():
    # attend(current | committed) == the Fig. 10(a) masked forward restricted to Z_C
    M, n = 3, 16
    tags, spans = _fig10_tags(n, M)
    N = len(tags[0])
    q = RNG.standard_normal((N, 2, 64))
    k = RNG.standard_normal((N, 2, 64))
    v = RNG.standard_normal((N, 2, 64))
    o_full = oracle.attention(q, k, v, tags, tags)
    for c in range(1, M + 1):
        zi = [i for i, s in enumerate(spans) if s.kind == oracle.NOISY and s.chunk == c][0]
        rows = np.where(tags[2] == zi)[0]
        ctx = np.where((tags[1] == oracle.CLEAN) & (tags[0] < c))[0]
        kk = np.concatenate([k[ctx], k[rows]])
        vv = np.concatenate([v[ctx], v[rows]])
        kt = oracle.chunk_tags(list(range(c)) + [c], [oracle.CLEAN] * c + [oracle.NOISY],
                               [n] * c + [n])
        qt = (np.full(n, c, np.int32), np.full(n, oracle.NOISY, np.int32), np.full(n, c, np.int32))
        np.testing.assert_allclose(oracle.attention(q[rows], kk, vv, qt, kt), o_full[rows],
                                   rtol=1e-12, atol=1e-13)


# ----------------------------------------------- whole-path brute forces --
def _py_prologue(x, g, pos, rd, theta=10000.0, eps=1e-6):
    """Scalar pure-Python RMSNorm + RoPE (independent of oracle.c)."""
    n, H, D = x.shape
    out = np.zeros_like(x)
    for t in range(n):
        for h in range(H):
            row = [float(e) for e in x[t, h]]
            r = 1.0 / math.sqrt(math.fsum(e * e for e in row) / D + eps)
            y = [row[i] * r * float(g[h, i]) for i in range(D)]
            off = 0
            for a in range(3):
                for i in range(rd[a] // 2):
                    phi = float(pos[t, a]) * theta ** (-2.0 * i / rd[a])
                    u, w = y[off + 2 * i], y[off + 2 * i + 1]
                    y[off + 2 * i] = u * math.cos(phi) - w * math.sin(phi)
                    y[off + 2 * i + 1] = u * math.sin(phi) + w * math.cos(phi)
                off += rd[a]
            out[t, h] = y
    return out


def _c0_inputs(raw=True):
    w = synth.workload("C0")
    s = synth.draw_stream(w, 0)
    if raw:   # A18: the oracle-vs-brute-force pins use the fp32 draws
        ks, vs = [], []
        for c in range(w.cached_chunks):
            _, k, v = synth.draw_qkv(w, 0, c, 0, raw=True)
            ks.append(k)
            vs.append(v)
        q, k, v = synth.draw_qkv(w, 0, w.cached_chunks, 0, raw=True)
        s.cache_k, s.cache_v, s.cur_q, s.cur_k, s.cur_v = ks, vs, [q], [k], [v]
    gq, gk = synth.draw_gains(w)
    return w, s, gq, gk


def test_whole_oracle_vs_pure_python_fsum_c0():
    w, s, gq, gk = _c0_inputs()
    rd = w.rope_dims
    o = oracle.attend_chunk(gq, gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0],
                            s.cur_v[0], s.cur_pos, rd)
    f = lambda t: t.double().numpy()
    qn = _py_prologue(f(s.cur_q[0]), f(gq), s.cur_pos.numpy(), rd)
    kn = np.concatenate([_py_prologue(f(kc), f(gk), pc.numpy(), rd)
                         for kc, pc in zip(s.cache_k + [s.cur_k[0]], s.cache_pos + [s.cur_pos])])
    vv = np.concatenate([f(x) for x in s.cache_v + [s.cur_v[0]]])
    n, H, D = qn.shape
    want = np.zeros_like(qn)
    for h in range(H):
        for i in range(n):
            sc = [math.fsum(qn[i, h, d] * kn[j, h, d] for d in range(D)) / math.sqrt(D)
                  for j in range(kn.shape[0])]
            m = max(sc)
            e = [math.exp(x - m) for x in sc]
            den = math.fsum(e)
            for d in range(D):
                want[i, h, d] = math.fsum(e[j] * vv[j, h, d] for j in range(len(e))) / den
    rel = np.linalg.norm(o - want) / np.linalg.norm(want)
    assert rel <= 1e-13, rel
    np.testing.assert_allclose(o, want, rtol=1e-11, atol=1e-14)


def test_whole_oracle_vs_mpmath_slice_c0():
    mpmath = pytest.importorskip("mpmath")
    mp = mpmath.mp
    mp.dps = 50
    w, s, gq, gk = _c0_inputs()
    rd = w.rope_dims
    o = oracle.attend_chunk(gq, gk, s.cache_k, s.cache_v, s.cache_pos, s.cur_q[0], s.cur_k[0],
                            s.cur_v[0], s.cur_pos, rd)

    def pro(x, g, p):
        D = len(x)
        r = 1 / mp.sqrt(mp.fsum(mp.mpf(float(e)) ** 2 for e in x) / D + mp.mpf("1e-6"))
        y = [mp.mpf(float(x[i])) * r * mp.mpf(float(g[i])) for i in range(D)]
        off = 0
        for a in range(3):
            for i in range(rd[a] // 2):
                phi = int(p[a]) * mp.power(10000, mp.mpf(-2 * i) / rd[a])
                u, v_ = y[off + 2 * i], y[off + 2 * i + 1]
                y[off + 2 * i] = u * mp.cos(phi) - v_ * mp.sin(phi)
                y[off + 2 * i + 1] = u * mp.sin(phi) + v_ * mp.cos(phi)
            off += rd[a]
        return y

    h = 1
    keys = s.cache_k + [s.cur_k[0]]
    vals = s.cache_v + [s.cur_v[0]]
    poss = s.cache_pos + [s.cur_pos]
    kn, vn = [], []
    for kc, vc, pc in zip(keys, vals, poss):
        for j in range(kc.shape[0]):
            kn.append(pro(kc[j, h].tolist(), gk[h].tolist(), pc[j].tolist()))
            vn.append([mp.mpf(float(e)) for e in vc[j, h].tolist()])
    for i in (0, 17, 55, 63):
        qv = pro(s.cur_q[0][i, h].tolist(), gq[h].tolist(), s.cur_pos[i].tolist())
        sc = [mp.fsum(a * b for a, b in zip(qv, kv)) / mp.sqrt(64) for kv in kn]
        m = max(sc)
        e = [mp.exp(x - m) for x in sc]
        den = mp.fsum(e)
        for d in range(0, 64, 7):
            want = mp.fsum(e[j] * vn[j][d] for j in range(len(e))) / den
            assert abs(o[i, h, d] - float(want)) <= 1e-13 * max(1.0, abs(float(want)))


def test_whole_oracle_vs_torch_float64_sdpa():
    # library reduction: torch CPU float64 SDPA with an explicit boolean mask,
    # fed the oracle's own Q'/K' (tests attention + mask, not the prologue)
    tags, spans = _fig10_tags(24, 3)
    N = len(tags[0])
    q = RNG.standard_normal((N, 3, 64))
    k = RNG.standard_normal((N, 3, 64))
    v = RNG.standard_normal((N, 3, 64))
    o = oracle.attention(q, k, v, tags, tags)
    mask = np.array([[oracle.visible(tags[0][a], tags[1][a], tags[2][a], tags[0][b], tags[1][b], tags[2][b])
                      for b in range(N)] for a in range(N)])
    t = lambda x: torch.from_numpy(x).permute(1, 0, 2).unsqueeze(0)
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v),
                                                          attn_mask=torch.from_numpy(mask))
    ref = ref[0].permute(1, 0, 2).numpy()
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-13)


def test_append_reference_v_untouched_k_is_prologue():
    w = synth.workload("C0")
    _, k, v = synth.draw_qkv(w, 0, 1)
    _, gk = synth.draw_gains(w)
    pos = synth.chunk_positions(w, 1)
    kp, vp = oracle.append_reference(k, v, gk, pos, w.rope_dims)
    np.testing.assert_array_equal(vp, v.double().numpy())
    np.testing.assert_array_equal(kp, oracle.prologue(k, gk, pos, w.rope_dims))


def test_layout_generator_c1_shapes():
    w = synth.workload("C1")
    p = synth.chunk_positions(w, 3)
    assert p.shape == (1344, 3)
    assert int(p[:1320, 0].min()) == 6 and int(p[:1320, 0].max()) == 7
    assert int(p[:, 1].max()) == 10 and int(p[:, 2].max()) == 59
    assert (p[1320:] == torch.tensor([6, 0, 0], dtype=torch.int32)).all()
    assert w.useful_flop() == pytest.approx(184.97e9, rel=1e-4)
