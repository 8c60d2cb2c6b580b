"""Pins of the fp64 backward oracle (oracle/backward.py): central finite differences of the C
oracle's forward (oracle.prologue + oracle.attention), closed forms and invariants.  No GPU."""
import numpy as np
import pytest

import oracle
from oracle import backward as ob

RD = (4, 6, 6)                     # D = 16: axis slices t | h | w
SPANS = [(0, oracle.CLEAN, 5), (1, oracle.CLEAN, 4), (1, oracle.NOISY, 6), (2, oracle.NOISY, 3)]


def _inputs(seed=0, H=2, D=16):
    rng = np.random.default_rng(seed)
    n = sum(s[2] for s in SPANS)
    q, k, v, dout = (rng.standard_normal((n, H, D)) for _ in range(4))
    gq, gk = (rng.uniform(0.5, 1.5, (H, D)) for _ in range(2))
    pos = np.stack([rng.integers(0, 9, n), rng.integers(0, 5, n), rng.integers(0, 7, n)], axis=1).astype(np.int32)
    return q, k, v, dout, gq, gk, pos


def _loss(q, k, v, gq, gk, pos, dout, eps=1e-6):
    """L = sum(dO * O) through the C oracle's forward (the function the backward differentiates)."""
    qn = oracle.prologue(q, gq, pos, RD, 10000.0, eps)
    kn = oracle.prologue(k, gk, pos, RD, 10000.0, eps)
    tags = oracle.chunk_tags([c for c, _, _ in SPANS], [kd for _, kd, _ in SPANS], [n for _, _, n in SPANS])
    return float(np.sum(oracle.attention(qn, kn, v, tags, tags) * dout))


@pytest.mark.parametrize("which", ["q", "k", "v", "gq", "gk"])
def test_backward_matches_central_differences(which):
    q, k, v, dout, gq, gk, pos = _inputs(1)
    g = ob.spans_backward(gq, gk, q, k, v, pos, SPANS, dout, RD)
    grad = {"q": g["dq"], "k": g["dk"], "v": g["dv"], "gq": g["dgq"], "gk": g["dgk"]}[which]
    args = {"q": q, "k": k, "v": v, "gq": gq, "gk": gk}
    rng = np.random.default_rng(7)
    for _ in range(3):                              # directional derivatives along random directions
        d = rng.standard_normal(args[which].shape)
        h = 1e-5

        def at(sign):
            a = dict(args)
            a[which] = args[which] + sign * h * d
            return _loss(a["q"], a["k"], a["v"], a["gq"], a["gk"], pos, dout)

        fd = (at(+1) - at(-1)) / (2 * h)
        an = float(np.sum(grad * d))
        assert abs(fd - an) <= 1e-7 * max(1.0, abs(an)), (which, fd, an)


def test_backward_single_coordinates():
    # a handful of single-coordinate derivatives (catches a transposed or misplaced index)
    q, k, v, dout, gq, gk, pos = _inputs(2)
    g = ob.spans_backward(gq, gk, q, k, v, pos, SPANS, dout, RD)
    h = 1e-5
    for arr, grad, idx in ((q, g["dq"], (3, 1, 5)), (k, g["dk"], (10, 0, 15)), (v, g["dv"], (7, 1, 0)),
                           (q, g["dq"], (16, 0, 2)), (k, g["dk"], (0, 1, 9))):
        e = np.zeros_like(arr)
        e[idx] = h
        base = dict(q=q, k=k, v=v)
        name = [n for n, a in base.items() if a is arr][0]
        lp = _loss(**{**base, name: arr + e}, gq=gq, gk=gk, pos=pos, dout=dout)
        lm = _loss(**{**base, name: arr - e}, gq=gq, gk=gk, pos=pos, dout=dout)
        assert abs((lp - lm) / (2 * h) - grad[idx]) <= 1e-7 * max(1.0, abs(grad[idx])), (name, idx)


def test_self_only_layout_closed_form():
    # every query sees only itself (NOISY spans of one token each): P = 1, O = v, so dV = dO and
    # dq' = dk' = 0 (dz = P (dP - delta) = 0)
    rng = np.random.default_rng(3)
    n, H, D = 6, 2, 16
    spans = [(i, oracle.NOISY, 1) for i in range(n)]
    q, k, v, dout = (rng.standard_normal((n, H, D)) for _ in range(4))
    tags = oracle.chunk_tags([c for c, _, _ in spans], [kd for _, kd, _ in spans], [1] * n)
    dq, dk, dv, out, _ = ob.attention_backward(q, k, v, tags, tags, dout)
    assert np.allclose(out, v, atol=1e-15) and np.allclose(dv, dout, atol=1e-15)
    assert np.abs(dq).max() < 1e-15 and np.abs(dk).max() < 1e-15


def test_rmsnorm_gradient_orthogonal_to_input():
    # RMSNorm with eps = 0 is scale-invariant (x^(a x) = x^(x)), so dL/dx is orthogonal to x
    rng = np.random.default_rng(4)
    x = rng.standard_normal((5, 2, 16))
    g = rng.uniform(0.5, 1.5, (2, 16))
    pos = rng.integers(0, 20, (5, 3)).astype(np.int32)
    dxp = rng.standard_normal((5, 2, 16))
    dx, _ = ob.prologue_backward(x, g, pos, dxp, RD, eps=0.0)
    assert np.abs(np.sum(dx * x, axis=-1)).max() < 1e-12


def test_rope_backward_preserves_pair_norms():
    # with unit gains and x of unit RMS the gain and norm steps are identities on dy, so the RoPE
    # backward (a rotation) keeps each pair's norm: |dy pair| = |dx' pair|
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 1, 16))
    x /= np.sqrt(np.mean(x * x, axis=-1, keepdims=True))
    pos = rng.integers(0, 50, (4, 3)).astype(np.int32)
    dxp = rng.standard_normal((4, 1, 16))
    _, dg = ob.prologue_backward(x, np.ones((1, 16)), pos, dxp, RD, eps=0.0)
    # read dy off dg = sum_t dy * x^ with one-token calls whose x^ is a basis vector
    for t in range(4):
        dy_pairs = []
        for i in range(16):
            e = np.zeros((1, 1, 16))
            e[0, 0, i] = 4.0                        # x = 4 e_i: mean(x^2) = 1, so x^ = x and dg_i = 4 dy_i
            _, dgi = ob.prologue_backward(e, np.ones((1, 16)), pos[t:t + 1], dxp[t:t + 1], RD, eps=0.0)
            dy_pairs.append(dgi[0, i] / 4.0)
        dy = np.array(dy_pairs)
        a = dxp[t, 0]
        assert np.allclose(np.hypot(dy[0::2], dy[1::2]), np.hypot(a[0::2], a[1::2]), atol=1e-12)
