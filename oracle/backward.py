"""fp64 backward of the hot path -- TEST INFRASTRUCTURE (same rules as oracle/__init__.py: only tests/
may import it; it shares no code with paper_2602_15922_b200/).

The gradient of L = sum(dO * O) for the forward that ``oracle`` computes -- per-head RMSNorm with
gains, 3D RoPE, Fig. 10-masked softmax attention (the "trajectory-level
updates" of teacher-forced training, l.115-119, Alg. 1 l.512-553) -- written out from the chain
rule, step by step in the forward's order, reversed:

  forward:   x^ = x / r,  r = sqrt(mean_i x_i^2 + eps)          (RMSNorm, reading A2)
             y  = x^ * g                                        (gain, reading A3)
             x' = R(p) y        (RoPE: per pair (2i, 2i+1) of an axis slice, rotation by p_a w_i)
             z_sj = <q'_s, k'_j> * scale over visible j,  P = softmax_j(z),  O = P V
  backward:  dP = dO V^T;  dz = P * (dP - delta),  delta_s = sum_j P_sj dP_sj (= <dO_s, O_s>)
             dq' = scale dz k';  dk' = scale dz^T q';  dV = P^T dO
             dy = R(p)^T dx' = R(-p) dx'   (a rotation's transpose is its inverse)
             dg = sum over tokens of dy * x^;   dx^ = dy * g
             dx = (dx^ - x^ * mean_i(dx^_i x^_i)) / r

Pinned by tests/test_oracle_backward.py against central finite differences of the C oracle's forward
(oracle.prologue / oracle.attention) on small inputs, not against these formulas themselves.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np

import oracle


def _rope_angles(pos: np.ndarray, rope_dims: Sequence[int], theta: float) -> np.ndarray:
    """phi[n][D/2]: the rotation angle of each pair (slices t | h | w, omega_i = theta^(-2i/d_a))."""
    cols = []
    for ax, d in enumerate(rope_dims):
        i = np.arange(d // 2, dtype=np.float64)
        omega = theta ** (-2.0 * i / d)
        cols.append(pos[:, ax:ax + 1].astype(np.float64) * omega[None, :])
    return np.concatenate(cols, axis=1)


def prologue_backward(x, gain, pos, dxp, rope_dims, theta=10000.0, eps=1e-6):
    """Given x [n][H][D] (raw), gain [H][D], positions [n][3] and dx' = dL/dx' [n][H][D]:
    returns (dx [n][H][D], dgain [H][D]), all fp64."""
    x = oracle._f64(x)
    g = oracle._f64(gain)
    dxp = oracle._f64(dxp)
    pos = oracle._i32(pos)
    n, H, D = x.shape
    r = np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)      # [n][H][1]
    xh = x / r
    phi = _rope_angles(pos, rope_dims, theta)[:, None, :]          # [n][1][D/2]
    c, s = np.cos(phi), np.sin(phi)
    a, b = dxp[..., 0::2], dxp[..., 1::2]
    dy = np.empty_like(dxp)                                        # R(-phi) applied to (a, b)
    dy[..., 0::2] = a * c + b * s
    dy[..., 1::2] = -a * s + b * c
    dgain = np.sum(dy * xh, axis=0)
    dxh = dy * g[None]
    dx = (dxh - xh * np.mean(dxh * xh, axis=-1, keepdims=True)) / r
    return dx, dgain


def attention_backward(qn, kn, v, q_tags, k_tags, dout, scale=None):
    """Given the post-prologue q' [nq][H][D], k' [nk][H][D], v [nk][H][D], the Fig. 10 tags and
    dO [nq][H][D]: returns (dq', dk', dv, O, lse), fp64.  Plain definition per (head, query row)."""
    qn, kn, v, dout = (oracle._f64(t) for t in (qn, kn, v, dout))
    nq, H, D = qn.shape
    nk = kn.shape[0]
    if scale is None:
        scale = D ** -0.5
    # the oracle's own visibility rule (oracle.visible), evaluated once per distinct pair of
    # (chunk, kind, span) tags and broadcast to the tokens carrying them
    qtag = np.stack([oracle._i32(t) for t in q_tags], axis=1)
    ktag = np.stack([oracle._i32(t) for t in k_tags], axis=1)
    uq, qi = np.unique(qtag, axis=0, return_inverse=True)
    uk, ki = np.unique(ktag, axis=0, return_inverse=True)
    table = np.array([[oracle.visible(*map(int, a), *map(int, b)) for b in uk] for a in uq], dtype=bool)
    vis = table[qi.reshape(-1)][:, ki.reshape(-1)]
    dq, dk, dv = np.zeros_like(qn), np.zeros_like(kn), np.zeros_like(v)
    out = np.zeros_like(qn)
    lse = np.zeros((nq, H))
    for h in range(H):
        z = (qn[:, h] @ kn[:, h].T) * scale
        z = np.where(vis, z, -np.inf)
        m = z.max(axis=1, keepdims=True)
        e = np.exp(z - m)
        den = e.sum(axis=1, keepdims=True)
        p = e / den
        out[:, h] = p @ v[:, h]
        lse[:, h] = (m + np.log(den))[:, 0]
        dp = dout[:, h] @ v[:, h].T
        delta = np.sum(p * dp, axis=1, keepdims=True)
        dz = p * (dp - delta)
        dq[:, h] = scale * dz @ kn[:, h]
        dk[:, h] = scale * dz.T @ qn[:, h]
        dv[:, h] = p.T @ dout[:, h]
    return dq, dk, dv, out, lse


def spans_backward(gq, gk, q, k, v, pos, spans, dout, rope_dims, theta=10000.0, eps=1e-6, scale=None):
    """The whole path for one batch element of a span layout with an empty cache (teacher forcing,
    Fig. 10(a)): spans = [(chunk, kind, n_tokens)].  Returns dict(dq, dk, dv, dgq, dgk, out, lse)."""
    qn = oracle.prologue(q, gq, pos, rope_dims, theta, eps)
    kn = oracle.prologue(k, gk, pos, rope_dims, theta, eps)
    tags = oracle.chunk_tags([c for c, _, _ in spans], [kd for _, kd, _ in spans], [n for _, _, n in spans])
    dqn, dkn, dv, out, lse = attention_backward(qn, kn, v, tags, tags, dout, scale)
    dq, dgq = prologue_backward(q, gq, pos, dqn, rope_dims, theta, eps)
    dk, dgk = prologue_backward(k, gk, pos, dkn, rope_dims, theta, eps)
    return {"dq": dq, "dk": dk, "dv": dv, "dgq": dgq, "dgk": dgk, "out": out, "lse": lse}
