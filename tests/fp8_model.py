"""Numerics model of the FP8 (E4M3) QK^T variant (DZ_FLAG_FP8_QK) -- test
infrastructure.

The variant stores Q' * (scale * log2e) * 2^a and K' * 2^-a as E4M3 (round to nearest even, satfinite)
and computes everything else as the bf16 path.  This model applies exactly that quantization to the
fp64 oracle's Q' and K' and then runs the oracle's exact attention: it is the attention the variant
approximates to within the bf16 path's error.  The exponent a follows dz.h: a = round(log2(bk / bq) / 2)
with bq = sqrt(D) G scale log2e, bk = sqrt(D) G, G = max |gain|.
"""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle

LOG2E = 1.4426950408889634


def e4m3(x: np.ndarray) -> np.ndarray:
    """Round to nearest-even E4M3 (finite range +-448) and back to fp64."""
    assert np.abs(x).max() <= 448.0
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.float8_e4m3fn).to(torch.float64).numpy()


def exponent(head_dim: int, gmax: float, scale: float) -> int:
    bq = math.sqrt(head_dim) * gmax * scale * LOG2E
    bk = math.sqrt(head_dim) * gmax
    return int(round(0.5 * math.log2(bk / bq)))


def quantized_qk(qn: np.ndarray, kn: np.ndarray, a: int, scale: float):
    """(q, k) for oracle.attention(..., scale) whose scores are those of the E4M3 operands."""
    q8 = e4m3(qn * (scale * LOG2E) * 2.0 ** a)
    k8 = e4m3(kn * 2.0 ** -a)
    return q8 * 2.0 ** -a / (scale * LOG2E), k8 * 2.0 ** a


def attend_chunk_fp8(gq, gk, cache_k, cache_v, cache_pos, q, k, v, pos, rope_dims, theta=10000.0, eps=1e-6):
    """oracle.attend_chunk with the variant's E4M3 rounding of Q' and K' (one batch element)."""
    D = q.shape[-1]
    scale = D ** -0.5
    gmax = float(max(np.abs(np.asarray(gq)).max(), np.abs(np.asarray(gk)).max()))
    a = exponent(D, gmax, scale)
    C = len(cache_k)
    ks = [oracle.prologue(kc, gk, pc, rope_dims, theta, eps) for kc, pc in zip(cache_k, cache_pos)]
    ks.append(oracle.prologue(k, gk, pos, rope_dims, theta, eps))
    vs = [oracle._f64(vc) for vc in cache_v] + [oracle._f64(v)]
    qn = oracle.prologue(q, gq, pos, rope_dims, theta, eps)
    qm, km = quantized_qk(qn, np.concatenate(ks), a, scale)
    n = qn.shape[0]
    kt = oracle.chunk_tags(list(range(C)) + [C], [oracle.CLEAN] * C + [oracle.NOISY], [x.shape[0] for x in ks])
    qt = (np.full(n, C, np.int32), np.full(n, oracle.NOISY, np.int32), np.full(n, C, np.int32))
    return oracle.attention(qm, km, np.concatenate(vs), qt, kt, scale)
