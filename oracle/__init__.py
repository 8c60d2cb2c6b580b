"""fp64 CPU oracle for the DreamZero chunk-attention hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2602_15922_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain C, fp64, OpenMP over
(query, head) rows); this module compiles it with gcc, loads it with ctypes
and composes its steps in the paper's order:

* ``prologue``   -- per-head RMSNorm then 3D RoPE (BJ:5; readings A1-A9).
* ``attention``  -- masked softmax attention under the Fig. 10 rule
                    (Alg. 2 l.558-607).
* ``tile_map``   -- SKIP/PARTIAL/FULL per (q-tile, kv-tile).
* ``attend_chunk`` -- the whole denoise-step path for one batch element:
  committed clean chunks (K' = prologue(K), V as is: the cache append of
  Alg. 2 l.601-602) plus the current noisy chunk, which sees all of them and
  itself (Alg. 2 l.584-585, update=False).

Every function is pinned by ``tests/test_oracle_pins.py``; the backward
(``oracle/backward.py``: gradients of the same path for teacher-forced training,
NEXT-1) by ``tests/test_oracle_backward.py`` against central finite differences of
this forward.  Parity pinned for all functions (no "parity unpinned" entries).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC", "-std=c99"]

CLEAN, NOISY = 0, 1
SKIP, PARTIAL, FULL = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2 -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.oracle_rmsnorm.argtypes = [P, P, I64, I32, I32, D, P]
        L.oracle_rope3d.argtypes = [P, P, I64, I32, I32, P, D]
        L.oracle_prologue.argtypes = [P, P, P, I64, I32, I32, P, D, D, P]
        L.oracle_visible.argtypes = [I32] * 6
        L.oracle_attention.argtypes = [P, P, P, I64, I64, I32, I32, D, P, P, P, P, P, P, P, P]
        L.oracle_tile_map.argtypes = [I64, I64, I32, I32, P, P, P, P, P, P, P]
        for f in (L.oracle_rmsnorm, L.oracle_rope3d, L.oracle_prologue, L.oracle_visible,
                  L.oracle_attention, L.oracle_tile_map, L.oracle_num_threads):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def _f64(x) -> np.ndarray:
    if hasattr(x, "detach"):                       # torch tensor (any dtype) -> fp64
        x = x.detach().cpu().double().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _i32(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what}: invalid arguments (rc={rc})")


def rmsnorm(x, gain, eps: float = 1e-6) -> np.ndarray:
    x, g = _f64(x), _f64(gain)
    n, H, D = x.shape
    out = np.empty_like(x)
    _check(lib().oracle_rmsnorm(_p(x), _p(g), n, H, D, eps, _p(out)), "rmsnorm")
    return out


def rope3d(x, pos, rope_dims: Sequence[int], theta: float = 10000.0) -> np.ndarray:
    out = _f64(x).copy()
    pos = _i32(pos)
    rd = _i32(list(rope_dims))
    n, H, D = out.shape
    _check(lib().oracle_rope3d(_p(out), _p(pos), n, H, D, _p(rd), theta), "rope3d")
    return out


def prologue(x, gain, pos, rope_dims: Sequence[int], theta: float = 10000.0,
             eps: float = 1e-6) -> np.ndarray:
    x, g, pos = _f64(x), _f64(gain), _i32(pos)
    rd = _i32(list(rope_dims))
    n, H, D = x.shape
    out = np.empty_like(x)
    _check(lib().oracle_prologue(_p(x), _p(g), _p(pos), n, H, D, _p(rd), theta, eps, _p(out)),
           "prologue")
    return out


def visible(qc: int, qk: int, qs: int, kc: int, kk: int, ks: int) -> bool:
    return bool(lib().oracle_visible(qc, qk, qs, kc, kk, ks))


def attention(q, k, v, q_tags, k_tags, scale: float | None = None,
              with_lse: bool = False):
    """q [nq,H,D], k/v [nk,H,D] post-prologue; tags = (chunk, kind, span) int32 vectors."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    nq, H, D = q.shape
    nk = k.shape[0]
    if scale is None:
        scale = D ** -0.5
    qt = [_i32(t) for t in q_tags]
    kt = [_i32(t) for t in k_tags]
    out = np.zeros((nq, H, D), dtype=np.float64)
    lse = np.zeros((nq, H), dtype=np.float64)
    _check(lib().oracle_attention(_p(q), _p(k), _p(v), nq, nk, H, D, float(scale),
                                  _p(qt[0]), _p(qt[1]), _p(qt[2]), _p(kt[0]), _p(kt[1]), _p(kt[2]),
                                  _p(out), _p(lse)), "attention")
    return (out, lse) if with_lse else out


def tile_map(q_tags, k_tags, BM: int, BN: int) -> np.ndarray:
    qt = [_i32(t) for t in q_tags]
    kt = [_i32(t) for t in k_tags]
    nq, nk = len(qt[0]), len(kt[0])
    n_qt, n_kt = -(-nq // BM), -(-nk // BN)
    out = np.zeros((n_qt, n_kt), dtype=np.uint8)
    _check(lib().oracle_tile_map(nq, nk, BM, BN, _p(qt[0]), _p(qt[1]), _p(qt[2]),
                                 _p(kt[0]), _p(kt[1]), _p(kt[2]), _p(out)), "tile_map")
    return out


def tile_map_str(m: np.ndarray) -> str:
    return "/".join("".join("SPF"[int(c)] for c in row) for row in m)


def chunk_tags(chunk_ids: Sequence[int], kinds: Sequence[int], sizes: Sequence[int]):
    """Per-token (chunk, kind, span) tags for consecutive spans."""
    ch, kd, sp = [], [], []
    for i, (c, k, n) in enumerate(zip(chunk_ids, kinds, sizes)):
        ch += [c] * n
        kd += [k] * n
        sp += [i] * n
    return (np.asarray(ch, np.int32), np.asarray(kd, np.int32), np.asarray(sp, np.int32))


def append_reference(k_raw, v_raw, gain_k, pos, rope_dims, theta=10000.0, eps=1e-6):
    """Cache append of a clean chunk (Alg. 2 l.601-602): K' = prologue(K), V' = V."""
    return prologue(k_raw, gain_k, pos, rope_dims, theta, eps), _f64(v_raw)


def attend_chunk(gain_q, gain_k, cache_k: List, cache_v: List, cache_pos: List,
                 q, k, v, pos, rope_dims, theta: float = 10000.0, eps: float = 1e-6,
                 scale: float | None = None, with_lse: bool = False):
    """One batch element of one denoise step (Alg. 2 l.584-585, update=False).

    The current chunk (id C = len(cache_k), NOISY) attends to the committed
    clean chunks 0..C-1 and to itself.  Inputs are the raw bf16 values (as
    tensors or arrays); every step runs here in fp64.
    """
    C = len(cache_k)
    ks, vs, tags_sizes = [], [], []
    for c in range(C):
        kc, vc = append_reference(cache_k[c], cache_v[c], gain_k, cache_pos[c], rope_dims, theta, eps)
        ks.append(kc)
        vs.append(vc)
        tags_sizes.append(kc.shape[0])
    qn = prologue(q, gain_q, pos, rope_dims, theta, eps)
    kn = prologue(k, gain_k, pos, rope_dims, theta, eps)
    ks.append(kn)
    vs.append(_f64(v))
    n = qn.shape[0]
    k_tags = chunk_tags(list(range(C)) + [C], [CLEAN] * C + [NOISY], tags_sizes + [n])
    q_tags = (np.full(n, C, np.int32), np.full(n, NOISY, np.int32), np.full(n, C, np.int32))
    return attention(qn, np.concatenate(ks, 0), np.concatenate(vs, 0), q_tags, k_tags,
                     scale, with_lse)
