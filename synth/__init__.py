"""Seeded synthetic workloads for the DreamZero chunk-attention hot path.

This module is the ONE place both sides of the parity check get their inputs
from (the fp64 oracle under ``oracle/`` and the CUDA path under
``paper_2602_15922_b200/``).  It holds none of the method's arithmetic: no
normalisation, no rotation, no softmax.  It only draws seeded Gaussian tensors,
states workload shapes and lays tokens out on the (t, h, w) grid.

Sources
-------
* Shapes and distributions: BASELINE.json ``configs`` C0..C4 (BJ:7-11).
* Token layout: PAPER.md l.94 ("we concatenate all views into a single
  frame"), l.99 (chunks of K latent frames), Fig. 10 / l.505 (video tokens Z
  then action tokens Y inside a chunk).  Readings A8, A9, A11 of DESIGN.md:
  views concatenated along width; video token i of chunk c, frame f, row r,
  column col gets (t, h, w) = (c*K + f, r, col); action tokens get
  (c*K, 0, 0).
* Seeds: DESIGN.md "input recipe":
  seed = 1_000_000*x + 100_000*b + 1000*c + s for config Cx, batch element b,
  chunk c (cache chunks 0..C-1, current chunk C) and denoise step s; the
  tensors Q, K, V are drawn in that order from one ``torch.Generator``.
  C2 adds 1 % raw-K outliers of magnitude 8 (reading A19).  Gains use
  seed 1_000_000*x + 999_000 and U(0.5, 1.5) (C0: all ones).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Dict, List, Tuple

import torch

CLEAN = 0
NOISY = 1


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (BJ:7-11)."""

    name: str
    index: int                 # x in the seed formula
    batch: int
    heads: int
    head_dim: int
    rope_dims: Tuple[int, int, int]
    frames: int                # K latent frames per chunk
    grid_h: int
    grid_w: int                # per-view width
    views: int                 # views concatenated along width
    actions: int               # action tokens per chunk
    cached_chunks: int
    steps: int = 1             # denoise steps over one cache (C3: 4)
    outliers: bool = False     # C2: 1 % of raw K replaced by +-8
    unit_gain: bool = False    # C0: RMSNorm gains all ones
    draw_dtype: str = "bf16"   # C0 is drawn fp32 and cast to bf16 for the GPU (A18)
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6
    max_gpus: int = 1
    notes: str = ""

    @property
    def video_tokens(self) -> int:
        return self.frames * self.grid_h * self.views * self.grid_w

    @property
    def chunk_tokens(self) -> int:
        return self.video_tokens + self.actions

    @property
    def cache_tokens(self) -> int:
        return self.cached_chunks * self.chunk_tokens

    @property
    def kv_tokens(self) -> int:
        return self.cache_tokens + self.chunk_tokens

    @property
    def softmax_scale(self) -> float:
        return self.head_dim ** -0.5

    def useful_flop(self) -> float:
        """4*D per visible (q, k) pair summed over batch and heads."""
        return 4.0 * self.head_dim * self.batch * self.heads * self.chunk_tokens * self.kv_tokens


WORKLOADS: Dict[str, Workload] = {
    "C0": Workload("C0", 0, batch=1, heads=2, head_dim=64, rope_dims=(16, 24, 24), frames=2,
                   grid_h=4, grid_w=7, views=1, actions=8, cached_chunks=2, unit_gain=True,
                   draw_dtype="fp32", notes="tiny, fp32 draws (BJ:7)"),
    "C1": Workload("C1", 1, batch=1, heads=40, head_dim=128, rope_dims=(44, 42, 42), frames=2,
                   grid_h=11, grid_w=20, views=3, actions=24, cached_chunks=4,
                   notes="Wan-14B layer, 4 cached chunks (BJ:8)"),
    "C2": Workload("C2", 2, batch=1, heads=40, head_dim=128, rope_dims=(44, 42, 42), frames=2,
                   grid_h=11, grid_w=20, views=3, actions=24, cached_chunks=16, outliers=True,
                   notes="long cache, K outliers (BJ:9)"),
    "C3": Workload("C3", 3, batch=2, heads=40, head_dim=128, rope_dims=(44, 42, 42), frames=2,
                   grid_h=11, grid_w=20, views=3, actions=24, cached_chunks=8, steps=4,
                   max_gpus=2, notes="CFG batch 2, 4 steps over one cache (BJ:10)"),
    "C4": Workload("C4", 4, batch=1, heads=40, head_dim=128, rope_dims=(44, 42, 42), frames=4,
                   grid_h=11, grid_w=20, views=3, actions=48, cached_chunks=32, max_gpus=8,
                   notes="Ulysses SP, 32 cached chunks of 2688 (BJ:11)"),
}


def workload(name: str) -> Workload:
    return WORKLOADS[name]


def scaled(w: Workload, **kw) -> Workload:
    """A copy of ``w`` with some fields overridden (for small parity cases)."""
    return replace(w, **kw)


# --------------------------------------------------------------------------
# token layout: positions and span tags
# --------------------------------------------------------------------------

def chunk_positions(w: Workload, chunk: int) -> torch.Tensor:
    """int32 [n, 3] (t, h, w) of the tokens of chunk ``chunk`` (readings A8, A9, A11).

    Video tokens first, frame-major, then row-major over the view-concatenated
    grid (grid_h x views*grid_w); then ``actions`` action tokens at (chunk*K, 0, 0).
    """
    K, gh, W = w.frames, w.grid_h, w.views * w.grid_w
    f = torch.arange(K, dtype=torch.int32).view(K, 1, 1).expand(K, gh, W)
    r = torch.arange(gh, dtype=torch.int32).view(1, gh, 1).expand(K, gh, W)
    c = torch.arange(W, dtype=torch.int32).view(1, 1, W).expand(K, gh, W)
    vid = torch.stack([f + chunk * K, r, c], dim=-1).reshape(-1, 3)
    act = torch.zeros(w.actions, 3, dtype=torch.int32)
    act[:, 0] = chunk * K
    return torch.cat([vid, act], dim=0).contiguous()


@dataclass
class Span:
    """A run of tokens with one (chunk id, kind) tag (Fig. 10)."""

    chunk: int
    kind: int          # CLEAN or NOISY
    n_tokens: int


def span_tags(spans: List[Span]) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Per-token (chunk, kind, span index) int32 vectors for a list of spans."""
    ch, kd, sp = [], [], []
    for i, s in enumerate(spans):
        ch += [s.chunk] * s.n_tokens
        kd += [s.kind] * s.n_tokens
        sp += [i] * s.n_tokens
    t = lambda a: torch.tensor(a, dtype=torch.int32)
    return t(ch), t(kd), t(sp)


def teacher_forcing_spans(n_chunks: int, tokens_per_chunk: int) -> List[Span]:
    """Fig. 10(a) training layout [C0 .. C_{M-1}; Z1 .. Z_M]."""
    clean = [Span(c, CLEAN, tokens_per_chunk) for c in range(n_chunks)]
    noisy = [Span(c, NOISY, tokens_per_chunk) for c in range(1, n_chunks + 1)]
    return clean + noisy


# --------------------------------------------------------------------------
# seeded draws
# --------------------------------------------------------------------------

def seed_for(w: Workload, b: int, chunk: int, step: int = 0) -> int:
    return 1_000_000 * w.index + 100_000 * b + 1000 * chunk + step


def draw_qkv(w: Workload, b: int, chunk: int, step: int = 0,
             heads: Tuple[int, int] | None = None,
             raw: bool = False) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Raw Q, K, V of one chunk of batch element ``b`` as bf16 [n, H, D] (CPU).

    Drawn full-size fp32 N(0,1) in the order Q, K, V (then the C2 outlier
    draws), then rounded to bf16 (round-to-nearest-even).  ``heads=(h0, h1)``
    slices the result after drawing, so a slice equals the same heads of the
    full draw.  ``raw=True`` returns the fp32 draws before rounding (C0's
    oracle-vs-brute-force pins run on those, reading A18).
    """
    g = torch.Generator(device="cpu")
    g.manual_seed(seed_for(w, b, chunk, step))
    n, H, D = w.chunk_tokens, w.heads, w.head_dim
    q = torch.randn(n, H, D, generator=g, dtype=torch.float32)
    k = torch.randn(n, H, D, generator=g, dtype=torch.float32)
    v = torch.randn(n, H, D, generator=g, dtype=torch.float32)
    if w.outliers:
        u1 = torch.rand(n, H, D, generator=g, dtype=torch.float32)
        u2 = torch.rand(n, H, D, generator=g, dtype=torch.float32)
        k = torch.where(u1 < 0.01, 8.0 * torch.sign(u2 - 0.5), k)
    out = [x if raw else x.to(torch.bfloat16) for x in (q, k, v)]
    if heads is not None:
        out = [x[:, heads[0]:heads[1]].contiguous() for x in out]
    return out[0], out[1], out[2]


def draw_gains(w: Workload) -> Tuple[torch.Tensor, torch.Tensor]:
    """RMSNorm gains g_q, g_k as fp32 [H, D] (reading A3)."""
    if w.unit_gain:
        one = torch.ones(w.heads, w.head_dim, dtype=torch.float32)
        return one, one.clone()
    g = torch.Generator(device="cpu")
    g.manual_seed(1_000_000 * w.index + 999_000)
    gq = torch.rand(w.heads, w.head_dim, generator=g, dtype=torch.float32) + 0.5
    gk = torch.rand(w.heads, w.head_dim, generator=g, dtype=torch.float32) + 0.5
    return gq, gk


@dataclass
class ChunkStream:
    """All inputs of one batch element: cached chunks and the current chunk's steps."""

    cache_k: List[torch.Tensor] = field(default_factory=list)
    cache_v: List[torch.Tensor] = field(default_factory=list)
    cache_pos: List[torch.Tensor] = field(default_factory=list)
    cur_q: List[torch.Tensor] = field(default_factory=list)   # one per step
    cur_k: List[torch.Tensor] = field(default_factory=list)
    cur_v: List[torch.Tensor] = field(default_factory=list)
    cur_pos: torch.Tensor | None = None


def draw_stream(w: Workload, b: int, heads: Tuple[int, int] | None = None,
                steps: int | None = None) -> ChunkStream:
    s = ChunkStream()
    C = w.cached_chunks
    for c in range(C):
        _, k, v = draw_qkv(w, b, c, 0, heads)
        s.cache_k.append(k)
        s.cache_v.append(v)
        s.cache_pos.append(chunk_positions(w, c))
    for st in range(w.steps if steps is None else steps):
        q, k, v = draw_qkv(w, b, C, st, heads)
        s.cur_q.append(q)
        s.cur_k.append(k)
        s.cur_v.append(v)
    s.cur_pos = chunk_positions(w, C)
    return s


def span_inputs(w: Workload, spans: List[Span], b: int = 0):
    """Raw bf16 Q, K, V [n_total, H, D] and int32 positions [n_total, 3] for a
    list of spans laid out consecutively (the general Fig. 10 form).

    Span i of chunk c and kind k draws its own seeded tensors (seed
    ``seed_for(w, b, c, 100 + k)``, Q, K, V in that order, N(0, 1) -> bf16; C2
    outliers as in ``draw_qkv``) and takes the first n positions of chunk c's
    layout, cycling when n exceeds a chunk.
    """
    qs, ks, vs, ps = [], [], [], []
    H, D = w.heads, w.head_dim
    for s in spans:
        g = torch.Generator(device="cpu")
        g.manual_seed(seed_for(w, b, s.chunk, 100 + s.kind))
        n = s.n_tokens
        q = torch.randn(n, H, D, generator=g, dtype=torch.float32)
        k = torch.randn(n, H, D, generator=g, dtype=torch.float32)
        v = torch.randn(n, H, D, generator=g, dtype=torch.float32)
        if w.outliers:
            u1 = torch.rand(n, H, D, generator=g, dtype=torch.float32)
            u2 = torch.rand(n, H, D, generator=g, dtype=torch.float32)
            k = torch.where(u1 < 0.01, 8.0 * torch.sign(u2 - 0.5), k)
        qs.append(q.to(torch.bfloat16))
        ks.append(k.to(torch.bfloat16))
        vs.append(v.to(torch.bfloat16))
        cp = chunk_positions(w, s.chunk)
        ps.append(cp[torch.arange(n) % cp.shape[0]])
    cat = lambda xs: torch.cat(xs, 0).contiguous()
    return cat(qs), cat(ks), cat(vs), cat(ps)
