"""paper_2602_15922_b200 -- B200-native block-causal chunk attention (DreamZero, arXiv 2602.15922).

A thin ctypes binding over ``libdz.so`` (C ABI: ``include/dz.h``).  Every step
of the hot path -- the fused RMSNorm + 3D RoPE prologue, the tcgen05 flash
attention over the KV cache, the cache append and the Ulysses exchange -- runs
inside the library.  This module only marshals arguments: it checks dtypes,
shapes and devices, passes ``data_ptr()`` values and the current torch CUDA
stream, and owns the device buffers (PyTorch is used for memory, streams and
process groups only).  There is no CPU fallback: if ``libdz.so`` is missing or
was built for another architecture, importing :func:`lib` raises.

Paper mapping: ``ChunkKVCache.append`` is the update=True cache
write of Alg. 2 (l.569-570, l.601-602); ``ChunkKVCache.attend`` is one
denoising step's self-attention, update=False (l.584-585), under the Fig. 10
mask (l.502-507).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

__all__ = ["DzError", "lib", "ChunkKVCache", "CLEAN", "NOISY", "FLAG_WRITE_LSE", "nccl_unique_id",
           "nccl_comm_init", "nccl_comm_destroy", "status_string"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DZ_LIB_PATH") or os.path.join(_HERE, "libdz.so")  # override: A/B diagnostics only

CLEAN, NOISY = 0, 1
FLAG_WRITE_LSE = 1
FLAG_PROFILE = 2
FLAG_ONLINE_SOFTMAX = 4
FLAG_TILE_MAP = 8
FLAG_EXTERNAL_EXCHANGE = 16
FLAG_WHOLE_UNITS = 32
FLAG_HOST_ONLY = 64
FLAG_PEER_STORE = 128
FLAG_FP8_QK = 256
FLAG_BACKWARD = 512

STATUS = {0: "DZ_OK", -1: "DZ_EINVAL", -2: "DZ_ESHAPE", -3: "DZ_ECAPACITY", -4: "DZ_ESTATE",
          -5: "DZ_ECUDA", -6: "DZ_ENCCL", -7: "DZ_ERANGE"}


class DzError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class DzConfig(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32), ("heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
        ("rope_dims", ctypes.c_int32 * 3),
        ("rope_theta", ctypes.c_float), ("rms_eps", ctypes.c_float), ("softmax_scale", ctypes.c_float),
        ("cache_capacity_tokens", ctypes.c_int64), ("max_chunk_tokens", ctypes.c_int32),
        ("window_slack_tokens", ctypes.c_int32),
        ("q_gain", ctypes.c_void_p), ("k_gain", ctypes.c_void_p), ("max_abs_gain", ctypes.c_float),
        ("cache_storage", ctypes.c_void_p), ("cache_bytes", ctypes.c_size_t),
        ("nccl_comm", ctypes.c_void_p), ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class DzXfer(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("tensor", ctypes.c_int32), ("send_off", ctypes.c_int64),
                ("recv_off", ctypes.c_int64), ("bytes", ctypes.c_int64)]


class DzSpan(ctypes.Structure):
    _fields_ = [("chunk_id", ctypes.c_int32), ("kind", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
                ("pos_thw", ctypes.c_void_p)]


# every entry point declared in include/dz.h: (name, restype, argtypes)
P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
SIGNATURES = [
    ("dz_cache_bytes", SZ, [ctypes.POINTER(DzConfig)]),
    ("dz_create", I32, [ctypes.POINTER(DzConfig), ctypes.POINTER(P)]),
    ("dz_append_kv", I32, [P, P, P, ctypes.POINTER(DzSpan), P]),
    ("dz_attend_chunk", I32, [P, P, P, P, ctypes.POINTER(DzSpan), P, P]),
    ("dz_attend_spans", I32, [P, P, P, P, P, ctypes.POINTER(DzSpan), I32, P, P]),
    ("dz_append_attend", I32, [P, P, P, ctypes.POINTER(DzSpan), P, P, P, ctypes.POINTER(DzSpan), P, P]),
    ("dz_commit_staged", I32, [P, I32, P]),
    ("dz_attend_spans_backward", I32, [P, P, P, P, P, ctypes.POINTER(DzSpan), I32, P, P, P, P, P, P, P, P, P]),
    ("dz_evict_front", I32, [P, I32, P]),
    ("dz_cache_state", I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I32), ctypes.POINTER(I32)]),
    ("dz_cache_view", I32, [P, I32, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(I64)]),
    ("dz_copy_lse", I32, [P, P, SZ, P]),
    ("dz_get_tile_map", I32, [P, P, SZ, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32),
                              ctypes.POINTER(I32)]),
    ("dz_destroy", I32, [P]),
    ("dz_status_string", ctypes.c_char_p, [I32]),
    ("dz_last_error", ctypes.c_char_p, [P]),
    ("dz_nccl_unique_id", I32, [P]),
    ("dz_nccl_comm_init", I32, [I32, P, I32, ctypes.POINTER(P)]),
    ("dz_nccl_comm_destroy", I32, [P]),
    ("dz_attention_units", I32, [P, I32]),
    ("dz_sp_plan", I32, [P, I32, I32, ctypes.POINTER(DzXfer), I32]),
    ("dz_sp_pending", I32, [P, ctypes.POINTER(I32), ctypes.POINTER(DzXfer), I32]),
    ("dz_sp_resume", I32, [P, P]),
    ("dz_sp_set_peers", I32, [P, P, I32]),
    ("dz_debug_sp_unpack", I32, [P, P, I32, I32, I32, I32, I32, P]),
    ("dz_debug_watchdog", I32, [P, I32]),
    ("dz_profile_last", I32, [P, P]),
    ("dz_profile_enable", I32, [P, I32]),
    ("dz_debug_trace", I32, [I32, P, SZ]),
    ("dz_kernel_launches", I64, []),
    ("dz_debug_l2_discard", I32, [P, SZ, P]),
    ("dz_debug_k2_clock", I32, [P, I32]),
]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libdz.so (built by ``python -m paper_2602_15922_b200.build``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2602_15922_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            if os.environ.get("DZ_LIB_PATH") and not hasattr(L, name):
                continue  # an older library under A/B comparison
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def status_string(s: int) -> str:
    return lib().dz_status_string(s).decode()


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need(t: torch.Tensor, name: str, dtype: torch.dtype, shape: Sequence[int], device: torch.device):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def kernel_launches() -> int:
    """Kernels the library has enqueued in this process (host-side count at launch)."""
    return int(lib().dz_kernel_launches())


def k2_clock(reset: bool = False):
    """(SM cycles, ns) summed over attention CTAs since the last reset (dz_debug_k2_clock)."""
    buf = (ctypes.c_uint64 * 2)()
    s = lib().dz_debug_k2_clock(ctypes.cast(buf, ctypes.c_void_p), 1 if reset else 0)
    if s:
        raise DzError(s, "dz_debug_k2_clock")
    return int(buf[0]), int(buf[1])


def l2_discard(buf) -> None:
    """Benchmark helper: drop a device tensor's L2 lines without write-back (dz_debug_l2_discard)."""
    import torch
    nbytes = buf.numel() * buf.element_size() // 128 * 128
    s = lib().dz_debug_l2_discard(ctypes.c_void_p(buf.data_ptr()), nbytes,
                                  ctypes.c_void_p(torch.cuda.current_stream(buf.device).cuda_stream))
    if s:
        raise DzError(s, "dz_debug_l2_discard")


def watchdog(reset: bool = True):
    """The attention kernel's hang record: (fired, block, warp, bar addr, parity, smid, bars base, 0)."""
    buf = (ctypes.c_uint32 * 8)()
    s = lib().dz_debug_watchdog(ctypes.cast(buf, P), int(reset))
    if s:
        raise DzError(s, "dz_debug_watchdog")
    return list(buf)


def debug_trace(enable: bool, read: bool = False) -> Optional[np.ndarray]:
    """Toggle / read the attention kernel's traces: uint32 [8192] cycle trace of CTA 0, then
    [160][64] per-CTA timeline (globaltimer ns); see dz.h and attention.cu."""
    n = 8192 + 160 * 64
    buf = np.zeros(n, dtype=np.uint32) if read else None
    s = lib().dz_debug_trace(int(enable), buf.ctypes.data if read else None, n if read else 0)
    if s:
        raise DzError(s, "dz_debug_trace")
    return buf


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    s = lib().dz_nccl_unique_id(ctypes.cast(buf, P))
    if s:
        raise DzError(s, "ncclGetUniqueId failed")
    return buf.raw


def nccl_comm_init(world_size: int, uid: bytes, rank: int) -> int:
    buf = ctypes.create_string_buffer(uid, 128)
    comm = P()
    s = lib().dz_nccl_comm_init(world_size, ctypes.cast(buf, P), rank, ctypes.byref(comm))
    if s:
        raise DzError(s, "ncclCommInitRank failed")
    return comm.value


def nccl_comm_destroy(comm: int):
    lib().dz_nccl_comm_destroy(comm)


class ChunkKVCache:
    """One layer's KV cache of clean chunks plus the chunk-attention step.

    Shapes: activations bf16 ``[batch, n_local, heads, head_dim]``; positions
    int32 ``[n_local, 3]`` (t, h, w); gains fp32 ``[heads, head_dim]``.
    ``world_size > 1`` shards the sequence Ulysses-style over ranks (needs an
    NCCL communicator from :func:`nccl_comm_init`).
    """

    def __init__(self, batch: int, heads: int, head_dim: int, capacity: int, max_chunk: int,
                 rope_dims: Sequence[int], q_gain: torch.Tensor, k_gain: torch.Tensor,
                 rope_theta: float = 10000.0, rms_eps: float = 1e-6, softmax_scale: float = 0.0,
                 window_slack: int = 0, world_size: int = 1, rank: int = 0, nccl_comm: int = 0,
                 flags: int = 0, device: Optional[torch.device] = None):
        L = lib()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.type != "cuda":
            raise ValueError(f"ChunkKVCache needs a CUDA device, got {dev} (there is no CPU path)")
        self.device = dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())
        self.batch, self.heads, self.head_dim = batch, heads, head_dim
        self.world_size, self.rank = world_size, rank
        self.heads_local = heads // world_size
        _need(q_gain, "q_gain", torch.float32, (heads, head_dim), self.device)
        _need(k_gain, "k_gain", torch.float32, (heads, head_dim), self.device)
        self.q_gain, self.k_gain = q_gain, k_gain
        cfg = DzConfig()
        cfg.batch, cfg.heads, cfg.head_dim = batch, heads, head_dim
        for i in range(3):
            cfg.rope_dims[i] = int(rope_dims[i])
        cfg.rope_theta, cfg.rms_eps, cfg.softmax_scale = rope_theta, rms_eps, softmax_scale
        cfg.cache_capacity_tokens, cfg.max_chunk_tokens = capacity, max_chunk
        cfg.window_slack_tokens = window_slack
        cfg.q_gain, cfg.k_gain = q_gain.data_ptr(), k_gain.data_ptr()
        cfg.max_abs_gain = 0.0   # dz_create reads the gains and derives the bound itself
        cfg.nccl_comm = nccl_comm or None
        cfg.world_size, cfg.rank, cfg.flags = world_size, rank, flags
        nbytes = L.dz_cache_bytes(ctypes.byref(cfg))
        if nbytes == 0:
            raise DzError(-2, "invalid configuration")
        self.storage = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        cfg.cache_storage, cfg.cache_bytes = self.storage.data_ptr(), nbytes
        self._cfg = cfg
        ctx = P()
        s = L.dz_create(ctypes.byref(cfg), ctypes.byref(ctx))
        if s:
            raise DzError(s, "dz_create")
        self._ctx = ctx

    # -- helpers -----------------------------------------------------------
    def _check(self, s: int, what: str):
        if s:
            raise DzError(s, f"{what}: {lib().dz_last_error(self._ctx).decode()}")

    def _span(self, chunk_id: int, kind: int, n_local: int, pos: torch.Tensor) -> DzSpan:
        _need(pos, "pos", torch.int32, (n_local, 3), self.device)
        return DzSpan(chunk_id, kind, n_local * self.world_size, pos.data_ptr())

    def _act(self, t: torch.Tensor, name: str, n_local: int):
        _need(t, name, torch.bfloat16, (self.batch, n_local, self.heads, self.head_dim), self.device)

    # -- the hot path --------------------------------------------------------
    def append(self, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, chunk_id: int,
               stream: Optional[torch.cuda.Stream] = None):
        """Cache append of a clean chunk (Alg. 2 update=True): K' = RoPE(RMSNorm(k)), V = v."""
        n_local = k.shape[1]
        self._act(k, "k", n_local)
        self._act(v, "v", n_local)
        span = self._span(chunk_id, CLEAN, n_local, pos)
        self._check(lib().dz_append_kv(self._ctx, k.data_ptr(), v.data_ptr(), ctypes.byref(span),
                                       _stream_ptr(stream)), "dz_append_kv")

    def attend(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, chunk_id: int,
               kind: int = NOISY, out: Optional[torch.Tensor] = None,
               stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """One denoising step's self-attention of chunk ``chunk_id`` over the cache and itself."""
        n_local = q.shape[1]
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            self._act(t, nm, n_local)
        if out is None:
            out = torch.empty_like(q)
        else:
            self._act(out, "out", n_local)
        span = self._span(chunk_id, kind, n_local, pos)
        self._check(lib().dz_attend_chunk(self._ctx, q.data_ptr(), k.data_ptr(), v.data_ptr(), ctypes.byref(span),
                                          out.data_ptr(), _stream_ptr(stream)), "dz_attend_chunk")
        return out

    def append_attend(self, k_gt: torch.Tensor, v_gt: torch.Tensor, pos_gt: torch.Tensor, gt_chunk_id: int,
                      q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor, chunk_id: int,
                      kind: int = NOISY, out: Optional[torch.Tensor] = None,
                      stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Append the ground-truth chunk ``gt_chunk_id`` then attend chunk ``chunk_id`` (Alg. 2's cache update
        followed by the next chunk's denoising step) -- the same as ``append`` then ``attend``, with both
        prologues in one kernel launch on one GPU."""
        n_gt = k_gt.shape[1]
        self._act(k_gt, "k_gt", n_gt)
        self._act(v_gt, "v_gt", n_gt)
        n_local = q.shape[1]
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            self._act(t, nm, n_local)
        if out is None:
            out = torch.empty_like(q)
        else:
            self._act(out, "out", n_local)
        gspan = self._span(gt_chunk_id, CLEAN, n_gt, pos_gt)
        span = self._span(chunk_id, kind, n_local, pos)
        self._check(lib().dz_append_attend(self._ctx, k_gt.data_ptr(), v_gt.data_ptr(), ctypes.byref(gspan),
                                           q.data_ptr(), k.data_ptr(), v.data_ptr(), ctypes.byref(span),
                                           out.data_ptr(), _stream_ptr(stream)), "dz_append_attend")
        return out

    def attend_spans(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, pos: torch.Tensor,
                     spans: Sequence[Tuple[int, int, int]], out: Optional[torch.Tensor] = None,
                     stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Fig. 10 general form: the new tokens are consecutive spans ``(chunk_id, kind, n_tokens)``
        (global token counts); queries = new tokens, keys = committed chunks + new tokens."""
        n_local = q.shape[1]
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            self._act(t, nm, n_local)
        _need(pos, "pos", torch.int32, (n_local, 3), self.device)
        if out is None:
            out = torch.empty_like(q)
        else:
            self._act(out, "out", n_local)
        arr = (DzSpan * len(spans))(*[DzSpan(int(c), int(kd), int(n), None) for c, kd, n in spans])
        self._check(lib().dz_attend_spans(self._ctx, q.data_ptr(), k.data_ptr(), v.data_ptr(), pos.data_ptr(), arr,
                                          len(spans), out.data_ptr(), _stream_ptr(stream)), "dz_attend_spans")
        return out

    # -- caller-driven exchange (FLAG_EXTERNAL_EXCHANGE) ------------------------
    def sp_pending(self):
        """(phase, [(peer, tensor, send_off, recv_off, bytes), ...]) of the exchange the last call
        stopped at; phase -1 and [] if none (offsets are into ``self.storage``)."""
        ph = I32()
        cnt = lib().dz_sp_pending(self._ctx, ctypes.byref(ph), None, 0)
        if cnt < 0:
            raise DzError(cnt, "dz_sp_pending")
        arr = (DzXfer * max(cnt, 1))()
        lib().dz_sp_pending(self._ctx, ctypes.byref(ph), arr, cnt)
        return ph.value, [(x.peer, x.tensor, x.send_off, x.recv_off, x.bytes) for x in arr[:cnt]]

    def set_peers(self, storages: Sequence[int]):
        """FLAG_PEER_STORE: every rank's storage base address (as mapped in this process), by rank."""
        arr = (P * len(storages))(*[int(x) for x in storages])
        self._check(lib().dz_sp_set_peers(self._ctx, arr, len(storages)), "dz_sp_set_peers")

    def sp_resume(self, stream: Optional[torch.cuda.Stream] = None):
        """Continue the suspended call after its pending transfers have been delivered."""
        self._check(lib().dz_sp_resume(self._ctx, _stream_ptr(stream)), "dz_sp_resume")

    def attend_spans_backward(self, q, k, v, pos, spans, out, lse, dout, stream=None):
        """Gradients of sum(dout * out) for a teacher-forced span layout (FLAG_BACKWARD, empty cache):
        returns (dq, dk, dv) bf16 like q and (dq_gain, dk_gain) fp32 [heads, head_dim]."""
        n_local = q.shape[1]
        for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out"), (dout, "dout")):
            self._act(t, nm, n_local)
        _need(pos, "pos", torch.int32, (n_local, 3), self.device)
        _need(lse, "lse", torch.float32, (self.batch, self.heads_local, n_local), self.device)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        dgq = torch.empty(self.heads, self.head_dim, dtype=torch.float32, device=self.device)
        dgk = torch.empty_like(dgq)
        arr = (DzSpan * len(spans))(*[DzSpan(int(c), int(kd), int(nn), None) for c, kd, nn in spans])
        self._check(lib().dz_attend_spans_backward(self._ctx, q.data_ptr(), k.data_ptr(), v.data_ptr(), pos.data_ptr(),
                                                   arr, len(spans), out.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                                                   dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dgq.data_ptr(),
                                                   dgk.data_ptr(), _stream_ptr(stream)), "dz_attend_spans_backward")
        return dq, dk, dv, dgq, dgk

    def commit_staged(self, chunk_id: int, stream: Optional[torch.cuda.Stream] = None):
        self._check(lib().dz_commit_staged(self._ctx, chunk_id, _stream_ptr(stream)), "dz_commit_staged")

    def evict_front(self, n_chunks: int, stream: Optional[torch.cuda.Stream] = None):
        self._check(lib().dz_evict_front(self._ctx, n_chunks, _stream_ptr(stream)), "dz_evict_front")

    # -- introspection ---------------------------------------------------------
    def state(self) -> Tuple[int, int, int]:
        v, n, last = I64(), I32(), I32()
        self._check(lib().dz_cache_state(self._ctx, ctypes.byref(v), ctypes.byref(n), ctypes.byref(last)),
                    "dz_cache_state")
        return v.value, n.value, last.value

    def cache_view(self, b: int = 0, tokens: Optional[int] = None) -> Tuple[torch.Tensor, torch.Tensor]:
        """(K' fp16, V bf16) views [tokens, heads_local, head_dim] of batch element b, committed slots first."""
        k0, v0, stride = P(), P(), I64()
        self._check(lib().dz_cache_view(self._ctx, b, ctypes.byref(k0), ctypes.byref(v0), ctypes.byref(stride)),
                    "dz_cache_view")
        if tokens is None:
            tokens = self.state()[0]
        base = self.storage.data_ptr()

        def view(ptr, dt, es):
            off = ptr - base
            return self.storage[off:off + tokens * stride.value * es].view(dt).view(tokens, self.heads_local,
                                                                                self.head_dim)
        fp8 = bool(self._cfg.flags & FLAG_FP8_QK)
        return (view(k0.value, torch.float8_e4m3fn if fp8 else torch.float16, 1 if fp8 else 2),
                view(v0.value, torch.bfloat16, 2))

    def tile_map(self, with_tiles: bool = False):
        """The kernel's tile decisions of the last attend for (b, h) = (0, 0) (needs FLAG_TILE_MAP):
        uint8 [query tiles][key steps], 0 SKIP / 1 PARTIAL / 2 FULL; with_tiles: (map, bm, bn)."""
        nq, nk, bm, bn = I32(), I32(), I32(), I32()
        self._check(lib().dz_get_tile_map(self._ctx, None, 0, ctypes.byref(nq), ctypes.byref(nk),
                                          ctypes.byref(bm), ctypes.byref(bn)), "dz_get_tile_map")
        buf = np.zeros((nq.value, nk.value), dtype=np.uint8)
        self._check(lib().dz_get_tile_map(self._ctx, buf.ctypes.data, buf.size, ctypes.byref(nq),
                                          ctypes.byref(nk), ctypes.byref(bm), ctypes.byref(bn)),
                    "dz_get_tile_map")
        return (buf, bm.value, bn.value) if with_tiles else buf

    def lse(self, n: int, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        out = torch.empty(self.batch, self.heads_local, n, dtype=torch.float32, device=self.device)
        self._check(lib().dz_copy_lse(self._ctx, out.data_ptr(), out.numel(), _stream_ptr(stream)), "dz_copy_lse")
        return out

    def profile_last(self) -> dict:
        """Device ms of the last attend/append phases (needs FLAG_PROFILE); host-syncs."""
        buf = (ctypes.c_float * 6)()
        self._check(lib().dz_profile_last(self._ctx, ctypes.cast(buf, P)), "dz_profile_last")
        keys = ("prologue", "exchange_pre", "attention", "exchange_post", "attend_total", "append")
        return dict(zip(keys, list(buf)))

    def profile_enable(self, on: bool):
        """Record per-kernel events (FLAG_PROFILE) or not (kernels then overlap programmatically)."""
        self._check(lib().dz_profile_enable(self._ctx, 1 if on else 0), "dz_profile_enable")

    def attention_units(self, n_tokens: int) -> int:
        return int(lib().dz_attention_units(self._ctx, n_tokens))

    def close(self):
        if getattr(self, "_ctx", None):
            lib().dz_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
