"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/dz.h declares, and validates arguments before anything is enqueued."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2602_15922_b200 as dz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dz.h")).read()
    return sorted(set(re.findall(r"DZ_API\s+[\w\s\*]+?\b(dz_\w+)\s*\(", src)))


def test_header_declares_the_four_core_calls():
    syms = header_symbols()
    for s in ("dz_create", "dz_append_kv", "dz_attend_chunk", "dz_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = dz.lib()
    out = subprocess.check_output(["nm", "-D", "--defined-only", dz.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for s in header_symbols():
        assert s in exported, s
        assert getattr(L, s) is not None
    # and the binding declares a signature for each of them
    assert {n for n, _, _ in dz.SIGNATURES} == set(header_symbols())


def test_library_is_sm100a_only():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dz.LIB_PATH], text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _cfg(**kw):
    c = dz.DzConfig()
    c.batch, c.heads, c.head_dim = 1, 4, 128
    for i, d in enumerate((44, 42, 42)):
        c.rope_dims[i] = d
    c.cache_capacity_tokens, c.max_chunk_tokens = 512, 256
    c.q_gain = c.k_gain = 0x10000
    c.max_abs_gain = 1.5
    c.world_size, c.rank = 1, 0
    c.flags = dz.FLAG_HOST_ONLY   # placeholder device pointers: the context never dereferences them
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_cache_bytes_formula():
    c = _cfg()
    n = dz.lib().dz_cache_bytes(ctypes.byref(c))
    slots = 512 + 256
    assert n >= 2 * slots * 4 * 128 * 2 + 256 * 4 * 128 * 2
    bad = _cfg(head_dim=96)
    assert dz.lib().dz_cache_bytes(ctypes.byref(bad)) == 0
    bad = _cfg()
    bad.rope_dims[0] = 43
    assert dz.lib().dz_cache_bytes(ctypes.byref(bad)) == 0


@pytest.mark.parametrize("kw,status", [
    (dict(head_dim=96), -2),
    (dict(heads=5, world_size=2, rank=0, nccl_comm=1), -2),
    (dict(max_abs_gain=1e4), -7),
    (dict(cache_storage=None), -1),
    (dict(world_size=2, rank=0), -1),  # SP without a communicator
])
def test_create_validation(kw, status):
    c = _cfg(**kw)
    if "cache_storage" not in kw:
        c.cache_storage = 0x100000
    c.cache_bytes = 1 << 40
    ctx = ctypes.c_void_p()
    assert dz.lib().dz_create(ctypes.byref(c), ctypes.byref(ctx)) == status
    assert not ctx.value


def test_create_capacity_check():
    c = _cfg()
    c.cache_storage = 0x100000
    c.cache_bytes = 1000
    ctx = ctypes.c_void_p()
    assert dz.lib().dz_create(ctypes.byref(c), ctypes.byref(ctx)) == -3


def test_call_validation_before_enqueue():
    L = dz.lib()
    c = _cfg()
    c.cache_storage = 0x100000
    c.cache_bytes = L.dz_cache_bytes(ctypes.byref(c))
    ctx = ctypes.c_void_p()
    assert L.dz_create(ctypes.byref(c), ctypes.byref(ctx)) == 0
    try:
        pos = 0x200000
        span = dz.DzSpan(0, dz.NOISY, 128, pos)
        # null pointers
        assert L.dz_attend_chunk(ctx, None, 0x300000, 0x300000, ctypes.byref(span), 0x300000, None) == -1
        # misaligned
        assert L.dz_attend_chunk(ctx, 0x300001, 0x300000, 0x300000, ctypes.byref(span), 0x300000, None) == -1
        # chunk too large
        big = dz.DzSpan(0, dz.NOISY, 257, pos)
        assert L.dz_attend_chunk(ctx, 0x300000, 0x300000, 0x300000, ctypes.byref(big), 0x300000, None) == -3
        # bad kind
        bad = dz.DzSpan(0, 7, 128, pos)
        assert L.dz_attend_chunk(ctx, 0x300000, 0x300000, 0x300000, ctypes.byref(bad), 0x300000, None) == -1
        # noisy chunks never enter the cache (Alg. 2 l.603)
        assert L.dz_append_kv(ctx, 0x300000, 0x300000, ctypes.byref(span), None) == -4
        # nothing staged
        assert L.dz_commit_staged(ctx, 0, None) == -4
        # cannot evict what is not there
        assert L.dz_evict_front(ctx, 1, None) == -1
        v, n, last = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        assert L.dz_cache_state(ctx, ctypes.byref(v), ctypes.byref(n), ctypes.byref(last)) == 0
        assert (v.value, n.value, last.value) == (0, 0, -1)
        assert b"chunk" in L.dz_last_error(ctx) or b"evict" in L.dz_last_error(ctx)
    finally:
        assert L.dz_destroy(ctx) == 0


def test_status_strings():
    for s in range(-7, 1):
        assert dz.status_string(s).startswith("DZ_")


def test_host_only_context_validates_then_refuses_to_enqueue():
    L = dz.lib()
    c = _cfg()
    c.cache_storage = 0x100000
    c.cache_bytes = L.dz_cache_bytes(ctypes.byref(c))
    ctx = ctypes.c_void_p()
    assert L.dz_create(ctypes.byref(c), ctypes.byref(ctx)) == 0
    try:
        span = dz.DzSpan(0, dz.NOISY, 128, 0x200000)
        assert L.dz_attend_chunk(ctx, 0x300000, 0x300000, 0x300000, ctypes.byref(span), 0x300000, None) == -4
        assert b"host-only" in L.dz_last_error(ctx)
        clean = dz.DzSpan(0, dz.CLEAN, 128, 0x200000)
        assert L.dz_append_kv(ctx, 0x300000, 0x300000, ctypes.byref(clean), None) == -4
        assert L.dz_cache_state(ctx, None, None, None) == 0
        # nothing pending: dz_sp_pending lists no transfer, dz_sp_resume has nothing to resume
        ph = ctypes.c_int32()
        assert L.dz_sp_pending(ctx, ctypes.byref(ph), None, 0) == 0 and ph.value == -1
        assert L.dz_sp_resume(ctx, None) == -4
    finally:
        L.dz_destroy(ctx)


def test_external_exchange_allows_sp_without_nccl():
    L = dz.lib()
    c = _cfg(world_size=2, rank=1)
    c.flags |= dz.FLAG_EXTERNAL_EXCHANGE
    c.cache_storage = 0x100000
    c.cache_bytes = L.dz_cache_bytes(ctypes.byref(c))
    ctx = ctypes.c_void_p()
    assert L.dz_create(ctypes.byref(c), ctypes.byref(ctx)) == 0
    assert L.dz_sp_plan(ctx, 0, 128, None, 0) == 3 * 2
    L.dz_destroy(ctx)


def test_peer_store_validation():
    # DZ_FLAG_PEER_STORE (NEXT-3): 2..8 ranks, token-loop prologue heads, n / world_size a multiple of 8;
    # compute calls need dz_sp_set_peers first, whose entry `rank` must be the context's own storage
    L = dz.lib()
    bad = _cfg(world_size=1)
    bad.flags |= dz.FLAG_PEER_STORE
    bad.cache_storage, bad.cache_bytes = 0x100000, 1 << 40
    ctx = ctypes.c_void_p()
    assert L.dz_create(ctypes.byref(bad), ctypes.byref(ctx)) == -2
    c = _cfg(world_size=2, rank=1, nccl_comm=1)
    c.flags |= dz.FLAG_PEER_STORE
    c.cache_storage = 0x100000
    c.cache_bytes = L.dz_cache_bytes(ctypes.byref(c))
    assert L.dz_create(ctypes.byref(c), ctypes.byref(ctx)) == 0
    try:
        span = dz.DzSpan(0, dz.NOISY, 128, 0x200000)
        assert L.dz_attend_chunk(ctx, 0x300000, 0x300000, 0x300000, ctypes.byref(span), 0x300000, None) == -4
        peers = (ctypes.c_void_p * 2)(0x200000, 0x100000)
        assert L.dz_sp_set_peers(ctx, peers, 1) == -1              # one entry per rank
        wrong = (ctypes.c_void_p * 2)(0x100000, 0x200000)
        assert L.dz_sp_set_peers(ctx, wrong, 2) == -1              # entry 1 must be this rank's storage
        assert L.dz_sp_set_peers(ctx, peers, 2) == 0
        odd = dz.DzSpan(0, dz.NOISY, 2 * 60, 0x200000)             # 60 tokens per rank: not a multiple of 8
        assert L.dz_attend_chunk(ctx, 0x300000, 0x300000, 0x300000, ctypes.byref(odd), 0x300000, None) == -2
    finally:
        L.dz_destroy(ctx)
