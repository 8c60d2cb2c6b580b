"""Ulysses sequence-parallel exchange (BASELINE.json C4) on CPU.

The library's exchange plan (dz_sp_plan -- the same entries it issues as one
grouped ncclSend/ncclRecv each) is executed here with torch.distributed's
gloo backend between world_size CPU processes, on byte buffers standing in for
each rank's cache storage.  Checks, for every rank:
  * pre-exchange: the sequence shard [B, n/N, H, D] of Q', K', V becomes the head
    shard [B, n, H/N, D]: Q' in its scratch, K'/V in the cache staging slots
    right after the committed tokens (the contiguous key range K2 reads);
  * post-exchange + the K5 unpack layout: O's head shard goes back to the
    sequence shard [B, n/N, H, D];
  * all-to-all then its inverse is the identity, bitwise.
No GPU and no NCCL are used: the context is created with placeholder device
pointers that nothing dereferences on this path.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2602_15922_b200 as dz

FAKE_STORAGE = 1 << 32       # placeholder device address (256-byte aligned), never dereferenced here
FAKE_COMM = 0x1000


def _ctx(world, rank, B, H, D, n, capacity, rope):
    L = dz.lib()
    c = dz.DzConfig()
    c.batch, c.heads, c.head_dim = B, H, D
    for i in range(3):
        c.rope_dims[i] = rope[i]
    c.cache_capacity_tokens, c.max_chunk_tokens = capacity, n
    c.q_gain = c.k_gain = FAKE_STORAGE
    c.max_abs_gain = 1.0
    c.world_size, c.rank, c.nccl_comm = world, rank, FAKE_COMM
    c.flags = dz.FLAG_HOST_ONLY   # planning context: placeholder pointers, nothing dereferenced
    nbytes = L.dz_cache_bytes(ctypes.byref(c))
    assert nbytes > 0
    c.cache_storage, c.cache_bytes = FAKE_STORAGE, nbytes
    ctx = ctypes.c_void_p()
    assert L.dz_create(ctypes.byref(c), ctypes.byref(ctx)) == 0
    return ctx, nbytes


def _plan(ctx, phase, n):
    L = dz.lib()
    cnt = L.dz_sp_plan(ctx, phase, n, None, 0)
    assert cnt > 0
    arr = (dz.DzXfer * cnt)()
    assert L.dz_sp_plan(ctx, phase, n, arr, cnt) == cnt
    return [(x.peer, x.tensor, x.send_off, x.recv_off, x.bytes) for x in arr]


def _exchange(buf, plan, rank):
    """Run the plan: every entry is a send to / receive from its peer (gloo; self-copies locally)."""
    reqs, t = [], torch.from_numpy(buf)
    for peer, _, so, ro, nb in plan:
        if peer == rank:
            buf[ro:ro + nb] = buf[so:so + nb]
        else:
            reqs.append(dist.isend(t[so:so + nb].clone(), dst=peer))
            reqs.append(dist.irecv(t[ro:ro + nb], src=peer))
    for r in reqs:
        r.wait()
    dist.barrier()


def _tensor(tag, B, n, H, D):
    """Unique int16 content per (tensor, b, token, head, d) so any misplaced block is caught."""
    i = np.arange(B * n * H * D, dtype=np.int64).reshape(B, n, H, D)
    return ((i * 7 + tag * 1009) % 32749).astype(np.int16)


def _worker(rank, world, port, B, H, D, n, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        Hl, nl = H // world, n // world
        row = Hl * D * 2
        ctx, nbytes = _ctx(world, rank, B, H, D, n, 2 * n, (16, 24, 24) if D == 64 else (44, 42, 42))
        L = dz.lib()
        buf = np.zeros(nbytes, dtype=np.uint8)
        X = [_tensor(w, B, n, H, D) for w in range(4)]   # Q', K', V, O (global, identical on every rank)

        # ---- pre-exchange (attend): fill the send blocks as K1 writes them, exchange, check
        plan = _plan(ctx, 0, n)
        assert len(plan) == 3 * world * B
        for peer, w, so, ro, nb in plan:
            b = [p for p in plan if p[1] == w and p[0] == peer].index((peer, w, so, ro, nb))
            blk = X[w][b, rank * nl:(rank + 1) * nl, peer * Hl:(peer + 1) * Hl]
            assert nb == blk.nbytes
            buf[so:so + nb] = blk.reshape(-1).view(np.uint8)
        _exchange(buf, plan, rank)
        k0, v0, stride = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        for b in range(B):
            assert L.dz_cache_view(ctx, b, ctypes.byref(k0), ctypes.byref(v0), ctypes.byref(stride)) == 0
            assert stride.value == Hl * D
            kb, vb = k0.value - FAKE_STORAGE, v0.value - FAKE_STORAGE
            want = {w: X[w][b, :, rank * Hl:(rank + 1) * Hl] for w in range(3)}
            # K'/V: n staging slots right after the committed tokens (valid = 0 here), token-major
            for w, base in ((1, kb), (2, vb)):
                got = buf[base:base + n * row].view(np.int16).reshape(n, Hl, D)
                assert np.array_equal(got, want[w]), f"rank {rank} b {b} tensor {w}"
            # Q': scratch [B][n][Hl][D]; its base is where peer 0's block of batch 0 lands
            qb = min(p[3] for p in plan if p[1] == 0) + b * n * row
            got = buf[qb:qb + n * row].view(np.int16).reshape(n, Hl, D)
            assert np.array_equal(got, want[0]), f"rank {rank} b {b} Q'"

        # ---- post-exchange: O head shard -> receive blocks [N][B][n_loc][Hl][D] -> unpack (K5 layout)
        post = _plan(ctx, 2, n)
        assert len(post) == world * B
        ol = min(p[2] for p in post)           # O local [B][n][Hl][D]
        buf[ol:ol + B * n * row] = X[3][:, :, rank * Hl:(rank + 1) * Hl].reshape(-1).view(np.uint8)
        _exchange(buf, post, rank)
        orecv = min(p[3] for p in post)
        recv = buf[orecv:orecv + world * B * nl * row].view(np.int16).reshape(world, B, nl, Hl, D)
        unpacked = recv.transpose(1, 2, 0, 3, 4).reshape(B, nl, H, D)   # K5: [N][B][nl][Hl][D] -> [B][nl][H][D]
        assert np.array_equal(unpacked, X[3][:, rank * nl:(rank + 1) * nl]), f"rank {rank} O"

        # ---- all-to-all followed by its inverse is the identity (bitwise)
        plan1 = _plan(ctx, 1, n)            # append pre-exchange: K', V only
        assert all(p[1] in (1, 2) for p in plan1) and len(plan1) == 2 * world * B
        snap = buf.copy()
        inv = [(p, w, ro, so, nb) for p, w, so, ro, nb in plan1]
        _exchange(buf, plan1, rank)
        _exchange(buf, inv, rank)
        for p, w, so, ro, nb in plan1:
            assert np.array_equal(buf[so:so + nb], snap[so:so + nb])
        L.dz_destroy(ctx)
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        errq.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,B,H,D,n", [(2, 2, 4, 64, 64), (2, 1, 40, 128, 96), (4, 2, 8, 64, 128)])
def test_ulysses_exchange_plan_gloo(world, B, H, D, n):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, H, D, n, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), errs


def test_sp_plan_validation():
    ctx, _ = _ctx(2, 0, 1, 4, 64, 64, 64, (16, 24, 24))
    L = dz.lib()
    assert L.dz_sp_plan(ctx, 3, 64, None, 0) < 0
    assert L.dz_sp_plan(ctx, 0, 63, None, 0) < 0      # not a multiple of world_size
    assert L.dz_sp_plan(ctx, 0, 64, None, 0) == 3 * 2 * 1
    L.dz_destroy(ctx)
