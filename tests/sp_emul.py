"""Ulysses ranks emulated on one GPU (reading A21).

N contexts of one cache (world_size N, rank r), created with
FLAG_EXTERNAL_EXCHANGE: every call stops at each all-to-all and this helper
delivers the transfers the library lists (dz_sp_pending) with one device copy
per transfer between the ranks' storages, then resumes every rank.  Everything
the N-GPU path runs -- K1 writing the [N][B][n/N][H/N][D] send layout, the
exchange plan, K2 on a head shard over the head-sharded cache, the O exchange
and the K5 unpack -- runs here; only the transport (NCCL send/recv over
NVLink) is replaced by cudaMemcpyAsync.  With peer=True (DZ_FLAG_PEER_STORE, NEXT-3) there is no
transfer at all: the kernels store into the other ranks' storages and the exchanges are barriers.  No kernel waits on another rank's
kernel: the ranks' stages are enqueued one after the other on one stream.
"""
from __future__ import annotations

from typing import List, Sequence

import torch

import synth


class SpRanks:
    def __init__(self, w: synth.Workload, N: int, gq: torch.Tensor, gk: torch.Tensor, dev, capacity=None,
                 slack=0, flags=0, batch=None, max_chunk=None, peer=False):
        import paper_2602_15922_b200 as dz
        self.dz, self.w, self.N, self.dev = dz, w, N, torch.device(dev)
        self.batch = w.batch if batch is None else batch
        cap = w.cache_tokens if capacity is None else capacity
        mc = w.chunk_tokens if max_chunk is None else max_chunk
        self.caches = [dz.ChunkKVCache(self.batch, w.heads, w.head_dim, cap, mc, w.rope_dims, gq.to(self.dev),
                                       gk.to(self.dev), rope_theta=w.rope_theta, rms_eps=w.rms_eps,
                                       window_slack=slack, world_size=N, rank=r,
                                       flags=flags | dz.FLAG_EXTERNAL_EXCHANGE | (dz.FLAG_PEER_STORE if peer else 0),
                                       device=self.dev)
                       for r in range(N)]
        if peer:   # NEXT-3: every rank stores into the others' storages (here: the same GPU's memory)
            bases = [c.storage.data_ptr() for c in self.caches]
            for c in self.caches:
                c.set_peers(bases)
        self.transfers = 0
        self.phases = []

    # ------------------------------------------------------------------ transport
    def drive(self):
        """Deliver every pending exchange of all ranks and resume them, until none is pending."""
        while True:
            pend = [c.sp_pending() for c in self.caches]
            phases = {p for p, _ in pend}
            if phases == {-1}:
                return
            assert len(phases) == 1, f"ranks stopped at different exchanges: {phases}"
            self.phases.append(phases.pop())
            for r, (_, xs) in enumerate(pend):
                seen = {}
                for peer, t, so, ro, nb in xs:
                    k = seen.get((peer, t), 0)
                    seen[(peer, t)] = k + 1
                    # this rank's k-th send to `peer` of tensor t is peer's k-th receive from this rank
                    m = [x for x in pend[peer][1] if x[0] == r and x[1] == t][k]
                    assert m[4] == nb, (r, peer, t, k)
                    dst, src = self.caches[peer].storage, self.caches[r].storage
                    dst[m[3]:m[3] + nb].copy_(src[so:so + nb])
                    self.transfers += 1
            for c in self.caches:
                c.sp_resume()

    def shard(self, x: torch.Tensor, r: int) -> torch.Tensor:
        """Rank r's sequence shard of a [B, n, ...] tensor (tokens on dim 1)."""
        nl = x.shape[1] // self.N
        return x[:, r * nl:(r + 1) * nl].contiguous()

    def pos_shard(self, pos: torch.Tensor, r: int) -> torch.Tensor:
        nl = pos.shape[0] // self.N
        return pos[r * nl:(r + 1) * nl].contiguous()

    # ------------------------------------------------------------------ calls
    def append(self, k, v, pos, chunk_id):
        for r, c in enumerate(self.caches):
            c.append(self.shard(k, r).to(self.dev), self.shard(v, r).to(self.dev), self.pos_shard(pos, r).to(self.dev),
                     chunk_id)
        self.drive()

    def attend(self, q, k, v, pos, chunk_id, kind=1) -> torch.Tensor:
        outs = [c.attend(self.shard(q, r).to(self.dev), self.shard(k, r).to(self.dev), self.shard(v, r).to(self.dev),
                         self.pos_shard(pos, r).to(self.dev), chunk_id, kind=kind)
                for r, c in enumerate(self.caches)]
        self.drive()
        return torch.cat(outs, dim=1)

    def attend_spans(self, q, k, v, pos, spans: Sequence) -> torch.Tensor:
        outs = [c.attend_spans(self.shard(q, r).to(self.dev), self.shard(k, r).to(self.dev),
                               self.shard(v, r).to(self.dev), self.pos_shard(pos, r).to(self.dev), spans)
                for r, c in enumerate(self.caches)]
        self.drive()
        return torch.cat(outs, dim=1)

    def commit_staged(self, chunk_id):
        for c in self.caches:
            c.commit_staged(chunk_id)

    def evict_front(self, n):
        for c in self.caches:
            c.evict_front(n)

    def cache_views(self, b=0) -> List:
        return [c.cache_view(b) for c in self.caches]

    def close(self):
        for c in self.caches:
            c.close()
