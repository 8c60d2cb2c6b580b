#!/usr/bin/env python
"""bench.py -- block-causal chunk-attention throughput on B200 (DreamZero, arXiv 2602.15922).

Metric (BASELINE.json): useful TFLOP/s of the block-causal chunk-attention step
(4*D FLOP per visible (query, key) pair, summed over batch and heads) and its
fraction of the measured bf16 tensor-core peak (MEASURED_PEAKS.json).

One step = one pass of the whole hot path for one chunk, as
Alg. 2 runs it in the DreamZero-Flash 1-step regime:
  attend  -- K1 RMSNorm+3D-RoPE prologue of the noisy chunk's Q/K/V (+ Ulysses
             all-to-all under SP) and K2 tcgen05 attention over the KV cache plus
             the chunk itself (update=False);
  evict   -- the oldest chunk leaves the window, keeping the context length
             fixed (l.510 sliding context), so every step sees the same shapes;
  append  -- K4: the ground-truth clean chunk's K'/V written into the cache
             (update=True, l.601-602).
Useful FLOP counts only the attention.  Inputs are resident in HBM before
the timed region; the L2 is flushed (a 512 MB write) before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dz|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...    (Ulysses SP, C4)

Prints one JSON line (rank 0).  ``--impl reference`` times the fp64 CPU
oracle (the tier's reference arm) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "block-causal chunk-attn TFLOP/s and % bf16 TC peak at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["dz", "reference"], default="dz")
    ap.add_argument("--workload", default=None, help="C1 (default at 1 GPU) .. C4 (default under SP)")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="warm L2 (secondary measurement)")
    ap.add_argument("--tf-chunks", type=int, default=4, help="tf mode: M clean + M noisy chunks")
    ap.add_argument("--mode", choices=["chunk", "denoise", "tf"], default="chunk",
                    help="chunk: attend + evict + append per step; denoise: the denoising steps of one "
                         "chunk over a fixed cache (Alg. 2 update=False; C3: 4 steps x CFG batch 2); tf: the "
                         "teacher-forcing training layout [C0..C_{M-1}; Z1..Z_M] of Fig. 10(a) in one attend_spans")
    ap.add_argument("--denoise-steps", type=int, default=None, help="denoise mode: steps per chunk "
                    "(default: the workload's, C3 = 4)")
    ap.add_argument("--graph", action="store_true", help="denoise mode: replay the steps as one CUDA graph")
    ap.add_argument("--no-profile", action="store_true", help="no per-kernel events in the library (diagnostics)")
    ap.add_argument("--online", action="store_true", help="force the online-softmax (running max) kernel")
    ap.add_argument("--flush-read", action="store_true",
                    help="after the 512 MB flush write, read 256 MB of it so no dirty flush lines stay in L2")
    return ap.parse_args()


def visible_pairs(spans) -> int:
    """Visible (query, key) pairs of a span layout under the Fig. 10 rule (PAPER.md l.505,
    DESIGN.md R3): a NOISY query of chunk k sees CLEAN keys of chunks < k and its own span;
    a CLEAN query of chunk j sees CLEAN keys of chunks <= j.  (Checked against the oracle's
    pair enumeration in tests/test_bench_host.py.)"""
    total = 0
    for i, qs in enumerate(spans):
        qth = qs.chunk if qs.kind == synth.NOISY else qs.chunk + 1
        for j, ks in enumerate(spans):
            if i == j or (ks.kind == synth.CLEAN and ks.chunk < qth):
                total += qs.n_tokens * ks.n_tokens
    return total


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"   # B200_PROFILING.md fallback figures


class ClockSampler:
    """NVML SM clock + clock-event reasons sampled during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- oracle legs
_STREAMS = {}


def oracle_sample(w: synth.Workload, heads=(0, 1), q_rows=None):
    """Run the fp64 oracle (as it stands) on heads [h0, h1) and optional query rows; return (FLOP, seconds)."""
    import oracle
    if w.name not in _STREAMS:          # draw once; samples slice heads out of the full draw
        _STREAMS[w.name] = synth.draw_stream(w, 0, steps=1)
    full = _STREAMS[w.name]
    h0, h1 = heads
    hs = lambda x: x[:, h0:h1].contiguous()
    s = synth.ChunkStream([hs(k) for k in full.cache_k], [hs(v) for v in full.cache_v], full.cache_pos,
                          [hs(full.cur_q[0])], [hs(full.cur_k[0])], [hs(full.cur_v[0])], full.cur_pos)
    gq, gk = synth.draw_gains(w)
    q, pos = s.cur_q[0], s.cur_pos
    if q_rows is not None:
        q, pos_q = q[:q_rows], pos[:q_rows]
    else:
        pos_q = pos
    nq = q.shape[0]
    t0 = time.perf_counter()
    # the oracle's own composition, with the sampled queries only
    ks = [oracle.prologue(k, gk[h0:h1], p, w.rope_dims, w.rope_theta, w.rms_eps) for k, p in zip(s.cache_k, s.cache_pos)]
    ks.append(oracle.prologue(s.cur_k[0], gk[h0:h1], pos, w.rope_dims, w.rope_theta, w.rms_eps))
    vs = [v.double().numpy() for v in s.cache_v + [s.cur_v[0]]]
    qn = oracle.prologue(q, gq[h0:h1], pos_q, w.rope_dims, w.rope_theta, w.rms_eps)
    C = len(s.cache_k)
    kt = oracle.chunk_tags(list(range(C)) + [C], [oracle.CLEAN] * C + [oracle.NOISY],
                           [k.shape[0] for k in ks])
    qt = (np.full(nq, C, np.int32), np.full(nq, oracle.NOISY, np.int32), np.full(nq, C, np.int32))
    oracle.attention(qn, np.concatenate(ks), np.concatenate(vs), qt, kt)
    dt = time.perf_counter() - t0
    flop = 4.0 * w.head_dim * (h1 - h0) * nq * w.kv_tokens
    return flop, dt


def cpu_baseline(w: synth.Workload, budget_s: float):
    import oracle
    flop = secs = 0.0
    reps = 0
    h = 0
    while secs < budget_s or reps == 0:
        f, d = oracle_sample(w, heads=(h % w.heads, h % w.heads + 1))
        flop, secs, reps, h = flop + f, secs + d, reps + 1, h + 1
    return {"value": flop / secs / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{w.name}: {reps} single-head passes (head i mod {w.heads}, all {w.chunk_tokens} queries x "
                      f"{w.kv_tokens} keys incl. the cache prologue), fp64, {secs:.1f} s",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, w: synth.Workload, rank: int):
    if rank != 0:
        return
    import oracle
    q_rows = max(1, w.chunk_tokens // 4)
    for _ in range(args.warmup):
        oracle_sample(w, heads=(0, 1), q_rows=q_rows)
    flop = secs = 0.0
    for i in range(args.steps):
        f, d = oracle_sample(w, heads=(i % w.heads, i % w.heads + 1), q_rows=q_rows)
        flop, secs = flop + f, secs + d
    value = flop / secs / 1e12
    sample = (f"{w.name}: per step one head x first {q_rows} queries x {w.kv_tokens} keys "
              f"(incl. the cache prologue), fp64 oracle")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "batch": w.batch, "heads": w.heads, "head_dim": w.head_dim,
                       "chunk_tokens": w.chunk_tokens, "cache_tokens": w.cache_tokens, "sample": sample},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and not (world == 1 and args.gpus == 1):
        if world == 1 and args.gpus > 1:
            print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} processes"}))
            sys.exit(2)
    wname = args.workload or ("C1" if world == 1 else "C4")
    w = synth.workload(wname)

    if args.impl == "reference":
        run_reference(args, w, rank)
        return

    import paper_2602_15922_b200 as dz
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    comm = 0
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(dz.nccl_unique_id()), dtype=torch.uint8)
        uid = uid.to(dev)
        dist.broadcast(uid, 0)
        comm = dz.nccl_comm_init(world, bytes(uid.cpu().numpy().tobytes()), rank)

    N = world
    n, H, D = w.chunk_tokens, w.heads, w.head_dim
    n_loc = n // N
    gq, gk = synth.draw_gains(w)
    C = w.cached_chunks
    slack = 16 * n
    cache = dz.ChunkKVCache(w.batch, H, D, w.cache_tokens, n, w.rope_dims, gq.to(dev), gk.to(dev),
                            rope_theta=w.rope_theta, rms_eps=w.rms_eps, window_slack=slack, world_size=N,
                            rank=rank, nccl_comm=comm,
                            flags=(0 if args.no_profile else dz.FLAG_PROFILE) | (dz.FLAG_ONLINE_SOFTMAX if args.online else 0),
                            device=dev)
    sl = slice(rank * n_loc, (rank + 1) * n_loc)

    def dev_chunk(x):   # [B][n][H][D] bf16 -> this rank's tokens on the device
        return x[:, sl].contiguous().to(dev)

    S = (args.denoise_steps or w.steps) if args.mode == "denoise" else 1
    streams = [synth.draw_stream(w, b, steps=max(2, S)) for b in range(w.batch)]
    stack = lambda key, c: torch.stack([getattr(s, key)[c] for s in streams])
    for c in range(C):
        cache.append(dev_chunk(stack("cache_k", c)), dev_chunk(stack("cache_v", c)),
                     streams[0].cache_pos[c][sl].contiguous().to(dev), c)
    q, k, v = (dev_chunk(stack(x, 0)) for x in ("cur_q", "cur_k", "cur_v"))
    kc, vc = dev_chunk(stack("cur_k", 1)), dev_chunk(stack("cur_v", 1))   # the ground-truth clean chunk
    pos = streams[0].cur_pos[sl].contiguous().to(dev)
    out = torch.empty_like(q)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    chunk_id = [C]

    def step(qq=q, kk=k, vv=v, kkc=kc, vvc=vc, pp=pos, oo=out):
        cid = chunk_id[0]
        cache.attend(qq, kk, vv, pp, cid, out=oo)
        cache.evict_front(1)               # window full: the oldest chunk leaves ...
        cache.append(kkc, vvc, pp, cid)    # ... and the ground-truth chunk enters
        chunk_id[0] += 1

    graph = None
    flop_one = w.useful_flop()
    if args.mode == "tf":
        # Fig. 10(a) teacher forcing at the Wan shape: M clean chunks then M noisy chunks, one call
        tf_spans = synth.teacher_forcing_spans(args.tf_chunks, n)
        n_tf = sum(sp.n_tokens for sp in tf_spans)
        tq, tk, tv, tpos = synth.span_inputs(w, tf_spans)
        tf_cache = dz.ChunkKVCache(w.batch, H, D, 0, n_tf, w.rope_dims, gq.to(dev), gk.to(dev),
                                   rope_theta=w.rope_theta, rms_eps=w.rms_eps, flags=dz.FLAG_PROFILE, device=dev)
        tq, tk, tv = (x[None].expand(w.batch, -1, -1, -1).contiguous().to(dev) for x in (tq, tk, tv))
        tpos = tpos.to(dev)
        tout = torch.empty_like(tq)
        span_list = [(sp.chunk, sp.kind, sp.n_tokens) for sp in tf_spans]
        flop_one = 4.0 * D * w.batch * H * visible_pairs(tf_spans)
        cache = tf_cache

        def tf_step():
            tf_cache.attend_spans(tq, tk, tv, tpos, span_list, out=tout)

        step = tf_step
    if args.mode == "denoise":
        # S denoising steps of chunk C over the fixed cache: new Q, K, V per step (Alg. 2 l.584-585)
        qs = [[dev_chunk(stack(x, st)) for x in ("cur_q", "cur_k", "cur_v")] for st in range(S)]
        outs = [torch.empty_like(q) for _ in range(S)]

        def denoise():
            for st in range(S):
                cache.attend(*qs[st], pos, C, out=outs[st])

        step = denoise
        if args.graph:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                denoise()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                denoise()
            step = graph.replay
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region: per-step CUDA events, L2 flushed between steps.  The library's
    # per-kernel events are off in the timed steps: an event between two kernels ends their
    # programmatic overlap (PDL), so the kernels are timed in a profiled step after each timed one.
    flop_step = flop_one * S                         # global useful FLOP of one step
    profiled = graph is None and not args.no_profile
    if profiled:
        cache.profile_enable(False)

    def flush_l2():
        if not args.no_flush:
            flush.zero_()
            if args.flush_read:
                flush_sum = flush[: flush.numel() // 2].sum()  # noqa: F841

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    attn_ms, pro_ms, app_ms = [], [], []
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush_l2()
            ev[i][0].record()
            step()
            ev[i][1].record()
            if profiled:  # a profiled step between two timed ones (same load and clocks), not in the sum
                cache.profile_enable(True)
                flush_l2()
                step()
                prof = cache.profile_last()         # host-syncs on the library's events (last call)
                attn_ms.append(prof["attention"])
                pro_ms.append(prof["prologue"])
                app_ms.append(prof["append"])
                cache.profile_enable(False)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if pg:
        t = torch.tensor([total_ms], device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
        pg.barrier()
    value = flop_step * args.steps / (total_ms * 1e-3) / 1e12

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0 and args.mode == "chunk":  # (other modes: device-resident only)
        # End to end through the public API with host buffers: every step copies its inputs from
        # pinned host memory (H2D) and reads its output back (D2H), double-buffered so that the
        # copies of step i+1 and the read-back of step i-1 overlap the kernels of step i (a
        # user's pipelined denoising loop).  PCIe, not the kernels, bounds this number.
        pin = lambda x: x.cpu().pin_memory()
        hin = [pin(x) for x in (q, k, v, kc, vc, pos)]
        houts = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        h2d = sum(x.numel() * x.element_size() for x in hin)
        d2h = houts[0].numel() * houts[0].element_size()
        dins = [[torch.empty_like(x, device=dev) for x in (q, k, v, kc, vc, pos)] for _ in range(2)]
        douts = [torch.empty_like(out) for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
        main = torch.cuda.current_stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def h2d_copy(i):
            sl = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(consumed[sl])          # the step that read this buffer is done
                for d_, h_ in zip(dins[sl], hin):
                    d_.copy_(h_, non_blocking=True)
                copied[sl].record(s_h2d)

        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s_h2d.wait_stream(main)
        s_d2h.wait_stream(main)
        h2d_copy(0)
        for i in range(args.e2e_steps):
            sl = i % 2
            if i + 1 < args.e2e_steps:
                h2d_copy(i + 1)
            main.wait_event(copied[sl])
            if i >= 2:
                main.wait_event(drained[sl])                 # douts[sl] has been read back
            dq, dk, dv, dkc, dvc, dpos = dins[sl]
            step(dq, dk, dv, dkc, dvc, dpos, douts[sl])
            consumed[sl].record(main)
            computed[sl].record(main)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(computed[sl])
                houts[sl].copy_(douts[sl], non_blocking=True)
                drained[sl].record(s_d2h)
        main.wait_stream(s_d2h)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        if pg:
            t = torch.tensor([e2e_ms], device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": flop_step * args.e2e_steps / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": args.e2e_steps,
               "path": "pinned host -> ChunkKVCache.attend/append/evict -> pinned host, copies of "
                       "neighbouring steps overlapped on two copy streams"}

    peak, peak_sus, hbm, src = peaks()
    if not profiled:   # no per-kernel events: K1 + K2 of every step together
        attn_ms = [m / S for m in step_ms]
        pro_ms, app_ms = [float("nan")], [float("nan")]
    attn_mean = statistics.mean(attn_ms)
    flop_launch = flop_step / N / S
    achieved = flop_launch / (attn_mean * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_attention_traffic.json")
    if os.path.exists(tp):
        d = json.load(open(tp))
        if d.get("workload") == w.name:
            traffic = d.get("dram_bytes_per_launch")
    n_new = n_tf if args.mode == "tf" else n_loc
    # attend prologue: read q, k (+ v) and write q', k' (+ the V staging copy); with one GPU and the
    # new keys starting at a 128-key step the attention reads V in place (dz.h), no V copy
    v_in_place = N == 1 and (0 if args.mode == "tf" else w.cache_tokens) % 128 == 0
    pro_bytes = 2 * (2 if v_in_place else 3) * w.batch * n_new * H * D * 2
    app_bytes = 2 * 2 * w.batch * n_loc * H * D * 2     # read k,v + write k',v
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": N, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if N == 1 else "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w.name, "batch": w.batch, "heads": H, "head_dim": D, "chunk_tokens": n,
                   "cache_tokens": w.cache_tokens, "kv_tokens": w.kv_tokens, "useful_flop_per_step": flop_step,
                   "parallelism": "single GPU" if N == 1 else f"ulysses sp{N}",
                   "step": ("attend (K1+K2) + append (K4) + evict, sliding window" if args.mode == "chunk" else
                            f"teacher forcing [C0..C{args.tf_chunks - 1}; Z1..Z{args.tf_chunks}] x {n} tokens, "
                            "one attend_spans (K1+K2, SKIP tiles never loaded)" if args.mode == "tf" else
                            f"{S} denoising steps of one chunk (K1+K2 each) over a fixed cache"
                            + (", one CUDA graph replay" if graph is not None else ", eager")),
                   "l2": "flushed before every timed step (512 MB write)" if not args.no_flush else "warm",
                   "qk_storage": "fp16 (post-RMSNorm)", "pv": "bf16", "accumulate": "fp32"},
        "pct_peak": value / (N * peak), "pct_peak_sustained": value / (N * peak_sus),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "attn_fwd_kernel (K2)" if graph is None else "K1 + K2 per denoise step (graph replay)",
                     "timing": ("CUDA events around K2 on the library stream, in a profiled step after each "
                                "timed step (events between kernels end their PDL overlap)" if profiled else
                                "step events / steps (no per-kernel events)"),
                     "peak_source": f"MEASURED_PEAKS.json bf16_tflops ({src}, burst)",
                     "frac_vs_sustained": achieved / peak_sus, "attn_ms_mean": attn_mean,
                     "flop_per_launch": flop_launch},
        "kernels": {"prologue_ms": statistics.mean(pro_ms),  # (denoise mode: the last step's; graph: n/a)
                    "prologue_gbs": pro_bytes / (statistics.mean(pro_ms) * 1e-3) / 1e9,
                    "append_ms": statistics.mean(app_ms),
                    "append_gbs": (app_bytes / (statistics.mean(app_ms) * 1e-3) / 1e9
                                   if N == 1 and args.mode == "chunk" and statistics.mean(app_ms) > 0 else None),
                    "hbm_peak_gbs": hbm},
        "gpu_launches": args.steps * ((3 if N == 1 else 4) if args.mode == "chunk" else 2 * S),  # K1, K2 (K4)
        "clocks": clk.summary(),
        "e2e": e2e,
        "parity": "tests/test_gpu_parity.py (pytest -m gpu); bench.py runs no oracle on the GPU arm",
    }
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    cache.close()
    if comm:
        dz.nccl_comm_destroy(comm)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
