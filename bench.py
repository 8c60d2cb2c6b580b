#!/usr/bin/env python
"""bench.py -- block-causal chunk-attention throughput on B200 (DreamZero, arXiv 2602.15922).

Metric (BASELINE.json): useful TFLOP/s of the block-causal chunk-attention step
(4*D FLOP per visible (query, key) pair, summed over batch and heads) and its
fraction of the measured bf16 tensor-core peak (MEASURED_PEAKS.json).

One step = one pass of the whole hot path for one chunk, as
Alg. 2 runs it in the DreamZero-Flash 1-step regime:
  append  -- the ground-truth clean chunk c-1 enters the cache: K'/V written
             (update=True, l.601-602; its observation precedes chunk c's denoising);
  attend  -- the RMSNorm+3D-RoPE prologue of the noisy chunk c's Q/K (+ Ulysses
             all-to-all under SP) and K2 tcgen05 attention over the KV cache plus
             the chunk itself (update=False, l.584-585);
  evict   -- the oldest chunk leaves the window, keeping the context length
             fixed (l.510 sliding context), so every step sees the same shapes.
On one GPU append + attend are one dz_append_attend call: both prologues (the
K4 append and the K1 attend prologue) in one kernel launch, then K2.
Useful FLOP counts only the attention.  Inputs are resident in HBM before
the timed region; the L2 is flushed (a 512 MB write) before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dz|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...
        C4 (default under torchrun): Ulysses SP, 40/N heads per rank, NCCL all-to-all;
        --workload C3 at N=2: the CFG split (one batch element per GPU, no collective).

Prints one JSON line (rank 0).  ``--impl reference`` times the fp64 CPU
oracle (the tier's reference arm) on a bounded sample of the same workload.
At N=1 the line also carries secondary workloads (C2, C4 on one GPU, C3 as
4 graph-replayed denoising steps, Fig. 10(a) teacher forcing), each timed here.
"""
from __future__ import annotations

import argparse
import hashlib
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
TOL_MAX_ABS, TOL_REL_FRO = 2e-2, 5e-3     # BASELINE.json north_star


def parse(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["dz", "reference"], default="dz")
    ap.add_argument("--workload", default=None, help="C1 (default at 1 GPU) .. C4 (default under SP)")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle sample budget for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary workloads (N=1)")
    ap.add_argument("--secondary-steps", type=int, default=20)
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
    ap.add_argument("--fp8", action="store_true", help="FP8 (E4M3) QK^T variant (DZ_FLAG_FP8_QK; NEXT-2)")
    ap.add_argument("--cooldown", type=float, default=3.0,
                    help="idle seconds before each secondary workload (each starts at full clocks)")
    ap.add_argument("--no-discard", action="store_true",
                    help="keep the flush write's dirty lines in L2 (written back during the step)")
    ap.add_argument("--flush-read", action="store_true",
                    help="after the 512 MB flush write, read 256 MB of it so no dirty flush lines stay in L2")
    return ap.parse_args(argv)


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


def pct(xs, q):
    """q-th percentile (0..100) of a list, linear interpolation."""
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


def spread(xs):
    return {"median": pct(xs, 50), "p10": pct(xs, 10), "p90": pct(xs, 90), "mean": float(np.mean(xs)), "n": len(xs)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"   # B200_PROFILING.md fallback figures


def lib_sha():
    """Build identity: hash of the library's sources and build flags (paper_2602_15922_b200/build.py
    source_sha; the linked .so itself is not byte-reproducible)."""
    from paper_2602_15922_b200 import build as b
    return b.source_sha()


def stamped_traffic(workload: str):
    """DRAM bytes per K2 launch from the committed ncu capture, only if it was taken on this very
    library build (the sources' hash stamped into the file) and workload; else None."""
    tp = os.path.join(ROOT, "profiles", "ncu_attention_traffic.json")
    if not os.path.exists(tp):
        return None, "no capture"
    d = json.load(open(tp))
    if d.get("workload") != workload:
        return None, f"capture is of {d.get('workload')}"
    if d.get("lib_sha16") != lib_sha():
        return None, f"capture of another build ({d.get('lib_sha16')})"
    return d.get("dram_bytes_per_launch"), d.get("source")


class ClockSampler:
    """NVML SM clock + clock-event reasons sampled during the timed region (every 1 ms)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.power, self.reasons, self.max_mhz = [], [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv, self.err = None, str(e)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.001)

    def __enter__(self):
        if self.nv:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()
            self._sample()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(self.samples) if self.samples else None,
                "power_w_max": max(self.power) if self.power else None,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- oracle legs
_STREAMS = {}


def oracle_sample(w: synth.Workload, heads=(0, 1), q_rows=None, b=0):
    """Run the fp64 oracle (as it stands) on heads [h0, h1) and optional query rows of batch
    element b; return (FLOP, seconds, output [nq, h1-h0, D])."""
    import oracle
    key = (w.name, b)
    if key not in _STREAMS:          # draw once; samples slice heads out of the full draw
        _STREAMS[key] = synth.draw_stream(w, b, steps=1)
    full = _STREAMS[key]
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
    out = oracle.attention(qn, np.concatenate(ks), np.concatenate(vs), qt, kt)
    dt = time.perf_counter() - t0
    flop = 4.0 * w.head_dim * (h1 - h0) * nq * w.kv_tokens
    return flop, dt, out


def cpu_baseline(w: synth.Workload, budget_s: float, gpu_first=None):
    """The oracle timed on the host cores on single-head passes of the workload.  Its first two
    passes (heads 0 and H-1) are also the bench's parity check: the GPU output of the same
    attention (gpu_first, [n, H, D] of batch element 0, computed before the timed region)
    against the oracle within BASELINE.json's tolerance."""
    import oracle
    flop = secs = 0.0
    reps = 0
    heads = [0, w.heads - 1] + [h for h in range(1, w.heads - 1)]
    parity = []
    while secs < budget_s or reps < 2:
        h = heads[reps % len(heads)]
        f, d, out = oracle_sample(w, heads=(h, h + 1))
        if gpu_first is not None and reps < 2:
            got = gpu_first[:, h:h + 1].astype(np.float64)
            err = float(np.abs(got - out).max())
            rel = float(np.linalg.norm(got - out) / np.linalg.norm(out))
            parity.append({"head": h, "max_abs_err": err, "rel_fro_err": rel})
        flop, secs, reps = flop + f, secs + d, reps + 1
    res = {"value": flop / secs / 1e12, "unit": "TFLOP/s", "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{w.name}: {reps} single-head passes (heads 0, {w.heads - 1}, then 1.., all "
                     f"{w.chunk_tokens} queries x {w.kv_tokens} keys incl. the cache prologue), fp64, {secs:.1f} s",
           "cpu_model": _cpu_model()}
    if parity:
        res["parity"] = {"checks": parity, "tolerance": {"max_abs": TOL_MAX_ABS, "rel_fro": TOL_REL_FRO},
                         "pass": all(p["max_abs_err"] <= TOL_MAX_ABS and p["rel_fro_err"] <= TOL_REL_FRO
                                     for p in parity),
                         "what": "GPU attend of the bench's config (batch element 0, before the timed region) "
                                 "vs the fp64 oracle on the same seeded inputs"}
    return res


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
        f, d, _ = oracle_sample(w, heads=(i % w.heads, i % w.heads + 1), q_rows=q_rows)
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


# --------------------------------------------------------------------------- GPU timing
class Timer:
    """Times K steps with CUDA events at step boundaries only (an event between two kernels
    would end their programmatic overlap), the L2 flushed before every step; the library's
    per-kernel events are measured in K profiled steps run after the timed ones (not part of
    the sum)."""

    def __init__(self, dev, flush=True, flush_read=False, discard=True):
        self.flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if flush else None
        self.flush_read = flush_read
        self.discard = discard

    def flush(self):
        if self.flush_buf is not None:
            self.flush_buf.zero_()
            if self.flush_read:
                self.flush_buf[: self.flush_buf.numel() // 2].sum()
            if self.discard:  # the flush's dirty lines leave L2 without a write-back inside the step
                import paper_2602_15922_b200 as dz
                dz.l2_discard(self.flush_buf)

    def run(self, step, steps, cache=None, profiled=True, clock_dev=None):
        import paper_2602_15922_b200 as dz
        if profiled:
            cache.profile_enable(False)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        prof = {"prologue": [], "attention": [], "append": []}
        launches = 0
        torch.cuda.synchronize()
        dz.k2_clock(reset=True)  # SM cycles / ns summed over the attention CTAs of the timed steps
        sampler = ClockSampler(clock_dev) if clock_dev is not None else None
        if sampler:
            sampler.__enter__()
        # the timed steps are enqueued back to back with no host synchronisation, so the host runs
        # ahead of the device and the events time device work only (host launch latency is part of
        # the e2e measurement); the profiled steps (per-kernel library events, one host sync each)
        # follow in a loop of their own
        for i in range(steps):
            self.flush()
            torch.cuda.nvtx.range_push(f"dz step {i}")  # NVTX ranges: visible to nsys / ncu --nvtx
            ev[i][0].record()
            n0 = dz.kernel_launches()
            step()
            launches += dz.kernel_launches() - n0
            ev[i][1].record()
            torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        cyc, ns = dz.k2_clock()
        self.k2_ghz = cyc / ns if ns else None
        if sampler:
            sampler.__exit__()
        for i in range(steps if profiled else 0):
            cache.profile_enable(True)
            self.flush()
            torch.cuda.nvtx.range_push(f"dz profiled step {i}")
            step()
            torch.cuda.nvtx.range_pop()
            p = cache.profile_last()         # host-syncs on the library's events (last call)
            for k in prof:
                prof[k].append(p[k])
            cache.profile_enable(False)
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in ev]
        return step_ms, prof, launches, (sampler.summary() if sampler else None)


# cache slack before a compaction, in chunks: the window slides by one chunk per step and the cache
# is compacted (one device copy of the window) once per SLACK_CHUNKS steps; 64 chunks of C1 are 1.8 GB
SLACK_CHUNKS = int(os.environ.get("DZ_BENCH_SLACK_CHUNKS", "64"))


def make_cache(dz, w, dev, gq, gk, batch=None, world=1, rank=0, comm=0, flags=0, slack=None, max_chunk=None):
    n = w.chunk_tokens
    return dz.ChunkKVCache(w.batch if batch is None else batch, w.heads, w.head_dim, w.cache_tokens,
                           n if max_chunk is None else max_chunk, w.rope_dims, gq.to(dev), gk.to(dev),
                           rope_theta=w.rope_theta, rms_eps=w.rms_eps,
                           window_slack=SLACK_CHUNKS * n if slack is None else slack, world_size=world, rank=rank,
                           nccl_comm=comm, flags=flags, device=dev)


def device_inputs(w, dev, batch, seed, n_local=None):
    """Timing-only inputs drawn on the device (same shapes and distributions as synth: N(0,1) bf16,
    C2's 1% +-8 raw-K outliers)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    n = w.chunk_tokens if n_local is None else n_local
    shp = (batch, n, w.heads, w.head_dim)
    q, k, v = (torch.randn(shp, generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    if w.outliers:
        u1 = torch.rand(shp, generator=g, device=dev)
        u2 = torch.rand(shp, generator=g, device=dev)
        k = torch.where(u1 < 0.01, 8.0 * torch.sign(u2 - 0.5), k.float()).to(torch.bfloat16)
    return q, k, v


def secondary(dz, dev, steps, timer: Timer, cooldown=3.0):
    """Secondary workloads at one GPU, each timed like the primary (events at step boundaries,
    kernels in profiled steps): K2 TFLOP/s and fraction of the measured peak.  Timing only:
    inputs drawn on the device; parity of these configs is in tests/ (pytest -m gpu)."""
    peak, _, hbm, _ = peaks()
    out = {}

    def chunk_line(w, name, extra_flags=0):
        time.sleep(cooldown)   # the previous workload's power draw must not cap this one's clocks
        gq, gk = synth.draw_gains(w)
        cache = make_cache(dz, w, dev, gq, gk, flags=dz.FLAG_PROFILE | extra_flags)
        C = w.cached_chunks
        for c in range(C - 1):
            _, k, v = device_inputs(w, dev, w.batch, 10_000 + c)
            cache.append(k, v, synth.chunk_positions(w, c).to(dev), c)
        q, k, v = device_inputs(w, dev, w.batch, 20_000)
        _, kc, vc = device_inputs(w, dev, w.batch, 30_000)
        pos = synth.chunk_positions(w, C).to(dev)
        o = torch.empty_like(q)
        cid = [C - 1]

        def step():   # inject chunk cid, denoise chunk cid + 1 over C cached chunks, evict the oldest
            cache.append_attend(kc, vc, pos, cid[0], q, k, v, pos, cid[0] + 1, out=o)
            cache.evict_front(1)
            cid[0] += 1
        for _ in range(3):
            step()
        sm, prof, launches, clk = timer.run(step, steps, cache, clock_dev=dev.index)
        flop = w.useful_flop()
        k2 = statistics.median(prof["attention"])
        # the fused prologue reads k_gt, v_gt, q, k and writes K', V (cache) and Q', K' (noisy chunk)
        pro_bytes = 2 * 4 * w.batch * w.chunk_tokens * w.heads * w.head_dim * 2
        pro = statistics.median(prof["prologue"])
        pk = peak
        if extra_flags & dz.FLAG_FP8_QK:
            # half the useful FLOP (QK^T) at the FP8 rate, half (PV) at bf16: the mix's peak is
            # 2 / (1/P8 + 1/P16) with P8 = 2 x the measured bf16 peak (the nominal dense FP8:BF16
            # ratio, 4.5 : 2.25 PFLOP/s; no FP8 GEMM was measured) = 4/3 x 1630.3
            pk = peak * 4.0 / 3.0
        out[name] = {"workload": w.name, "mode": "chunk (append_attend + evict)",
                     "step_tflops": flop / (statistics.median(sm) * 1e-3) / 1e12,
                     "step_ms": spread(sm), "k2_ms": spread(prof["attention"]),
                     "k2_tflops": flop / (k2 * 1e-3) / 1e12, "k2_frac": flop / (k2 * 1e-3) / 1e12 / pk,
                     "k2_peak": pk,
                     "prologue_ms": spread(prof["prologue"]), "prologue_gbs": pro_bytes / (pro * 1e-3) / 1e9,
                     "prologue_frac_hbm": pro_bytes / (pro * 1e-3) / 1e9 / hbm,
                     "gpu_launches_per_step": launches / steps, "clocks": clk, "k2_sm_ghz": timer.k2_ghz}
        cache.close()

    chunk_line(synth.workload("C1"), "C1_fp8_qk", dz.FLAG_FP8_QK)   # NEXT-2: E4M3 QK^T, bf16 PV
    chunk_line(synth.workload("C2"), "C2")
    chunk_line(synth.workload("C4"), "C4@1")

    # C3: 4 denoising steps x CFG batch 2 over one cache of 8 chunks, one CUDA graph replay
    time.sleep(cooldown)
    w = synth.workload("C3")
    gq, gk = synth.draw_gains(w)
    cache = make_cache(dz, w, dev, gq, gk, slack=0)
    for c in range(w.cached_chunks):
        _, k, v = device_inputs(w, dev, w.batch, 40_000 + c)
        cache.append(k, v, synth.chunk_positions(w, c).to(dev), c)
    S = w.steps
    ins = [device_inputs(w, dev, w.batch, 50_000 + s) for s in range(S)]
    outs = [torch.empty_like(ins[0][0]) for _ in range(S)]
    pos = synth.chunk_positions(w, w.cached_chunks).to(dev)

    def denoise():
        for s in range(S):
            cache.attend(*ins[s], pos, w.cached_chunks, out=outs[s])
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        denoise()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        denoise()
    for _ in range(3):
        graph.replay()
    sm, _, launches, clk = timer.run(graph.replay, steps, profiled=False, clock_dev=dev.index)
    flop = w.useful_flop() * S
    out["C3_denoise_graph"] = {"workload": "C3", "mode": f"{S} denoising steps x batch 2 (K1 + K2 each), one CUDA "
                               "graph replay per step", "step_ms": spread(sm),
                               "step_tflops": flop / (statistics.median(sm) * 1e-3) / 1e12,
                               "step_frac": flop / (statistics.median(sm) * 1e-3) / 1e12 / peak,
                               "gpu_launches_per_step": 2 * S, "clocks": clk}
    cache.close()

    # Fig. 10(a) teacher forcing [C0..C3; Z1..Z4] x 1344 tokens, one attend_spans (SKIP tiles never loaded)
    time.sleep(cooldown)
    w = synth.workload("C1")
    gq, gk = synth.draw_gains(w)
    spans = synth.teacher_forcing_spans(4, w.chunk_tokens)
    n_tf = sum(s.n_tokens for s in spans)
    cache = dz.ChunkKVCache(1, w.heads, w.head_dim, 0, n_tf, w.rope_dims, gq.to(dev), gk.to(dev),
                            flags=dz.FLAG_PROFILE, device=dev)
    q, k, v = device_inputs(w, dev, 1, 60_000, n_local=n_tf)
    pos = torch.cat([synth.chunk_positions(w, s.chunk) for s in spans]).to(dev)
    o = torch.empty_like(q)
    sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
    step = lambda: cache.attend_spans(q, k, v, pos, sl, out=o)
    for _ in range(3):
        step()
    sm, prof, launches, clk = timer.run(step, steps, cache, clock_dev=dev.index)
    flop = 4.0 * w.head_dim * w.heads * visible_pairs(spans)
    k2 = statistics.median(prof["attention"])
    out["tf_fig10a"] = {"workload": "C1 shape, [C0..C3; Z1..Z4] x 1344", "mode": "teacher forcing (attend_spans)",
                        "visible_fraction": visible_pairs(spans) / n_tf ** 2, "step_ms": spread(sm),
                        "step_tflops": flop / (statistics.median(sm) * 1e-3) / 1e12,
                        "k2_ms": spread(prof["attention"]), "k2_tflops": flop / (k2 * 1e-3) / 1e12,
                        "k2_frac": flop / (k2 * 1e-3) / 1e12 / peak, "clocks": clk}
    cache.close()

    # NEXT-1 backward of the Fig. 10(a) layout [C0 C1; Z1 Z2] x 1344 (40 heads): the forward's prologue
    # recomputed, delta, the attention backward, the prologue backward; useful FLOP = 10 D per visible
    # pair (S, dP, dV, dK, dQ: 2 D each) summed over heads
    time.sleep(cooldown)
    spans = synth.teacher_forcing_spans(2, w.chunk_tokens)
    n_b = sum(s.n_tokens for s in spans)
    cache = dz.ChunkKVCache(1, w.heads, w.head_dim, 0, n_b, w.rope_dims, gq.to(dev), gk.to(dev),
                            flags=dz.FLAG_WRITE_LSE | dz.FLAG_BACKWARD, device=dev)
    q, k, v = device_inputs(w, dev, 1, 70_000, n_local=n_b)
    dout = device_inputs(w, dev, 1, 80_000, n_local=n_b)[0]
    pos = torch.cat([synth.chunk_positions(w, s.chunk) for s in spans]).to(dev)
    sl = [(s.chunk, s.kind, s.n_tokens) for s in spans]
    o = cache.attend_spans(q, k, v, pos, sl)
    lse = cache.lse(n_b)
    bstep = lambda: cache.attend_spans_backward(q, k, v, pos, sl, o, lse, dout)
    for _ in range(3):
        bstep()
    sm, _, launches, clk = timer.run(bstep, max(5, steps // 4), profiled=False, clock_dev=dev.index)
    bflop = 10.0 * w.head_dim * w.heads * visible_pairs(spans)
    out["tf_backward"] = {"workload": "C1 shape, [C0 C1; Z1 Z2] x 1344, 40 heads",
                          "mode": "dz_attend_spans_backward (prologue recompute + delta + attention backward + "
                                  "prologue backward)", "step_ms": spread(sm),
                          "step_tflops": bflop / (statistics.median(sm) * 1e-3) / 1e12,
                          "step_frac": bflop / (statistics.median(sm) * 1e-3) / 1e12 / peak,
                          "useful_flop": bflop, "gpu_launches_per_step": launches / max(5, steps // 4), "clocks": clk}
    cache.close()
    return out


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
    cfg_split = world > 1 and w.name == "C3"      # CFG parallelism: one batch element per GPU
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        if not cfg_split:
            uid = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                uid = torch.frombuffer(bytearray(dz.nccl_unique_id()), dtype=torch.uint8)
            uid = uid.to(dev)
            dist.broadcast(uid, 0)
            comm = dz.nccl_comm_init(world, bytes(uid.cpu().numpy().tobytes()), rank)
    if cfg_split and world != w.batch:
        print(json.dumps({"error": f"CFG split of {w.name} needs {w.batch} GPUs"}))
        sys.exit(2)

    N = 1 if cfg_split else world                 # Ulysses ranks
    n, H, D = w.chunk_tokens, w.heads, w.head_dim
    n_loc = n // N
    B = 1 if cfg_split else w.batch               # batch elements held by this rank
    b_elems = [rank] if cfg_split else list(range(w.batch))
    gq, gk = synth.draw_gains(w)
    C = w.cached_chunks
    flags = ((0 if args.no_profile else dz.FLAG_PROFILE) | (dz.FLAG_ONLINE_SOFTMAX if args.online else 0)
             | (dz.FLAG_FP8_QK if args.fp8 else 0))
    cache = make_cache(dz, w, dev, gq, gk, batch=B, world=N, rank=0 if cfg_split else rank, comm=comm, flags=flags)
    sl = slice(rank * n_loc, (rank + 1) * n_loc) if N > 1 else slice(0, n)

    def dev_chunk(x):   # [B][n][H][D] bf16 -> this rank's tokens on the device
        return x[:, sl].contiguous().to(dev)

    S = (args.denoise_steps or w.steps) if args.mode == "denoise" else 1
    streams = [synth.draw_stream(w, b, steps=max(2, S)) for b in b_elems]
    stack = lambda key, c: torch.stack([getattr(s, key)[c] for s in streams])
    for c in range(C):
        cache.append(dev_chunk(stack("cache_k", c)), dev_chunk(stack("cache_v", c)),
                     streams[0].cache_pos[c][sl].contiguous().to(dev), c)
    q, k, v = (dev_chunk(stack(x, 0)) for x in ("cur_q", "cur_k", "cur_v"))
    kc, vc = dev_chunk(stack("cur_k", 1)), dev_chunk(stack("cur_v", 1))   # the ground-truth clean chunk
    if os.environ.get("DZ_BENCH_DIAG_ZERO_VGT"):  # diagnostics only (operand-dependent clocks): V_gt = 0
        vc.zero_()
    pos = streams[0].cur_pos[sl].contiguous().to(dev)
    out = torch.empty_like(q)
    # parity sample (outside the timed region): the first attention of this config, batch element 0
    first = None
    if world == 1 and args.mode == "chunk":
        first = cache.attend(q, k, v, pos, C, out=torch.empty_like(q))[0].float().cpu().numpy()
    if args.mode == "chunk":
        cache.evict_front(1)               # C-1 chunks: each step injects one, attends with C, evicts one
    chunk_id = [C]

    def step(qq=q, kk=k, vv=v, kkc=kc, vvc=vc, pp=pos, oo=out):
        cid = chunk_id[0]
        # the ground-truth chunk cid enters, chunk cid + 1 is denoised ...
        cache.append_attend(kkc, vvc, pp, cid, qq, kk, vv, pp, cid + 1, out=oo)
        cache.evict_front(1)               # ... and the oldest chunk leaves the window
        chunk_id[0] += 1

    graph = None
    flop_one = w.useful_flop()                     # whole job: all batch elements, all ranks
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

    # ---------------- timed region
    flop_step = flop_one * S                         # global useful FLOP of one step (all ranks)
    profiled = graph is None and not args.no_profile
    timer = Timer(dev, flush=not args.no_flush, flush_read=args.flush_read, discard=not args.no_discard)
    if pg:
        pg.barrier()
    step_ms, prof, launches, clocks = timer.run(step, args.steps, cache, profiled=profiled, clock_dev=local)
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
        # Every step copies its inputs from pinned host memory (H2D) and reads its output back
        # (D2H), double-buffered so that the copies of step i+1 and the read-back of step i-1
        # overlap the kernels of step i (a user's pipelined denoising loop).  PCIe bounds it.
        pin = lambda x: x.cpu().pin_memory()
        hin = [pin(x) for x in (q, k, v, kc, vc, pos)]
        houts = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        h2d = sum(x.numel() * x.element_size() for x in hin)
        d2h = houts[0].numel() * houts[0].element_size()
        dins = [[torch.empty_like(x, device=dev) for x in (q, k, v, kc, vc, pos)] for _ in range(2)]
        douts = [torch.empty_like(out) for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
        main_s = torch.cuda.current_stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]

        def h2d_copy(i):
            s_ = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(consumed[s_])          # the step that read this buffer is done
                for d_, h_ in zip(dins[s_], hin):
                    d_.copy_(h_, non_blocking=True)
                copied[s_].record(s_h2d)

        if pg:
            pg.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s_h2d.wait_stream(main_s)
        s_d2h.wait_stream(main_s)
        h2d_copy(0)
        for i in range(args.e2e_steps):
            s_ = i % 2
            if i + 1 < args.e2e_steps:
                h2d_copy(i + 1)
            main_s.wait_event(copied[s_])
            if i >= 2:
                main_s.wait_event(drained[s_])                 # douts[s_] has been read back
            dq, dk, dv, dkc, dvc, dpos = dins[s_]
            step(dq, dk, dv, dkc, dvc, dpos, douts[s_])
            consumed[s_].record(main_s)
            computed[s_].record(main_s)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(computed[s_])
                houts[s_].copy_(douts[s_], non_blocking=True)
                drained[s_].record(s_d2h)
        main_s.wait_stream(s_d2h)
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
    peak_k2, peak_k2_src = peak, f"MEASURED_PEAKS.json bf16_tflops ({src}, burst)"
    if args.fp8:  # half the FLOP at the FP8 rate (2 x bf16, nominal ratio), half at bf16: 4/3 x bf16
        peak_k2, peak_k2_src = peak * 4.0 / 3.0, peak_k2_src + " x 4/3 (E4M3 QK^T + bf16 PV mix)"
    attn_ms = prof["attention"] if profiled else [m / S for m in step_ms]
    attn_med = statistics.median(attn_ms)
    ranks_work = 1 if cfg_split else N
    flop_launch = flop_step / S / (w.batch if cfg_split else ranks_work)   # one rank's K2 launch
    achieved = flop_launch / (attn_med * 1e-3) / 1e12
    traffic, traffic_src = stamped_traffic(w.name) if (N == 1 and not cfg_split and args.mode == "chunk") else (None, "n/a")
    n_new = n_tf if args.mode == "tf" else n_loc
    # attend prologue (K1): reads q, k (+ v) and writes q', k' (+ the V staging copy); with one GPU and
    # the new keys starting at a 128-key step the attention reads V in place (dz.h), no V copy
    v_in_place = N == 1 and (0 if args.mode == "tf" else w.cache_tokens) % 128 == 0
    pro_tensors = 2 if v_in_place else 3
    if N == 1 and args.mode == "chunk":
        pro_tensors += 2      # dz_append_attend: the ground-truth chunk's k, v (K4) in the same launch
    pro_bytes = 2 * pro_tensors * B * n_new * H * D * 2
    app_bytes = 2 * 2 * B * n_loc * H * D * 2     # read k,v + write k',v
    pro_med = statistics.median(prof["prologue"]) if profiled else float("nan")
    app_med = statistics.median(prof["append"]) if profiled else float("nan")
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": w.name, "batch": w.batch, "heads": H, "head_dim": D, "chunk_tokens": n,
                   "cache_tokens": w.cache_tokens, "kv_tokens": w.kv_tokens, "useful_flop_per_step": flop_step,
                   "parallelism": ("single GPU" if world == 1 else
                                   f"cfg split ({world} GPUs, one batch element each, no collective)" if cfg_split
                                   else f"ulysses sp{N}"),
                   "step": (("append_attend (one prologue launch for the K4 append and the K1 attend "
                             "prologue, then K2) + evict, sliding window" if N == 1 else
                             "append (K4 + exchange) + attend (K1 + exchange + K2 + exchange + K5) + evict")
                            if args.mode == "chunk" else
                            f"teacher forcing [C0..C{args.tf_chunks - 1}; Z1..Z{args.tf_chunks}] x {n} tokens, "
                            "one attend_spans (K1+K2, SKIP tiles never loaded)" if args.mode == "tf" else
                            f"{S} denoising steps of one chunk (K1+K2 each) over a fixed cache"
                            + (", one CUDA graph replay" if graph is not None else ", eager")),
                   "l2": ("warm" if args.no_flush else "flushed before every timed step (512 MB write"
                          + (")" if args.no_discard else ", then its L2 lines discarded without write-back)")),
                   "qk_storage": "e4m3 (FP8 variant)" if args.fp8 else "fp16 (post-RMSNorm)", "pv": "bf16",
                   "accumulate": "fp32"},
        "pct_peak": value / (world * peak), "pct_peak_sustained": value / (world * peak_sus),
        "step_ms": spread(step_ms),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_k2, "unit": "TFLOP/s",
                     "frac": achieved / peak_k2, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "attn_fwd_kernel (K2)" if profiled else "K1 + K2 per denoise step (no per-kernel events)",
                     "timing": ("median of CUDA events around K2 on the library stream, in a profiled step after "
                                "each timed step (events between kernels end their PDL overlap)" if profiled else
                                "step events / steps (no per-kernel events)"),
                     "k2_ms": spread(attn_ms),
                     "peak_source": peak_k2_src,
                     "frac_vs_sustained": achieved / peak_sus, "flop_per_launch": flop_launch,
                     # per-clock tensor efficiency: 148 SMs x 8192 dense bf16 FLOP/clk (tools/mma_bench.cu
                     # measures 8110-8170 for N >= 128) at the median SM clock sampled in the timed region
                     "frac_per_clock": (achieved * 1e12 / (148 * 8192 * clocks["sm_mhz"] * 1e6)
                                        if clocks and clocks.get("sm_mhz") else None),
                     # the SM clock K2 actually ran at in the timed steps (clock64 / globaltimer of every
                     # K2 CTA, dz_debug_k2_clock; NVML's 1 ms samples mostly see the flush and idle gaps)
                     "k2_sm_ghz": getattr(timer, "k2_ghz", None),
                     "frac_per_clock_k2": (achieved * 1e12 / (148 * 8192 * timer.k2_ghz * 1e9)
                                           if getattr(timer, "k2_ghz", None) else None)},
        "kernels": {"prologue_ms": spread(prof["prologue"]) if profiled else None,
                    "prologue_gbs": pro_bytes / (pro_med * 1e-3) / 1e9 if profiled else None,
                    "append_ms": spread(prof["append"]) if profiled else None,
                    "append_gbs": (app_bytes / (app_med * 1e-3) / 1e9
                                   if N == 1 and args.mode == "chunk" and profiled and app_med > 0 else None),
                    "hbm_peak_gbs": hbm},
        "gpu_launches": launches,
        "gpu_launches_how": "dz_kernel_launches() difference over the timed steps (host count at launch)",
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and N == 1 and not cfg_split and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args.cpu_seconds, first)
        if "parity" in line["cpu_baseline"]:
            line["parity"] = line["cpu_baseline"]["parity"]
    if rank == 0 and world == 1 and args.mode == "chunk" and not args.no_secondary and w.name == "C1":
        cache.close()
        line["secondary"] = secondary(dz, dev, args.secondary_steps, timer, args.cooldown)
    if rank == 0:
        print(json.dumps(line), flush=True)
    cache.close()
    if comm:
        dz.nccl_comm_destroy(comm)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
