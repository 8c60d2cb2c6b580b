// backward.cu -- NEXT-1 backward: gradients of the teacher-forced path (Fig. 10(a) spans, empty cache)
//   L = sum(dO * O),  O = softmax_masked(q' k'^T * scale) V,  x' = RoPE(RMSNorm(x) * g)
// ("trajectory-level updates", Alg. 1 l.512-553).
//
// Three kernels, run after the forward prologue (K1) has recomputed Q' (pre-scaled by
// scale * log2e, fp16) and K' (fp16):
//   B1 delta_kernel     delta_s = <dO_s, O_s> and lse2_s = lse_s * log2(e), per (b, h, query)
//   B2 attn_bwd_kernel  one CTA per (b, h, 128-key tile), looping over the 64-query steps that see any
//                       of its keys (SKIP steps never loaded); five tcgen05 MMAs per step, accumulators
//                       in TMEM (DESIGN.md §7 "Backward"):
//                         S^T = K' Q'^T          (M = keys, N = queries, K = D)           cols [0,64)
//                         dP^T = V dO^T          (M = keys, N = queries, K = D)           cols [64,128)
//                         -- 8 warps (thread = key row, 32 queries each): P^T = 2^(S^T - lse2) into TMEM
//                            (cols [192,256), two buffers), dS^T = P^T (dP^T - delta) into shared memory
//                            (two buffers), masked (Fig. 10) --
//                         dV += P^T dO           (A = P^T from TMEM, B = dO MN-major)     cols [256,384)
//                         dK += dS^T Q'          (B = Q' read MN-major)                   cols [384,512)
//                         dQ^T = K'^T dS^T       (A = K', B = dS^T, both MN-major)        cols [128,192)
//                       4 drain warps move dQ^T (thread = d row) to a staging tile, one TMA reduce-add per
//                       step into the fp32 dQ' workspace; dV (bf16) and dK' (fp32) are written once per CTA.
//   B3 prologue_bwd_kernel  dx = RMSNorm/RoPE backward of dx' for q and k, and the gain gradients.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace dz {
namespace {

constexpr int kBwdTile = 128;        // keys per CTA
constexpr int kQStep = 64;           // queries per step
#ifndef DZ_BWD_QW
#define DZ_BWD_QW 32
#endif
constexpr int kQW = DZ_BWD_QW;               // queries of a step per softmax-gradient warp
constexpr int kQS = 64 / kQW;                // query slices of a step
constexpr int kCompWarps = 4 * kQS;          // softmax-gradient warps: TMEM lane quadrant w % 4, slice w / 4
constexpr int kWarpProd = kCompWarps, kWarpMma = kCompWarps + 1, kWarpDrain = kCompWarps + 2;  // + 4 drain warps
constexpr int kBwdThreads = (kCompWarps + 6) * 32;
constexpr int kKTile = 128 * 128 * 2;      // [128 keys][128 d] 16-bit as two [128][64] SW128 boxes
constexpr int kKBox = 128 * 128;
constexpr int kQTile = 64 * 128 * 2;       // [64 q][128 d] as two [64][64] boxes
constexpr int kQBox = 64 * 128;
constexpr int kPTile = 128 * 64 * 2;       // [128 keys][64 q]: one box

// shared-memory map: K', V (whole launch), Q' / dO / lse2 / delta of the step's queries (a ring of
// kQStages: a step's tiles are loaded while the two before it run), P^T, dS^T, the dQ staging tile
constexpr int kQStages = 3;          // Q' / dO / lse2 / delta ring
constexpr int kOffK = 0, kOffV = kKTile, kOffQ = 2 * kKTile, kOffDO = kOffQ + kQStages * kQTile,
              kOffDST = kOffDO + kQStages * kQTile, kOffVec = kOffDST + 2 * kPTile,  // dS^T[2]
              kOffDQ = kOffVec + kQStages * 512,
              kDQTile = kQStep * 128 * 4,                    // dQ staging [64 q][128 d] fp32
              kOffBar = kOffDQ + kDQTile, kBwdSmem = kOffBar + 256 + 1024;
static_assert(kBwdSmem <= 232448, "backward shared memory");

#ifdef DZ_BWD_TRACE
// diagnostics build only: clock() per step of one CTA ([step][24] words)
__device__ uint32_t g_bwd_trace[128 * 24];
__device__ int g_bwd_trace_cta = -1;
__device__ uint32_t g_bwd_cta[4096 * 4];  // per CTA: globaltimer start / end (ns, low 32 bits), steps, SM id
__device__ __forceinline__ uint32_t bt_gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (uint32_t)t;
}
__device__ __forceinline__ uint32_t bt_smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#define BT_CTA(slot, v) do { if (blockIdx.x < 4096) g_bwd_cta[blockIdx.x * 4 + (slot)] = (v); } while (0)
#define BT(step, slot) do { if (bt_on && (step) < 128) g_bwd_trace[(step) * 24 + (slot)] = (uint32_t)clock(); } while (0)
#else
#define BT(step, slot) do { } while (0)
#define BT_CTA(slot, v) do { } while (0)
#endif

constexpr int kMaxRanges = 12;  // visible query-step ranges kept per key tile (more: the StepWalk path)
struct BwdBars {
  uint64_t kv_full, q_full[kQStages], q_empty[kQStages], s_full, s_read, dq_full, dq_free, p_ready[2], mma_done[2];
  uint32_t tmem_base;
  int32_t n_ranges;              // -1: more than kMaxRanges, walk the span table instead
  int32_t rng[kMaxRanges][2];    // [first, end) query steps, increasing, disjoint
};
static_assert(sizeof(BwdBars) <= 256, "backward barrier block");

__device__ __forceinline__ bool span_vis(const SpanTable& st, int qs, int ks) {
  return qs == ks || st.kc[ks] < st.qth[qs];
}
__device__ __forceinline__ int span_of(const SpanTable& st, int x) {
  int i = 0;
  while (i + 1 < st.n && st.start[i + 1] <= x) ++i;
  return i;
}
// The visible query steps of one key tile, walked in increasing order; each role keeps its own walk.
// The query-span cursor qc only moves forward and invisible query spans are skipped whole, so a walk
// costs O(steps + spans) reads of the (parameter-space) span table.
struct StepWalk {
  int qc = 0;         // query span holding the first query of the last step returned
  int ks_lo, ks_hi;   // key spans intersecting the tile
  __device__ __forceinline__ StepWalk(const SpanTable& st, int k0, int n)
      : ks_lo(span_of(st, k0)), ks_hi(span_of(st, min(k0 + kBwdTile, n) - 1)) {}
  // first step >= s with a visible (query, key) pair (n_qsteps if none)
  __device__ __forceinline__ int next(const SpanTable& st, int s, int n_qsteps) {
    if (s >= n_qsteps) return n_qsteps;
    const int q0 = s * kQStep;
    while (qc + 1 < st.n && st.start[qc + 1] <= q0) ++qc;
    int r = n_qsteps;
    for (int qs = qc; qs < st.n; ++qs) {
      bool v = false;
      for (int ks = ks_lo; ks <= ks_hi; ++ks) v |= span_vis(st, qs, ks);
      if (v) {
        r = max(s, st.start[qs] / kQStep);
        break;
      }
    }
    if (r < n_qsteps)
      while (qc + 1 < st.n && st.start[qc + 1] <= r * kQStep) ++qc;
    return r;
  }
};
// The visible steps of the tile in increasing order, from the ranges in shared memory (or the walk).
struct Steps {
  const BwdBars* bars;
  StepWalk walk;
  int r = 0;
  __device__ __forceinline__ Steps(const BwdBars* b_, const SpanTable& st, int k0, int n) : bars(b_), walk(st, k0, n) {}
  __device__ __forceinline__ int first(const SpanTable& st, int n_qsteps) {
    const int nr = bars->n_ranges;
    if (nr < 0) return walk.next(st, 0, n_qsteps);
    r = 0;
    return nr > 0 ? bars->rng[0][0] : n_qsteps;
  }
  __device__ __forceinline__ int next(const SpanTable& st, int s, int n_qsteps) {
    const int nr = bars->n_ranges;
    if (nr < 0) return walk.next(st, s + 1, n_qsteps);
    if (s + 1 < bars->rng[r][1]) return s + 1;
    ++r;
    return r < nr ? bars->rng[r][0] : n_qsteps;
  }
};
// Fill bars->rng / n_ranges (one warp, lanes over query spans): the steps overlapping any query span
// that sees a key span of the tile, merged into ranges.
__device__ __forceinline__ void build_ranges(const SpanTable& st, int k0, int n, BwdBars* bars, int lane) {
  const int ks_lo = span_of(st, k0), ks_hi = span_of(st, min(k0 + kBwdTile, n) - 1);
  int nr = 0, cur_lo = -1, cur_hi = -1;
  for (int q_base = 0; q_base < st.n; q_base += 32) {
    const int qs = q_base + lane;
    int lo = 0, hi = 0;
    if (qs < st.n) {
      bool v = false;
      for (int ks = ks_lo; ks <= ks_hi; ++ks) v |= span_vis(st, qs, ks);
      if (v && st.start[qs + 1] > st.start[qs]) {
        lo = st.start[qs] / kQStep;
        hi = (st.start[qs + 1] - 1) / kQStep + 1;
      }
    }
    uint32_t m = __ballot_sync(0xffffffffu, hi > lo);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const int l = __shfl_sync(0xffffffffu, lo, j), h = __shfl_sync(0xffffffffu, hi, j);
      if (cur_lo >= 0 && l <= cur_hi) {
        cur_hi = max(cur_hi, h);
      } else {
        if (cur_lo >= 0) {
          if (lane == 0 && nr < kMaxRanges) {
            bars->rng[nr][0] = cur_lo;
            bars->rng[nr][1] = cur_hi;
          }
          ++nr;
        }
        cur_lo = l;
        cur_hi = h;
      }
    }
  }
  if (cur_lo >= 0) {
    if (lane == 0 && nr < kMaxRanges) {
      bars->rng[nr][0] = cur_lo;
      bars->rng[nr][1] = cur_hi;
    }
    ++nr;
  }
  if (lane == 0) bars->n_ranges = nr <= kMaxRanges ? nr : -1;
}
// queries of [q0, q0 + 64) visible to a key of span ks (kc_ks = st.kc[ks]) as a 64-bit mask (two
// words); qc = the query span holding q0
__device__ __forceinline__ void visible_queries(const SpanTable& st, int ks, int kc_ks, int qc, int q0, int n,
                                                uint32_t (&m)[2]) {
  m[0] = m[1] = 0u;
  const int q1 = min(q0 + kQStep, n);
  for (int qs = qc; qs < st.n && st.start[qs] < q1; ++qs) {
    if (!(qs == ks || kc_ks < st.qth[qs])) continue;
    const int a = max(st.start[qs], q0) - q0, b = min(st.start[qs + 1], q1) - q0;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const int lo = min(max(a - 32 * w, 0), 32), hi = min(max(b - 32 * w, 0), 32);
      if (hi > lo) m[w] |= (hi == 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~(lo == 32 ? 0xffffffffu : ((1u << lo) - 1u));
    }
  }
}

// descriptors: K-major view (rows = M or N, 16-element K-steps along the 128-byte rows, boxes of 64
// columns box_bytes apart) and MN-major view (rows = K, 16-row K-steps, 64-column blocks box_bytes apart)
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int kk, uint32_t box_bytes) {
  return ptx::sdesc_sw128(tile + (kk / 4) * box_bytes + (kk % 4) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int kk, uint32_t box_bytes) {
  return ptx::sdesc_sw128(tile + kk * 16 * 128, box_bytes, 1024);
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq,
                    const float* __restrict__ lse2, const float* __restrict__ delta, float* __restrict__ dq_acc,
                    float* __restrict__ dk_out, __nv_bfloat16* __restrict__ dv_out, int B, int H, int n, int n_pad,
                    float scale_q, float scale_k, const __grid_constant__ SpanTable st) {
  extern __shared__ uint8_t smem_raw[];
#ifdef DZ_BWD_TRACE
  const bool bt_on = blockIdx.x == (unsigned)g_bwd_trace_cta;
#endif
  if (threadIdx.x == 0) BT(0, 15);
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + kOffBar);
  const float* vec = reinterpret_cast<const float*>(smem + kOffVec);  // [buffer][lse2 | delta][64]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_ktiles = (n + kBwdTile - 1) / kBwdTile, n_qsteps = (n + kQStep - 1) / kQStep;
  const int kt = blockIdx.x % n_ktiles, bh = blockIdx.x / n_ktiles, h = bh % H, b = bh / H;
  const int k0 = kt * kBwdTile;
  auto bar = [&](uint64_t& x) { return ptx::smem_u32(&x); };

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(bars->kv_full), 1);
    for (int i = 0; i < kQStages; ++i) {
      ptx::mbar_init(bar(bars->q_full[i]), 1);
      ptx::mbar_init(bar(bars->q_empty[i]), 1);
    }
    ptx::mbar_init(bar(bars->dq_full), 1);
    ptx::mbar_init(bar(bars->dq_free), 4);
    ptx::mbar_init(bar(bars->s_full), 1);
    ptx::mbar_init(bar(bars->s_read), kCompWarps);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(bar(bars->p_ready[i]), kCompWarps);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(bar(bars->mma_done[i]), 1);
    ptx::fence_mbar_init();
  }
  if (warp == kWarpProd) ptx::tmem_alloc<512>(ptx::smem_u32(&bars->tmem_base));
  if (warp == 0) build_ranges(st, k0, n, bars, lane);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::pdl_wait();
  const uint32_t tmem = bars->tmem_base;
#ifdef DZ_BWD_TRACE
  if (threadIdx.x == 0) {
    BT_CTA(0, bt_gtime());
    BT_CTA(3, bt_smid());
    BT(0, 13);
  }
#endif
  // TMEM: S^T [0, 64), dP^T [64, 128) (one step at a time: the next step's are computed once these are in
  // registers), dQ^T of step i in [128 + 64 (i & 1), +64) (drained while later steps run), dV [256, 384),
  // dK [384, 512)
  constexpr uint32_t kS = 0, kDP = 64, kDQ = 128, kPT = 192, kDV = 256, kDK = 384;
  const uint64_t pol = ptx::l2_policy_evict_last();
  const int64_t vrow = ((int64_t)b * H + h) * n_pad;  // lse2 / delta row of (b, h)

  if (warp == kWarpProd) {
    // ------------------------------------------------------------ TMA producer --
    if (lane == 0) {
      ptx::mbar_arrive_expect_tx(bar(bars->kv_full), 2 * kKTile);
      for (int x = 0; x < 2; ++x) {
        ptx::tma_load_4d(base + kOffK + x * kKBox, &tm_k, bar(bars->kv_full), x * 64, h, k0, b, pol);
        ptx::tma_load_4d(base + kOffV + x * kKBox, &tm_v, bar(bars->kv_full), x * 64, h, k0, b, pol);
      }
      uint32_t i = 0;
      Steps steps(bars, st, k0, n);
      for (int qs = steps.first(st, n_qsteps); qs < n_qsteps; qs = steps.next(st, qs, n_qsteps)) {
        const uint32_t bi = i % kQStages, u = i / kQStages;
        ptx::mbar_wait(bar(bars->q_empty[bi]), (u & 1) ^ 1);
        BT(i, 10);
        const uint32_t qb = base + kOffQ + bi * kQTile, ob = base + kOffDO + bi * kQTile;
        ptx::mbar_arrive_expect_tx(bar(bars->q_full[bi]), 2 * kQTile + 2 * kQStep * 4);
        for (int x = 0; x < 2; ++x) {
          ptx::tma_load_4d(qb + x * kQBox, &tm_q, bar(bars->q_full[bi]), x * 64, h, qs * kQStep, b, pol);
          ptx::tma_load_4d(ob + x * kQBox, &tm_do, bar(bars->q_full[bi]), x * 64, h, qs * kQStep, b, pol);
        }
        const uint32_t vb = base + kOffVec + bi * 512;
        ptx::bulk_load(vb, lse2 + vrow + qs * kQStep, kQStep * 4, bar(bars->q_full[bi]), pol);
        ptx::bulk_load(vb + 256, delta + vrow + qs * kQStep, kQStep * 4, bar(bars->q_full[bi]), pol);
        ++i;
      }
    }
    __syncwarp();
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------- MMA issuer --
    // The whole warp runs the loop; ptx::mma_ss_warp / tc_commit_warp elect the issuing lane inside the
    // asm (a lane-0 branch costs a per-MMA elect loop: ~63 vs ~40 cycles per issued MMA, measured in
    // tools/mma_bench.cu).  Software-pipelined: S^T / dP^T of step i + 1 are issued before waiting for
    // step i's P^T / dS^T, so the tensor pipe computes them while the softmax-gradient warps work on
    // step i, and they complete before step i's dV / dK / dQ^T, issued after them (one issuing thread:
    // the pipe runs its MMAs in this order).  Descriptors are formed once; a K-step only moves the start
    // address field (bits [0,14), address >> 4), which never carries for shared-memory addresses.
    constexpr uint32_t iS = ptx::idesc_f16(0, 0, 0, 0, 128, 64), iDP = ptx::idesc_f16(1, 1, 0, 0, 128, 64),
                       iDV = ptx::idesc_f16(1, 1, 0, 1, 128, 128), iDK = ptx::idesc_f16(0, 0, 0, 1, 128, 128),
                       iDQ = ptx::idesc_f16(0, 0, 1, 1, 128, 64);
    auto koff = [](int kk, uint32_t box) { return (uint64_t)(((kk / 4) * box + (kk % 4) * 32) >> 4); };
    auto moff = [](int kk) { return (uint64_t)((kk * 16 * 128) >> 4); };
    const uint64_t dK = desc_k(base + kOffK, 0, kKBox), dV = desc_k(base + kOffV, 0, kKBox),
                   dKm = desc_mn(base + kOffK, 0, kKBox);
    ptx::mbar_wait(bar(bars->kv_full), 0);
    auto issue_sdp = [&](uint32_t i) {
      const uint32_t bi = i % kQStages, u = i / kQStages;
      const uint64_t dQ = desc_k(base + kOffQ + bi * kQTile, 0, kQBox), dO = desc_k(base + kOffDO + bi * kQTile, 0, kQBox);
      if (lane == 0) BT(i, 0);
      ptx::mbar_wait(bar(bars->q_full[bi]), u & 1);
      if (lane == 0) BT(i, 11);
      if (i >= 1) ptx::mbar_wait(bar(bars->s_read), (i - 1) & 1);  // S^T / dP^T of step i - 1 are in registers
      if (lane == 0) BT(i, 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ptx::mma_ss_warp(tmem + kS, dK + koff(kk, kKBox), dQ + koff(kk, kQBox), iS, kk > 0);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ptx::mma_ss_warp(tmem + kDP, dV + koff(kk, kKBox), dO + koff(kk, kQBox), iDP, kk > 0);
      ptx::tc_commit_warp(bar(bars->s_full));
      if (lane == 0) BT(i, 16);
    };
    // (the walk runs one step ahead: the step after next is found while this step's P^T / dS^T are
    // being computed, off the issue path)
    Steps steps(bars, st, k0, n);
    int qs = steps.first(st, n_qsteps);
    int qn = qs < n_qsteps ? steps.next(st, qs, n_qsteps) : n_qsteps;
    if (qs < n_qsteps) issue_sdp(0);
    for (uint32_t i = 0; qs < n_qsteps; ++i) {
      const uint32_t bi = i & 1, qi = i % kQStages;
      if (qn < n_qsteps) issue_sdp(i + 1);  // (waits until step i's S^T / dP^T have been read)
      const int qnn = qn < n_qsteps ? steps.next(st, qn, n_qsteps) : n_qsteps;
      const uint64_t dQm = desc_mn(base + kOffQ + qi * kQTile, 0, kQBox), dOm = desc_mn(base + kOffDO + qi * kQTile, 0, kQBox);
      const uint64_t dST = desc_k(base + kOffDST + bi * kPTile, 0, kPTile), dSTm = desc_mn(base + kOffDST + bi * kPTile, 0, kPTile);
      // P^T (TMEM) and dS^T (shared memory) of step i are written.  One barrier per buffer: the
      // softmax-gradient warps may arrive for step i + 1 before this wait (they wait only for step i - 1's
      // MMAs), never for step i + 2 (that needs step i's MMAs)
      ptx::mbar_wait(bar(bars->p_ready[bi]), (i >> 1) & 1);
      if (lane == 0) BT(i, 12);
      ptx::tc_fence_after();
      // dV += P^T dO with A = P^T from TMEM (lane = key, 16-bit pairs along the queries), dK += dS^T Q'
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::mma_ts_warp(tmem + kDV, tmem + kPT + bi * 32 + kk * 8, dOm + moff(kk), iDV, (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        ptx::mma_ss_warp(tmem + kDK, dST + koff(kk, kPTile), dQm + moff(kk), iDK, (i > 0 || kk > 0) ? 1u : 0u);
      ptx::tc_commit_warp(bar(bars->q_empty[qi]));  // the last reads of this Q' / dO stage (dQ^T does not use it)
      if (i >= 1) {
        ptx::mbar_wait(bar(bars->dq_free), (i - 1) & 1);  // dQ^T(i - 1) has left TMEM
        ptx::tc_fence_after();
      }
      if (lane == 0) BT(i, 2);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) ptx::mma_ss_warp(tmem + kDQ, dKm + moff(kk), dSTm + moff(kk), iDQ, kk > 0);
      ptx::tc_commit_warp(bar(bars->mma_done[bi]));
      ptx::tc_commit_warp(bar(bars->dq_full));
      if (lane == 0) BT(i, 17);
      qs = qn;
      qn = qnn;
    }
    __syncwarp();
  } else if (warp >= kWarpDrain) {
    // ---------------------------------------------------------------- dQ drain --
    // dQ^T of step i (thread = d row r, all 64 queries) leaves TMEM once its MMAs complete (dq_full; the
    // next dQ^T MMAs wait for dq_free, so a drain can never fall a phase behind) and TMEM is released at
    // once; then the values go transposed into the staging tile [64 q][128 d] fp32 (thread r writes
    // column r: conflict-free) once the previous reduce has read it, and one TMA bulk reduce-add adds
    // the tile into dQ'[b][q0 .. q0 + 63][h][:] (rows past n clipped) while the next steps run.
    const int quad = warp % 4;
    const int r = quad * 32 + lane;
    const uint32_t lb = (uint32_t)(quad * 32) << 16;
    const uint32_t sb = base + kOffDQ;
    const bool leader = warp == kWarpDrain && lane == 0;
    Steps steps(bars, st, k0, n);
    uint32_t i = 0;
    for (int qs = steps.first(st, n_qsteps); qs < n_qsteps; qs = steps.next(st, qs, n_qsteps), ++i) {
      ptx::mbar_wait(bar(bars->dq_full), i & 1);
      ptx::tc_fence_after();
      uint32_t qa[32], qb[32];
      ptx::tmem_ld32(tmem + lb + kDQ, qa);
      ptx::tmem_ld32(tmem + lb + kDQ + 32, qb);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->dq_free));  // TMEM may take dQ^T(i + 1)
      if (leader) ptx::bulk_wait_read_all();                // the previous reduce has read the staging tile
      ptx::named_bar_sync(1, 128);
      if (leader) BT(i, 8);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + (j * 128 + r) * 4), "r"(qa[j]) : "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + ((32 + j) * 128 + r) * 4), "r"(qb[j]) : "memory");
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 128);
      if (leader) {
        ptx::tma_reduce_add_4d(&tm_dq, sb, 0, h, qs * kQStep, b);
        ptx::bulk_commit_group();
        BT(i, 7);
      }
    }
    if (leader) ptx::bulk_wait_all();  // the dQ reduces have completed
  } else {  // warps 0 .. kCompWarps - 1
    // ------------------------------------------ softmax gradient and epilogue --
    // warp w: TMEM lane quadrant w % 4 (key rows), query slice hq = w / 4 (kQW queries) of each step
    const int quad = warp % 4, hq = warp / 4;
    const int r = quad * 32 + lane;
    const uint32_t lb = (uint32_t)(quad * 32) << 16;
    const int key = k0 + r;
    const int ks = span_of(st, min(key, n - 1)), kc_ks = st.kc[ks];
    uint32_t i = 0;
    // (the walk and the visibility mask run one step ahead, while the step's math hides their
    // parameter-space loads)
    Steps steps(bars, st, k0, n);
    int qc = 0;  // query span holding the step's first query (only moves forward)
    auto step_mask = [&](int s) {
      const int q0 = s * kQStep;
      while (qc + 1 < st.n && st.start[qc + 1] <= q0) ++qc;
      uint32_t m[2];
      visible_queries(st, ks, kc_ks, qc, q0, n, m);
      const uint32_t wbits = (m[(hq * kQW) / 32] >> ((hq * kQW) % 32)) & (kQW == 32 ? 0xffffffffu : ((1u << kQW) - 1u));
      return key < n ? wbits : 0u;
    };
    int qs = steps.first(st, n_qsteps);
    uint32_t vm = qs < n_qsteps ? step_mask(qs) : 0u;
    while (qs < n_qsteps) {
      const uint32_t qi = i % kQStages, uq = i / kQStages;
      ptx::mbar_wait(bar(bars->q_full[qi]), uq & 1);    // this step's lse2 / delta are in shared memory
      ptx::mbar_wait(bar(bars->s_full), i & 1);
      if (threadIdx.x == 0) BT(i, 3);
      ptx::tc_fence_after();
      uint32_t sr[kQW], dr[kQW];
      if constexpr (kQW == 32) {
        ptx::tmem_ld32(tmem + lb + kS + hq * kQW, *reinterpret_cast<uint32_t(*)[32]>(sr));
        ptx::tmem_ld32(tmem + lb + kDP + hq * kQW, *reinterpret_cast<uint32_t(*)[32]>(dr));
      } else {
        ptx::tmem_ld16(tmem + lb + kS + hq * kQW, *reinterpret_cast<uint32_t(*)[16]>(sr));
        ptx::tmem_ld16(tmem + lb + kDP + hq * kQW, *reinterpret_cast<uint32_t(*)[16]>(dr));
      }
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->s_read));  // the next step's S^T / dP^T may be computed
      if (threadIdx.x == 0) BT(i, 4);
      const float4* lv = reinterpret_cast<const float4*>(vec + qi * 128 + hq * kQW);  // lse2 [64] | delta [64]
      uint32_t pk[kQW / 2], dk[kQW / 2];
      // pairs of queries in packed fp32x2 arithmetic, 2^x on MUFU (moving 1-4 pairs in 8 to the FMA-pipe
      // polynomial measured slower: the warps are bound by their instruction count, not by MUFU)
#pragma unroll
      for (int j4 = 0; j4 < kQW / 4; ++j4) {
        const float4 l4 = lv[j4], d4 = lv[16 + j4];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int j = 2 * j4 + h2, q = 2 * j;
          const float la = h2 ? l4.z : l4.x, lb2 = h2 ? l4.w : l4.y, da = h2 ? d4.z : d4.x, db = h2 ? d4.w : d4.y;
          // masked pairs (Fig. 10, queries or keys past n) get s = -inf: p = 2^-inf = 0 and dS = 0 x
          // (dP - delta) = 0 (dP and delta are finite: dO rows past n load as zeros, delta is padded)
          const float s0m = ((vm >> q) & 1u) ? __uint_as_float(sr[q]) : -INFINITY,
                      s1m = ((vm >> (q + 1)) & 1u) ? __uint_as_float(sr[q + 1]) : -INFINITY;
          const uint64_t x = ptx::f2_add(ptx::f2_pack(s0m, s1m), ptx::f2_pack(-la, -lb2));
          float x0, x1;
          ptx::f2_unpack(x, x0, x1);
          const uint64_t p = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
          const uint64_t dd = ptx::f2_add(ptx::f2_pack(__uint_as_float(dr[q]), __uint_as_float(dr[q + 1])),
                                          ptx::f2_pack(-da, -db));
          const uint64_t ds = ptx::f2_mul(p, dd);
          float p0, p1, s0, s1;
          ptx::f2_unpack(p, p0, p1);
          ptx::f2_unpack(ds, s0, s1);
          pk[j] = ptx::pack_bf16x2(p0, p1);
          __half2 hh = __floats2half2_rn(s0, s1);
          dk[j] = *reinterpret_cast<uint32_t*>(&hh);
        }
      }
      if (threadIdx.x == 0) BT(i, 5);
      const uint32_t pb = i & 1;  // P^T / dS^T buffer: free once the MMAs of step i - 2 are done
      if (i >= 2) {
        ptx::mbar_wait(bar(bars->mma_done[pb]), ((i >> 1) - 1) & 1);
        ptx::tc_fence_after();
      }
      // P^T into TMEM (A of the dV MMA: 16-bit pairs, query 2c in the low half of column c), dS^T into
      // shared memory (A of dK, K-major, and B of dQ^T, MN-major; SW128 rows of 64 queries)
      if constexpr (kQW == 32)
        ptx::tmem_st16(tmem + lb + kPT + pb * 32 + hq * (kQW / 2), *reinterpret_cast<uint32_t(*)[16]>(pk));
      else
        ptx::tmem_st8(tmem + lb + kPT + pb * 32 + hq * (kQW / 2), *reinterpret_cast<uint32_t(*)[8]>(pk));
#pragma unroll
      for (int j = 0; j < kQW / 8; ++j) {  // row r of the [128][64] tile: this warp's chunks of 8 queries, SW128
        const uint32_t o = r * 128 + (((hq * (kQW / 8) + j) ^ (r & 7)) << 4);
        ptx::st_shared_v4(base + kOffDST + pb * kPTile + o, dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
      }
      ptx::tmem_wait_st();
      ptx::fence_proxy_async_smem();  // generic stores -> the tensor core's reads
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->p_ready[pb]));
      if (threadIdx.x == 0) BT(i, 6);
      // the next step and its visibility mask (parameter-space loads) while the MMAs run
      const int qs_next = steps.next(st, qs, n_qsteps);
      const uint32_t vm_next = qs_next < n_qsteps ? step_mask(qs_next) : 0u;
      ++i;
      qs = qs_next;
      vm = vm_next;
    }
    if (i >= 1) {  // the final dV / dK (the pipe completes the MMAs of step i - 1 last)
      ptx::mbar_wait(bar(bars->mma_done[(i - 1) & 1]), ((i - 1) >> 1) & 1);
      ptx::tc_fence_after();
    }
#ifdef DZ_BWD_TRACE
    if (threadIdx.x == 0) {
      BT_CTA(2, i);
      BT(1, 13);
    }
#endif
    // dV (bf16) and dK' (fp32) of this thread's key row, columns [128 / kQS hq, + 128 / kQS) (tcgen05.ld
    // is warp-collective: every lane loads, only rows < n store)
    const int64_t row = (((int64_t)b * n + min(key, n - 1)) * H + h) * 128;
    const bool store = key < n;
    if (i == 0) {  // no query sees these keys: zero gradients
      if (store)
        for (int d = hq * (128 / kQS); d < (hq + 1) * (128 / kQS); d += 8) {
          *reinterpret_cast<uint4*>(dv_out + row + d) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<float4*>(dk_out + row + d) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(dk_out + row + d + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
#pragma unroll 1
      for (int c = hq * (4 / kQS); c < (hq + 1) * (4 / kQS); ++c) {
        uint32_t vr[32], kr[32];
        ptx::tmem_ld32(tmem + lb + kDV + c * 32, vr);
        ptx::tmem_ld32(tmem + lb + kDK + c * 32, kr);
        ptx::tmem_wait_ld();
        if (!store) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          *reinterpret_cast<uint4*>(dv_out + row + c * 32 + 8 * j) =
              make_uint4(ptx::pack_bf16x2(__uint_as_float(vr[8 * j]), __uint_as_float(vr[8 * j + 1])),
                         ptx::pack_bf16x2(__uint_as_float(vr[8 * j + 2]), __uint_as_float(vr[8 * j + 3])),
                         ptx::pack_bf16x2(__uint_as_float(vr[8 * j + 4]), __uint_as_float(vr[8 * j + 5])),
                         ptx::pack_bf16x2(__uint_as_float(vr[8 * j + 6]), __uint_as_float(vr[8 * j + 7])));
#pragma unroll
          for (int e = 0; e < 8; e += 4)
            *reinterpret_cast<float4*>(dk_out + row + c * 32 + 8 * j + e) =
                make_float4(__uint_as_float(kr[8 * j + e]) * scale_k, __uint_as_float(kr[8 * j + e + 1]) * scale_k,
                            __uint_as_float(kr[8 * j + e + 2]) * scale_k, __uint_as_float(kr[8 * j + e + 3]) * scale_k);
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == kWarpProd) ptx::tmem_dealloc<512>(tmem);
#ifdef DZ_BWD_TRACE
  if (threadIdx.x == 0) {
    BT_CTA(1, bt_gtime());
    BT(0, 14);
  }
#endif
}

// B1: delta = <dO, O> per (b, h, s) row and lse2 = lse * log2(e); one warp per row of D = 128
// B1: 16 lanes per (b, s, h) row of D = 128 (8 elements, one 16-byte load of O and of dO each), two
// rows per warp instruction, kDeltaRows rows per warp with all loads issued before the reductions.
constexpr int kDeltaRows = 8;
__global__ void __launch_bounds__(256) delta_kernel(const __nv_bfloat16* __restrict__ dout,
                                                   const __nv_bfloat16* __restrict__ out, const float* __restrict__ lse,
                                                   float* __restrict__ delta, float* __restrict__ lse2, int B, int n,
                                                   int H, int n_pad) {
  const int64_t rows = (int64_t)B * n * H;
  const int64_t w0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32) * kDeltaRows;
  const int lane = threadIdx.x % 32, half = lane / 16, l16 = lane % 16;
  uint4 o[kDeltaRows / 2], g[kDeltaRows / 2];
#pragma unroll
  for (int k = 0; k < kDeltaRows / 2; ++k) {
    const int64_t wid = w0 + 2 * k + half;
    if (wid < rows) {
      o[k] = __ldg(reinterpret_cast<const uint4*>(out + wid * 128) + l16);
      g[k] = __ldg(reinterpret_cast<const uint4*>(dout + wid * 128) + l16);
    } else {
      o[k] = g[k] = make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int k = 0; k < kDeltaRows / 2; ++k) {
    const uint32_t ov[4] = {o[k].x, o[k].y, o[k].z, o[k].w}, gv[4] = {g[k].x, g[k].y, g[k].z, g[k].w};
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      acc = fmaf(__uint_as_float(ov[e] << 16), __uint_as_float(gv[e] << 16), acc);
      acc = fmaf(__uint_as_float(ov[e] & 0xFFFF0000u), __uint_as_float(gv[e] & 0xFFFF0000u), acc);
    }
#pragma unroll
    for (int m = 8; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    const int64_t wid = w0 + 2 * k + half;
    if (l16 == 0 && wid < rows) {  // rows of n_pad (a multiple of 64: the attention backward reads whole steps)
      const int h = (int)(wid % H), s = (int)((wid / H) % n), b = (int)(wid / ((int64_t)H * n));
      const int64_t i = ((int64_t)b * H + h) * n_pad + s;
      delta[i] = acc;
      lse2[i] = lse[((int64_t)b * H + h) * n + s] * 1.4426950408889634f;
      if (s == n - 1)  // queries [n, n_pad): finite values, so masked scores (-inf) give p = 0 and dS = 0
        for (int e = 1; s + e < n_pad; ++e) delta[i + e] = lse2[i + e] = 0.f;
    }
  }
}

// B3: prologue backward for one tensor (blockIdx.z: 0 q, 1 k) -- per (token, head) row of D = 128,
// one warp per row, 4 elements (2 rotation pairs) per lane:
//   dy = R(-phi) dx';  dgain += dy * x^;  dx^ = dy * g;  dx = (dx^ - x^ mean(dx^ x^)) / r
// A CTA handles one head and a run of tokens; its gain gradient is reduced in shared memory and
// added once (fp32 atomics).
struct ProBwdArgs {
  const __nv_bfloat16* x[2];  // raw q, k [B][n][H][D]
  const float* dxp[2];        // dq', dk' fp32 [B][n][H][D], times dscale[w]
  float dscale[2];
  const float* gain[2];       // [H][D]
  __nv_bfloat16* dx[2];       // dq, dk bf16 [B][n][H][D]
  float* dgain[2];            // [H][D], accumulated
  const int32_t* pos;         // [n][3]
  const float2* tab;          // RoPE table [tab_len][D/2]
  int32_t tab_len;
  float eps;
  int32_t B, n, H;
  double omega[64];
  int8_t axis[64];
};
constexpr int kProBwdTokens = 64;

#ifndef DZ_PB_R  // rows per warp pass / CTAs per SM: 2 / 4 measured best (64 registers, no spills)
#define DZ_PB_R 2
#define DZ_PB_MIN 4
#endif
__global__ void __launch_bounds__(256, DZ_PB_MIN) prologue_bwd_kernel(const __grid_constant__ ProBwdArgs a) {
  constexpr int D = 128, R = DZ_PB_R;  // R rows per warp pass: all their loads are issued before the math
  // blockIdx.x = head (fastest: CTAs running together read the neighbouring heads of the same tokens,
  // whole [H][D] rows of the token-major tensors), blockIdx.y = run of tokens, blockIdx.z = q / k
  const int w = blockIdx.z, h = blockIdx.x, tb = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int j0 = 2 * lane;  // this lane's rotation pairs j0, j0 + 1 (elements 4 lane .. 4 lane + 3)
  const float* gp = a.gain[w] + h * D + 4 * lane;
  const float g4[4] = {gp[0], gp[1], gp[2], gp[3]};
  float dg[4] = {0.f, 0.f, 0.f, 0.f};
  const int ax0 = a.axis[j0], ax1 = a.axis[j0 + 1];
  const int items = a.B * a.n, it_end = min(items, (tb + 1) * kProBwdTokens);
  for (int it0 = tb * kProBwdTokens + warp * R; it0 < it_end; it0 += 8 * R) {
    uint2 xr[R];
    float4 d4[R];
    int p0[R], p1[R];
    int64_t row[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int it = min(it0 + k, it_end - 1);
      const int b = it / a.n, t = it - b * a.n;
      row[k] = (((int64_t)b * a.n + t) * a.H + h) * D + 4 * lane;
      xr[k] = __ldg(reinterpret_cast<const uint2*>(a.x[w] + row[k]));
      d4[k] = __ldcs(reinterpret_cast<const float4*>(a.dxp[w] + row[k]));
      p0[k] = __ldg(a.pos + 3 * t + ax0);
      p1[k] = __ldg(a.pos + 3 * t + ax1);
    }
    float2 c0[R], c1[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      c0[k] = (unsigned)p0[k] < (unsigned)a.tab_len ? __ldg(a.tab + (size_t)p0[k] * (D / 2) + j0)
                                                  : make_float2((float)cos(p0[k] * a.omega[j0]), (float)sin(p0[k] * a.omega[j0]));
      c1[k] = (unsigned)p1[k] < (unsigned)a.tab_len
                  ? __ldg(a.tab + (size_t)p1[k] * (D / 2) + j0 + 1)
                  : make_float2((float)cos(p1[k] * a.omega[j0 + 1]), (float)sin(p1[k] * a.omega[j0 + 1]));
    }
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (it0 + k >= it_end) break;
      const float x4[4] = {__uint_as_float(xr[k].x << 16), __uint_as_float(xr[k].x & 0xFFFF0000u),
                           __uint_as_float(xr[k].y << 16), __uint_as_float(xr[k].y & 0xFFFF0000u)};
      float ss = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) ss = fmaf(x4[e], x4[e], ss);
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
      const float inv = rsqrtf(ss * (1.0f / D) + a.eps);
      // dy = R(-phi) dx' per pair
      const float sc = a.dscale[w];
      const float4 dd = make_float4(d4[k].x * sc, d4[k].y * sc, d4[k].z * sc, d4[k].w * sc);
      const float dy[4] = {dd.x * c0[k].x + dd.y * c0[k].y, -dd.x * c0[k].y + dd.y * c0[k].x,
                           dd.z * c1[k].x + dd.w * c1[k].y, -dd.z * c1[k].y + dd.w * c1[k].x};
      float xh[4], dxh[4], dot = 0.f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xh[e] = x4[e] * inv;
        dg[e] = fmaf(dy[e], xh[e], dg[e]);
        dxh[e] = dy[e] * g4[e];
        dot = fmaf(dxh[e], xh[e], dot);
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, m);
      const float mdot = dot * (1.0f / D);
      float dx[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) dx[e] = (dxh[e] - xh[e] * mdot) * inv;
      __stcs(reinterpret_cast<uint2*>(a.dx[w] + row[k]),
             make_uint2(ptx::pack_bf16x2(dx[0], dx[1]), ptx::pack_bf16x2(dx[2], dx[3])));
    }
  }
  __shared__ float red[8][D];
#pragma unroll
  for (int e = 0; e < 4; ++e) red[warp][4 * lane + e] = dg[e];
  __syncthreads();
  if (threadIdx.x < D) {
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += red[i][threadIdx.x];
    atomicAdd(a.dgain[w] + h * D + threadIdx.x, s);
  }
}

}  // namespace

cudaError_t launch_attention_backward(const BwdArgs& a, cudaStream_t s) {
  if (a.D != 128) return cudaErrorInvalidValue;
  // B1
  {
    const int64_t warps = ((int64_t)a.B * a.n * a.H + kDeltaRows - 1) / kDeltaRows;
    const int threads = 256;
    delta_kernel<<<(unsigned)((warps * 32 + threads - 1) / threads), threads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(a.dout), static_cast<const __nv_bfloat16*>(a.out), a.lse, a.delta, a.lse2,
        a.B, a.n, a.H, a.n_pad);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // B2
  {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.n + kBwdTile - 1) / kBwdTile;
    e = launch_pdl(attn_bwd_kernel, dim3((unsigned)(a.B * a.H * tiles)), dim3(kBwdThreads), (size_t)kBwdSmem, s,
                   a.tm_k, a.tm_v, a.tm_q, a.tm_do, a.tm_dq, a.lse2, a.delta, a.dq_acc, a.dk,
                   static_cast<__nv_bfloat16*>(a.dv),
                   a.B, a.H, a.n, a.n_pad, a.scale_q, a.scale_k, a.spans);
    if (e != cudaSuccess) return e;
  }
  // B3
  {
    ProBwdArgs p;
    p.x[0] = static_cast<const __nv_bfloat16*>(a.q_raw);
    p.x[1] = static_cast<const __nv_bfloat16*>(a.k_raw);
    p.dxp[0] = a.dq_acc;
    p.dxp[1] = a.dk;
    p.dscale[0] = a.scale_q;  // dQ' accumulates K'^T dS^T unscaled
    p.dscale[1] = 1.f;        // dK' is scaled in the attention epilogue
    p.gain[0] = a.gain[0];
    p.gain[1] = a.gain[1];
    p.dx[0] = static_cast<__nv_bfloat16*>(a.dq);
    p.dx[1] = static_cast<__nv_bfloat16*>(a.dk_raw);
    p.dgain[0] = a.dgain[0];
    p.dgain[1] = a.dgain[1];
    p.pos = a.pos;
    p.tab = a.tab;
    p.tab_len = a.tab_len;
    p.eps = a.eps;
    p.B = a.B;
    p.n = a.n;
    p.H = a.H;
    for (int j = 0; j < 64; ++j) {
      p.omega[j] = a.omega[j];
      p.axis[j] = a.axis[j];
    }
    const unsigned blocks = (unsigned)((a.B * a.n + kProBwdTokens - 1) / kProBwdTokens);
    prologue_bwd_kernel<<<dim3((unsigned)a.H, blocks, 2), 256, 0, s>>>(p);
    return cudaGetLastError();
  }
}

}  // namespace dz

#ifdef DZ_BWD_TRACE
// diagnostics build only: cta >= 0 arms the trace for that CTA; cta < 0 reads it ([128][24] words)
extern "C" __attribute__((visibility("default"))) int dz_debug_bwd_trace(int cta, uint32_t* host) {
  if (cta >= 0) {
    static uint32_t z[128 * 24];
    cudaMemcpyToSymbol(dz::g_bwd_trace, z, sizeof z);
    return (int)cudaMemcpyToSymbol(dz::g_bwd_trace_cta, &cta, sizeof(int));
  }
  if (cta == -2) return (int)cudaMemcpyFromSymbol(host, dz::g_bwd_cta, sizeof(uint32_t) * 4096 * 4);
  if (cta == -3) return (int)cudaMemcpyFromSymbol(host, dz::ptx::g_dz_watchdog, sizeof(uint32_t) * 8);
  return (int)cudaMemcpyFromSymbol(host, dz::g_bwd_trace, sizeof(uint32_t) * 128 * 24);
}
#endif
