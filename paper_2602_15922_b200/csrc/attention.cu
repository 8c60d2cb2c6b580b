// attention.cu -- K2: block-causal chunk attention on tcgen05 tensor cores, CTA pairs.
//
// Computes, for every (b, h, query s) of the new tokens,
//     O_s = sum_j softmax_j(<q'_s, k'_j> * scale) v_j
// over the visible keys j: the committed clean chunks plus the new tokens under the
// Fig. 10 rule (Alg. 2 l.584-585; BJ:5).  For attend_chunk every
// committed key and every own-chunk key is visible, so the only masked pairs are the
// out-of-bounds columns of the last key step.
//
// Work unit: a cluster of two CTAs (one SM each, same TPC) owns (batch, head, query
// group of 256 rows); CTA r keeps q-tile 2g + r in shared memory.  Every MMA is
// tcgen05.mma.cta_group::2 (M = 256: 128 rows per CTA), issued by one thread of the
// leader CTA, fp32 accumulators in TMEM:
//   S = Q K_j^T   SS, f16 x f16 -> f32; each CTA supplies its 128 query rows and half
//                 of the step's keys
//   O += P V_j    TS, P bf16 from TMEM; each CTA supplies D/2 of V's columns
// so each byte of K and V in shared memory is read by one SM.
//
// Two variants:
//   * ping-pong (fixed softmax base, the production path): 128-key steps; TMEM per CTA
//     S[2] [0,256) fp32, P[2] [256,384) bf16 pairs, O [384,512).  The two softmax warp
//     groups take alternate steps; S is released as soon as it is in registers, P has
//     its own double buffer, so the tensor pipe holds the next QK and the previous PV.
//   * lock-step (online base): 256-key steps split in two 128-key halves between the
//     groups, which exchange row maxima and rescale O lazily.
//
// Warps per CTA (12):
//   11     QK issuer (leader CTA)
//   10     K (+Q) TMA producer (both CTAs; bytes counted on the leader's barriers)
//   9      PV issuer (leader CTA)
//   8      TMEM allocator, then V TMA producer
//   0..7   softmax + epilogue: warp w owns TMEM lanes 32*(w%4).. (query rows); ping-pong:
//          every other step (group w/4), lock-step: key half w/4; O columns (w/4)*D/2..
//          exp2 on MUFU.EX2 with 1 of every 8 pairs on an FMA-pipe polynomial.
// Schedule: stream-K over executed steps (one span: the first units dealt whole,
// round-robin), pieces of split units combined in key order by the last to finish.
// Epilogue: O through swizzled shared memory and one TMA tensor store per warp.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "ptx.cuh"

namespace dz {
namespace {

constexpr int BM = 128;           // query rows per CTA (MMA M = 256 per pair)
constexpr int BN = 256;           // keys per KV step
constexpr int kThreads = 384;     // 12 warps
constexpr float kRescaleLog2 = 8.0f;
#ifndef DZ_POLY
#define DZ_POLY 2
#endif
// of every 16 exp2 pairs, this many go to the FMA-pipe polynomial (measured on the current ping-pong
// kernel at C1: 0/1/2/3/4/6 of 16 -> 179.5/174.1/174.1/175.5/176.1/179.1 us)
constexpr int kPolyPairs = DZ_POLY;
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;
constexpr int kWarpMma = 11, kWarpTma = 10, kWarpPv = 9, kWarpTmem = 8;
// setmaxnreg split, 128 * light + 256 * softmax = 384 * 168 (launch): ping-pong 104/200 (measured on
// C1: 88/208 182.8 us, 104/200 178.0, 120/192 179.7), lock-step 72/216 (its softmax holds more state;
// C1 forced online: 56/224 244.0 us, 72/216 234.0, 88/208 244.2; light must be 8 mod 16)
template <bool PP> __host__ __device__ constexpr uint32_t regs_light() { return PP ? 104 : 88; }
template <bool PP> __host__ __device__ constexpr uint32_t regs_softmax() { return PP ? 200 : 208; }

// Cycle trace of cluster 0's first unit (diagnostics, dz_debug_trace), per CTA
// rank r at [r * 16 * kTraceSteps]: per step j [8j+0,1] QK wait/issue,
// [8j+2,3] PV wait/issue (of step j), [8j+4,5] softmax S-ready / P-done
// (warp 0), [8j+6] S loaded, [8j+7] exp done.
#ifdef DZ_TRACE
constexpr bool kTrace = true;   // diagnostics build (libdz_trace.so): cycle trace + per-CTA timeline
#else
constexpr bool kTrace = false;  // production build: every trace statement below compiles away
#endif
constexpr int kTraceSteps = 256;
#ifndef DZ_SP
#define DZ_SP 0
#endif
// scheduling points of the softmax loop (experiment switch DZ_SP)
#if DZ_SP == 1
#define SCHED_POINT() do { uint32_t c_; asm volatile("mov.u32 %0, %%clock;" : "=r"(c_)); } while (0)
#elif DZ_SP == 2
#define SCHED_POINT() do { if (g_dz_trace_on == 12345) asm volatile("trap;"); } while (0)
#else
#define SCHED_POINT() do { } while (0)
#endif
__device__ uint32_t g_dz_trace[kTraceSteps * 32];
__device__ int g_dz_trace_on;
// Per-CTA timeline (globaltimer ns, low 32 bits), softmax warp 0 lane 0 of every CTA:
// [0] start, [1] end, [2] / [3] clock() at start / end, [4] segments, [5] combines; segment i < 14:
// [8 + 4i] start, [9 + 4i] last step's P written, [10 + 4i] O complete (o_full), [11 + 4i] end (clock()).
constexpr int kTimelineCtas = 160, kTimelineWords = 64, kTlSegs = 14;
__device__ uint32_t g_dz_timeline[kTimelineCtas * kTimelineWords];
// Effective SM clock under K2 (dz_debug_k2_clock): every CTA's thread 0 adds its SM's cycles and
// globaltimer nanoseconds from the end of the predecessor wait to the last cluster barrier.
__device__ unsigned long long g_dz_k2clk[2];
__device__ __forceinline__ uint64_t gtime64() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (uint32_t)t;
}

// PP (ping-pong, fixed softmax base): 128-key steps, S and P double-buffered, the two
// softmax warp groups take alternate steps.  !PP (online base): 256-key steps, each step
// split in two key halves between the two warp groups.
constexpr int kClsWords = kMaxStepTiles / 16;  // step-class table (several spans): at most 16 KB of shared memory

// F8 (DZ_FLAG_FP8_QK): Q' and K' are E4M3, one byte per element; QK^T by tcgen05.mma kind::f8f6f4
// (K = 32 per instruction), PV unchanged (bf16).
template <int D, bool PP, bool F8 = false>
struct Cfg {
  static constexpr int kBN = PP ? 128 : 256;               // keys per step
  static constexpr int kQKBytes = F8 ? 1 : 2;             // bytes per Q' / K' element
  static constexpr int kQBoxes = D * kQKBytes / 128;      // 128-byte SW128 boxes per Q / K row
  static constexpr int kBoxElems = 128 / kQKBytes;        // elements of a row per box
  static constexpr int kQTileBytes = BM * D * kQKBytes;   // one CTA's query tile
  static constexpr int kStageBytes = kBN * D;             // K (kBN/2 keys x D) or V (kBN keys x D/2) per CTA
  static constexpr int kKBytes = kBN / 2 * D * kQKBytes;  // bytes of a K stage one CTA loads
  static constexpr int kQKSteps = D * kQKBytes / 32;      // MMAs per QK (32 bytes of K per instruction)
#ifndef DZ_KST
#define DZ_KST 4   // measured on C1 (K/V stages), first kernel: 7/5 192.7 us, 6/4 190.3, 5/4 191.0, 5/3 190.0;
#endif               // current kernel: 6/3 176.5, 5/4 177.5, 5/3 175.4, 4/3 174.2, 4/2 176.8, 3/3 174.8, 3/2 176.9
#ifndef DZ_VST
#define DZ_VST 3
#endif
  // separate K and V rings: a V stage is held until its PV completes, several steps after
  // its QK, so a shared in-order ring would let V recycling throttle the K prefetch
  static constexpr int kKStages = (PP || D == 64) ? DZ_KST : 3;
  static constexpr int kVStages = (PP || D == 64) ? DZ_VST : 2;
  static constexpr int kStages = kKStages + kVStages;
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = kQTileBytes;
  static constexpr int kRedOff = kKVOff + kStages * kStageBytes;  // row max / row sum exchange [2][BM]
  static constexpr int kOOff = kRedOff + 2 * BM * 4;              // epilogue O staging: 8 warps x 32 rows x D/2 bf16
  static constexpr bool kTab = PP || D == 64;                     // static step-class table fits beside
  static constexpr int kBarOff = kOOff + 8 * 32 * D;
  static constexpr int kSmem = kBarOff + 1024 + 1024;             // + barriers/schedule + alignment slack
                                                                   // (+ the launch's step-class table)
  static_assert(kSmem + (kTab ? kClsWords * 4 : 0) <= 232448, "shared memory per CTA");
  static_assert(8 * 32 * D <= 32768 || !F8, "O staging");
  static constexpr uint32_t kIdescQK = ptx::idesc_f16(0, 0, 0, 0, 2 * BM, BN / 2);  // f16 x f16, K-major, per half
  static constexpr uint32_t kIdescPV = ptx::idesc_f16(1, 1, 0, 1, 2 * BM, D);   // P (TMEM) x V (MN-major)
  static constexpr int kVRowBytes = D;                      // V half row: D/2 bf16
};

constexpr int kMaxGroups = 64;    // stream-K schedule needs <= 64 query groups (16384 query rows)

struct Bars {
  uint64_t q_full, q_empty, s_full[2], s_free[2], p_full[2], p_empty[2], o_full, o_empty;
  uint64_t kv_full[12], kv_empty[12];
  uint64_t clk0, ns0;               // thread 0: SM clock64 / globaltimer after the predecessor wait
  uint32_t tmem_base;
  int32_t last_piece;               // combine election result (softmax warps)
  int32_t gpre[kMaxGroups + 1];     // prefix sums of executed steps per query group
  int32_t plo[kMaxPairs + 1];       // stream-K range boundaries of the CTA pairs (executed-step index)
};
static_assert(sizeof(Bars) <= 1024, "Bars must fit its shared-memory slot");

// p = 2^(x + nb) for 32 pairs of scores (already in log2 units); row-sum
// partials in acc, bf16 pairs in pk.
//   kMixed (fixed base, unmasked step: every x in [-60, 60], nb = 0): kPolyPairs
//     of every 16 pairs through the FMA-pipe polynomial, the rest through MUFU.EX2;
//   !kMixed (online base or masked step: x may be -inf): every pair through
//     MUFU.EX2 after adding nb (ex2(-inf) = +0 exactly, so masked keys add 0).
// Two variants only, to keep the softmax loop inside the instruction cache.
template <bool kMixed>
__device__ __forceinline__ void exp_half(const float* s, uint64_t nb2, uint32_t (&pk)[32], uint64_t (&acc)[4]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    uint64_t x = ptx::f2_pack(s[2 * i], s[2 * i + 1]);
    uint64_t p;
    if (kMixed && (i % 16) >= 16 - kPolyPairs) {
      p = ptx::f2_exp2_poly<false>(x);
    } else {
      if (!kMixed) x = ptx::f2_add(x, nb2);
      float x0, x1;
      ptx::f2_unpack(x, x0, x1);
      p = ptx::f2_pack(ptx::ex2(x0), ptx::ex2(x1));
    }
    acc[i % 4] = ptx::f2_add(acc[i % 4], p);
    float p0, p1;
    ptx::f2_unpack(p, p0, p1);
    pk[i] = ptx::pack_bf16x2(p0, p1);
  }
}

// ------------------------------------------------ Fig. 10 visibility (spans) --
// Every role of the kernel (TMA producer, both MMA issuers, softmax warps)
// evaluates the same pure functions below, so they agree on which steps run
// without exchanging anything.
constexpr uint8_t kSkip = 0, kPartial = 1, kFull = 2;  // oracle tile_map encoding

__device__ __forceinline__ bool span_vis(const SpanTable& st, int qs, int ks) {
  return qs == ks || st.kc[ks] < st.qth[qs];
}
// first span whose range ends after token x (x < start[n])
__device__ __forceinline__ int span_at(const SpanTable& st, int x) {
  int i = 0;
  while (i + 1 < st.n && st.start[i + 1] <= x) ++i;
  return i;
}
// Class of the (256-row query group g, 256-key step j) tile: SKIP if no
// (query, key) pair in it is visible, FULL if all are visible and in bounds,
// else PARTIAL.  Visibility is constant over a (query span, key span) pair, so
// the tile's class follows from the spans overlapping its row and key ranges.
// rows_in_bounds: judge only the rows < nq (the softmax's masking decision:
// rows past nq are computed but never stored, so they need no mask).
template <int TK>
__device__ __forceinline__ uint8_t step_class(const SpanTable& st, int g, int j, int nq, int kv_len, bool rows_in_bounds = false) {
  const int r0 = g * kTileQ, r1 = min(r0 + kTileQ, nq);
  const int k0 = j * TK, k1 = min(k0 + TK, kv_len);
  bool any = k0 < st.valid;  // committed keys are visible to every query
  bool all = (rows_in_bounds || r1 - r0 == kTileQ) && (k1 - k0 == TK);
  if (st.n == 1) return (any || k1 > st.valid) ? (all ? kFull : kPartial) : kSkip;
  if (k1 > st.valid) {
    const int ka = max(k0, st.valid) - st.valid, kb = k1 - st.valid;
    const int ks0 = span_at(st, ka);
    for (int qs = span_at(st, r0); qs < st.n && st.start[qs] < r1; ++qs)
      for (int ks = ks0; ks < st.n && st.start[ks] < kb; ++ks) {
        const bool v = span_vis(st, qs, ks);
        any |= v;
        all &= v;
      }
  }
  return !any ? kSkip : (all ? kFull : kPartial);
}
// Executed-step classes of the (query group, key step) tiles with several spans: 2 bits per tile
// (the rows_in_bounds class: SKIP, PARTIAL = needs a mask, FULL), built once per CTA in static
// shared memory so the single-thread roles (MMA issuers, TMA producers) never evaluate span loops
// on their critical path.  With one span, or a table too large, the class is evaluated on the fly.
// The table sits at the start of the dynamic shared memory, sized per launch (none with one span),
// so a single-span launch keeps those bytes for the K/V rings; the kernel's tiles follow it.
extern __shared__ __align__(16) uint32_t s_cls_tab[];
// bytes of the table for a launch (multiple of 16)
__host__ __device__ constexpr int cls_tab_bytes(bool tab, int n_spans, int n_groups, int nkv) {
  return (tab && n_spans != 1) ? ((n_groups * nkv + 63) / 64) * 16 : 0;
}
template <int TK, bool kTab>
__device__ __forceinline__ uint8_t cls_get(const SpanTable& st, int g, int j, int nq, int kv_len, int nkv) {
  if (kTab) {  // (the host rejects span layouts whose table would not fit: dz_attend_spans -> DZ_ESHAPE)
    const int x = g * nkv + j;
    return (uint8_t)((s_cls_tab[x >> 4] >> (2 * (x & 15))) & 3u);
  }
  return step_class<TK>(st, g, j, nq, kv_len, true);
}
// set bits [lo, hi) of a 128-bit mask
__device__ __forceinline__ void set_bits(uint32_t (&m)[4], int lo, int hi) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const int a = min(max(lo - 32 * w, 0), 32), b = min(max(hi - 32 * w, 0), 32);
    if (b > a) m[w] |= (b == 32 ? 0xffffffffu : ((1u << b) - 1u)) & ~((a == 32) ? 0xffffffffu : ((1u << a) - 1u));
  }
}
// Visible-key mask of query span qs over keys [kb0, kb0 + 128) of the key sequence.
__device__ __forceinline__ void visible_bits(const SpanTable& st, int qs, int kb0, int kv_len, uint32_t (&m)[4]) {
  m[0] = m[1] = m[2] = m[3] = 0u;
  const int kend = min(kb0 + 128, kv_len);
  set_bits(m, 0, min(st.valid, kend) - kb0);  // committed part
  if (kend <= st.valid) return;
  const int ka = max(kb0, st.valid) - st.valid, kb = kend - st.valid;
  for (int ks = span_at(st, ka); ks < st.n && st.start[ks] < kb; ++ks)
    if (span_vis(st, qs, ks))
      set_bits(m, max(st.start[ks], ka) + st.valid - kb0, min(st.start[ks + 1], kb) + st.valid - kb0);
}
// ------------------------------------------------------------ work schedule --
// Stream-K over executed steps: the sequence of (unit, executed step), units
// u = (b, h, g) in order and their non-SKIP steps in key order, is cut into
// ncl equal ranges, one per CTA pair, so every pair does the same number of
// steps (+-1) whatever the unit count.  A unit cut by a range boundary is
// computed in pieces, each a contiguous run of its steps; every piece writes
// its unnormalised O, row sum and base to the workspace and the last piece to
// finish (atomic count) combines them in key order -- deterministic, no
// waiting.  With more than kMaxGroups query groups the schedule falls back to
// whole units dealt round-robin.
struct Seg {
  int b, h, g;
  int k0, k1, cnt;  // executed-step range [k0, k1) of the unit's cnt steps
};
struct Sched {
  bool streamk;
  int lo, hi, wbh, W;  // stream-K: this pair's range, steps per (b, h), total steps (host keeps W * P < 2^31)
  int P;               // pairs
  int u;               // round-robin: next unit
  int rr_end;          // hybrid: units [0, rr_end) are dealt whole, unit u to pair u % P
  int x0;              // ... and stream-K covers the executed steps [x0, W) of the remaining units
  const int32_t* plo;  // range boundaries [P + 1] (shared memory)
};
// stream-K range boundary of pair p
__device__ __forceinline__ int pair_lo(const Sched& sc, int p) { return sc.plo[p]; }
__device__ __forceinline__ int pair_of(const Sched& sc, int x) {
  int p = sc.W > sc.x0 ? (int)((int64_t)(x - sc.x0) * sc.P / (sc.W - sc.x0)) : 0;  // a guess; the walks fix it
  while (p + 1 < sc.P && pair_lo(sc, p + 1) <= x) ++p;
  while (p > 0 && pair_lo(sc, p) > x) --p;
  return p;
}
template <int TK, bool kTab>
__device__ __forceinline__ bool next_seg(Sched& sc, const int32_t* gpre, int n_groups, int n_units, int H,
                                      const SpanTable& st, int nq, int kv_len, int nkv, Seg& sg) {
  if (sc.streamk) {
    if (sc.u < sc.rr_end) {  // hybrid: whole units, dealt round-robin (all query groups of a head at once)
      const int u = sc.u;
      sc.u += sc.P;
      sg.g = u % n_groups;
      const int bh = u / n_groups;
      sg.h = bh % H;
      sg.b = bh / H;
      sg.k0 = 0;
      sg.k1 = sg.cnt = gpre[sg.g + 1] - gpre[sg.g];  // the group's executed steps
      return true;
    }
    if (sc.lo >= sc.hi) return false;
    const int bh = sc.lo / sc.wbh;
    const int r = sc.lo - bh * sc.wbh;
    int g = 0;
    while (gpre[g + 1] <= r) ++g;
    sg.g = g;
    sg.h = bh % H;
    sg.b = bh / H;
    sg.cnt = gpre[g + 1] - gpre[g];
    sg.k0 = r - gpre[g];
    sg.k1 = min(sg.cnt, sg.k0 + (sc.hi - sc.lo));
    sc.lo += sg.k1 - sg.k0;
    return true;
  }
  if (sc.u >= n_units) return false;
  const int u = sc.u;
  sc.u += sc.P;
  sg.g = u % n_groups;
  const int bh = u / n_groups;
  sg.h = bh % H;
  sg.b = bh / H;
  sg.k0 = 0;
  int cnt = nkv;  // whole unit: all of its executed steps
  if (st.n != 1) {
    cnt = 0;
    for (int j = 0; j < nkv; ++j) cnt += cls_get<TK, kTab>(st, sg.g, j, nq, kv_len, nkv) != kSkip;
  }
  sg.k1 = sg.cnt = cnt;
  return true;
}
// key step of the k-th executed step of group g (k counted from the group's first executed step)
template <int TK, bool kTab>
__device__ __forceinline__ int step_of(const SpanTable& st, int g, int k, int nq, int kv_len, int nkv) {
  if (st.n == 1) return k;
  int j = 0;
  for (;; ++j) {
    if (cls_get<TK, kTab>(st, g, j, nq, kv_len, nkv) == kSkip) continue;
    if (k-- == 0) return j;
  }
}


template <int D, bool PP, bool F8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_k2,
                    const __grid_constant__ CUtensorMap tm_v2, const __grid_constant__ CUtensorMap tm_o, int cur_step,
                    __nv_bfloat16* __restrict__ out, int64_t o_bstride,
                    int64_t o_tstride, float* __restrict__ lse, uint8_t* __restrict__ tile_map, int B, int H,
                    int nq, int kv_len, float m_static, int dbg, float* __restrict__ ws, int* __restrict__ ws_cnt,
                    const __grid_constant__ SpanTable st, const __grid_constant__ PeerMaps pm) {
  using C = Cfg<D, PP, F8>;
  constexpr int BN = C::kBN;  // keys per step (shadows the file-level 256)
  ptx::pdl_launch_dependents();  // the next kernel may take SMs as our CTAs finish (it waits for us)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw) + cls_tab_bytes(C::kTab, st.n, (((nq + BM - 1) / BM) + 1) / 2,
                                                               (kv_len + BN - 1) / BN);
  const uint32_t base = (raw + 1023u) & ~1023u;           // SW128 tiles need 1024-byte alignment
  uint8_t* smem = smem_raw + (base - ptx::smem_u32(smem_raw));
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
  float* red = reinterpret_cast<float*>(smem + C::kRedOff);
  const uint32_t sQ = base + C::kQOff;
  const uint32_t sKV = base + C::kKVOff;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int n_qtiles = (nq + BM - 1) / BM;
  const int n_groups = (n_qtiles + 1) / 2;                 // 2 query tiles per cluster unit
  const int n_units = B * H * n_groups;
  const int nkv = (kv_len + BN - 1) / BN;                  // key steps
  const int cid = (int)ptx::cluster_id_x(), ncl = (int)ptx::nclusters_x();
  const bool trace_on = kTrace && g_dz_trace_on != 0 && cid == 0;
  uint32_t* const trace = g_dz_trace + rank * kTraceSteps * 16;
  constexpr uint16_t kBoth = 0x3;

  auto bar = [&](uint64_t& b) { return ptx::smem_u32(&b); };
  auto lbar = [&](uint64_t& b) { return ptx::mapa(ptx::smem_u32(&b), 0); };  // leader's copy
  // ring slots of the i-th K load and the i-th V load (barrier index; the V ring follows the K ring)
  auto kslot = [&](uint32_t i, uint32_t& st, uint32_t& ph) {
    st = i % C::kKStages;
    ph = (i / C::kKStages) & 1;
  };
  auto vslot = [&](uint32_t i, uint32_t& st, uint32_t& ph) {
    st = C::kKStages + i % C::kVStages;
    ph = (i / C::kVStages) & 1;
  };

  // executed steps per query group -> prefix sums (every role walks the same schedule)
  const bool streamk = ws != nullptr && n_groups <= kMaxGroups;
  constexpr bool kTab = C::kTab;
  if (kTab && st.n != 1) {
    for (int i = threadIdx.x; i < (n_groups * nkv + 15) / 16; i += kThreads) s_cls_tab[i] = 0u;
    __syncthreads();
    for (int x = threadIdx.x; x < n_groups * nkv; x += kThreads) {
      const uint32_t c = step_class<BN>(st, x / nkv, x % nkv, nq, kv_len, true);
      if (c != 0u) atomicOr(&s_cls_tab[x >> 4], c << (2 * (x & 15)));
    }
    __syncthreads();
  }
  if (streamk) {
    if (st.n == 1) {
      for (int g = threadIdx.x; g <= n_groups; g += kThreads) bars->gpre[g] = g * nkv;
    } else {
      for (int g = threadIdx.x; g <= n_groups; g += kThreads) bars->gpre[g] = 0;
      __syncthreads();
      for (int x = threadIdx.x; x < n_groups * nkv; x += kThreads)
        if (cls_get<BN, kTab>(st, x / nkv, x % nkv, nq, kv_len, nkv) != kSkip)
          atomicAdd(&bars->gpre[x / nkv + 1], 1);
      __syncthreads();
      if (threadIdx.x == 0)
        for (int g = 1; g <= n_groups; ++g) bars->gpre[g] += bars->gpre[g - 1];
    }
  }
  if (warp == kWarpTma && lane == 0) {
    ptx::mbar_init(bar(bars->q_full), 1);
    ptx::mbar_init(bar(bars->q_empty), 1);
    for (int hh = 0; hh < 2; ++hh) {
      ptx::mbar_init(bar(bars->s_full[hh]), 1);
      ptx::mbar_init(bar(bars->s_free[hh]), 8);  // 4 softmax warps of that key half x 2 CTAs
    }
    for (int pb = 0; pb < 2; ++pb) {
      // PP: one P buffer per warp group (4 warps x 2 CTAs); !PP: one P buffer for all 8 warps
      ptx::mbar_init(bar(bars->p_full[pb]), PP ? 8 : 16);
      ptx::mbar_init(bar(bars->p_empty[pb]), 1);
    }
    ptx::mbar_init(bar(bars->o_full), 1);
    ptx::mbar_init(bar(bars->o_empty), 16);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(bar(bars->kv_full[s]), 1);
      ptx::mbar_init(bar(bars->kv_empty[s]), 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
    if (cur_step != 0x7fffffff) {
      ptx::tma_prefetch_desc(&tm_k2);
      ptx::tma_prefetch_desc(&tm_v2);
    }
  }
  if (warp == kWarpTmem) ptx::tmem_alloc_2cta<512>(ptx::smem_u32(&bars->tmem_base));
  if (blockIdx.x == 0 && threadIdx.x == 0) ptx::g_dz_watchdog[6] = ptx::smem_u32(bars);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any remote traffic
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int32_t* gpre = bars->gpre;
  // Hybrid schedule: all but the last ~1.x waves of units are dealt whole, round-robin (unit u
  // to pair u mod P), so the query groups of a head run side by side and its K/V is read from
  // HBM about once; stream-K splits the executed steps of the remaining units so that every
  // pair's total (its whole units + its range) matches W / P as closely as the unit lengths
  // allow.  (Pure stream-K spreads each head's groups over the whole launch, and the K/V of
  // every head must then stay in L2 from start to end.)
  int rr_end = 0, x0 = 0;
  if (streamk) {
    const int wbh = gpre[n_groups], W = B * H * wbh;
    if (n_units >= 2 * ncl) {
      rr_end = (n_units / ncl - 1) * ncl;
      x0 = (rr_end / n_groups) * wbh + gpre[rr_end % n_groups];  // executed steps of units [0, rr_end)
    }
    int32_t* plo = bars->plo;
    // linear index of the first executed step of unit u
    auto lin = [&](int u) { return (u / n_groups) * wbh + gpre[u % n_groups]; };
    for (int p = threadIdx.x; p < ncl; p += kThreads) {
      // whole-unit steps of pairs 0..p: units w*P .. w*P + p of every round-robin wave w
      int rr = 0;
      for (int w0 = 0; w0 < rr_end; w0 += ncl) rr += lin(w0 + p + 1) - lin(w0);
      // pairs 0..p end where their whole-unit steps plus their ranges reach W (p + 1) / P
      plo[p + 1] = p + 1 == ncl ? W : min(W, max(x0, x0 + W * (p + 1) / ncl - rr));  // (host: W * P < 2^31)
    }
    if (threadIdx.x == 0) plo[0] = x0;
    __syncthreads();
    if (threadIdx.x == 0)  // keep the boundaries non-decreasing (uneven unit lengths)
      for (int p = 1; p <= ncl; ++p) plo[p] = max(plo[p], plo[p - 1]);
    __syncthreads();
  }

  // (the schedule above depends on the launch parameters only: it is computed while the
  // predecessor finishes)
  ptx::pdl_wait();      // the prologue's Q' / K' / V (and everything before it) are complete
  if (threadIdx.x == 0) {
    bars->clk0 = clock64();
    bars->ns0 = gtime64();
  }
  Sched sched0;
  sched0.streamk = streamk;
  sched0.P = ncl;
  sched0.u = cid;
  sched0.rr_end = rr_end;
  sched0.x0 = x0;
  sched0.plo = bars->plo;
  if (streamk) {
    sched0.wbh = gpre[n_groups];
    sched0.W = B * H * sched0.wbh;
    sched0.lo = pair_lo(sched0, cid);
    sched0.hi = pair_lo(sched0, cid + 1);
  }

  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(regs_light<PP>()));
  if (warp == kWarpTma || warp == kWarpTmem) {
    // ------------------------------------------------ TMA producers (K + Q, V) --
    // warp kWarpTma loads each piece's Q tiles and the K tiles into the K ring; warp
    // kWarpTmem (idle between TMEM alloc and dealloc) loads the V tiles into the V ring.
    const bool do_k = warp == kWarpTma;
    const uint64_t pol_q = ptx::l2_policy_evict_first();
    const uint64_t pol_kv = ptx::l2_policy_evict_last();
    uint32_t ld = 0, q_phase = 0;
    Sched sc = sched0;
    Seg sg;
    bool first_seg = true;
    while (next_seg<BN, kTab>(sc, gpre, n_groups, n_units, H, st, nq, kv_len, nkv, sg)) {
      const int b = sg.b, h = sg.h, g = sg.g;
      if (do_k) {
        ptx::mbar_wait(bar(bars->q_empty), q_phase ^ 1);
        q_phase ^= 1;
        const int qt = 2 * g + (int)rank;
        if (lane == 0) {
          if (leader) ptx::mbar_arrive_expect_tx(bar(bars->q_full), min(2, n_qtiles - 2 * g) * C::kQTileBytes);
          if (qt < n_qtiles)  // a tile wholly past nq is not loaded (its rows are never stored)
            for (int x = 0; x < C::kQBoxes; ++x)
              ptx::tma_load_4d_2cta(sQ + x * BM * 128, &tm_q, lbar(bars->q_full), x * C::kBoxElems, h, qt * BM, b,
                                    pol_q);
        }
      }
      int j = step_of<BN, kTab>(st, g, sg.k0, nq, kv_len, nkv);
      for (int k = sg.k0; k < sg.k1; ++k, ++j, ++ld) {
        if (st.n != 1)
          while (cls_get<BN, kTab>(st, g, j, nq, kv_len, nkv) == kSkip) ++j;
        uint32_t sl, ph;
        if (do_k)
          kslot(ld, sl, ph);
        else
          vslot(ld, sl, ph);
        ptx::mbar_wait(bar(bars->kv_empty[sl]), ph ^ 1);
        if (trace_on && first_seg && j < kTraceSteps && lane == 0) trace[2560 + 2 * j + (do_k ? 0 : 1)] = (uint32_t)clock();
        if (lane == 0 && (dbg & 1)) {  // diagnostics: no K/V traffic, MMAs read stale smem
          if (leader) ptx::mbar_arrive(bar(bars->kv_full[sl]));
        } else if (lane == 0) {
          if (leader) ptx::mbar_arrive_expect_tx(bar(bars->kv_full[sl]), do_k ? 2 * C::kKBytes : 2 * C::kStageBytes);
          const uint32_t dst = sKV + sl * C::kStageBytes;
          if (do_k) {
            // S half hh (keys 128hh..128hh+127 of the step) takes 64 keys from each CTA:
            // this CTA loads keys 128hh + 64*rank .. +63 into [hh][dim box] of 64 x 128 B
            // the new tokens' K' (j >= cur_step) come from the current-chunk buffer
            const bool cur = j >= cur_step;
            const CUtensorMap* tk = cur ? &tm_k2 : &tm_k;
            const int row0 = (cur ? j - cur_step : j) * BN + 64 * (int)rank;
            for (int hh = 0; hh < BN / 128; ++hh)
              for (int x = 0; x < C::kQBoxes; ++x)
                ptx::tma_load_4d_2cta(dst + (hh * C::kQBoxes + x) * 64 * 128, tk, lbar(bars->kv_full[sl]),
                                      x * C::kBoxElems, h, row0 + 128 * hh, b, pol_kv);
          } else {
            if (j >= cur_step)  // the new tokens' V, read in place from the caller's input (no staging copy)
              ptx::tma_load_4d_2cta(dst, &tm_v2, lbar(bars->kv_full[sl]), (int)rank * (D / 2), h, (j - cur_step) * BN,
                                    b, pol_kv);
            else
              ptx::tma_load_4d_2cta(dst, &tm_v, lbar(bars->kv_full[sl]), (int)rank * (D / 2), h, j * BN, b, pol_kv);
          }
        }
        __syncwarp();
      }
      first_seg = false;
    }
  } else if ((warp == kWarpMma || warp == kWarpPv) && leader) {
    // ------------------------------------------------------ MMA issuers --
    // Two single-thread issuers walk the same schedule: warp 11 issues QK(j),
    // warp 9 issues PV(j) once the softmax has written P(j).  tcgen05.mma
    // issue blocks at the tensor pipe's rate (the queue is shallow), so an
    // issuer that waits on a barrier starves the pipe; with two issuers, one
    // keeps it fed while the other waits.  QK and PV touch disjoint TMEM (S vs
    // P/O) and release their own K / V stages, so their streams need no mutual
    // order.
    const bool do_qk = warp == kWarpMma;
    uint32_t q_phase = 0, sf_phase = 0, pf_phase = 0, oe_phase = 0;
    int gs = 0;  // this issuer's running count of executed steps
    Sched sc = sched0;
    Seg sg;
    bool first_seg = true;
    while (next_seg<BN, kTab>(sc, gpre, n_groups, n_units, H, st, nq, kv_len, nkv, sg)) {
      const int g = sg.g;
      int j = step_of<BN, kTab>(st, g, sg.k0, nq, kv_len, nkv);
      for (int k = sg.k0; k < sg.k1; ++k, ++j) {
        if (st.n != 1)
          while (cls_get<BN, kTab>(st, g, j, nq, kv_len, nkv) == kSkip) ++j;
        const bool first = k == sg.k0, last = k == sg.k1 - 1;
        const bool tr = trace_on && first_seg && j < kTraceSteps && lane == 0;
        if (do_qk) {
          if (first) {  // first step of a piece: its Q tiles
            ptx::mbar_wait(bar(bars->q_full), q_phase);
            q_phase ^= 1;
          }
          uint32_t k_st, k_ph;
          kslot(gs, k_st, k_ph);
          ptx::mbar_wait(bar(bars->kv_full[k_st]), k_ph);
          // !PP: S in two halves of 128 keys (N = 128 each): the half-hh softmax warps release
          // their half as soon as they hold it, so each QK half waits only for the copy of the
          // same half of the previous step.  PP: one 128-key S per step, written into buffer
          // gs % 2, which the softmax of step gs - 2 has released.
          constexpr int kHalves = BN / 128;
          for (int hh = 0; hh < kHalves; ++hh) {
            const int sb = PP ? (gs & 1) : hh;  // S buffer written
            if (tr && hh == 0) trace[j * 8 + 0] = (uint32_t)clock();
            if constexpr (PP) {
              ptx::mbar_wait(bar(bars->s_free[sb]), ((gs >> 1) & 1) ^ 1);
            } else if (gs > 0) {
              ptx::mbar_wait(bar(bars->s_free[hh]), sf_phase);
              if (hh == 1) sf_phase ^= 1;
            }
            if (tr && hh == 0) trace[j * 8 + 1] = (uint32_t)clock();
            ptx::tc_fence_after();
            if (lane == 0) {
              const uint32_t ka = sKV + k_st * C::kStageBytes + hh * C::kQBoxes * 64 * 128;
              const uint64_t dq0 = ptx::sdesc_sw128(sQ, 16, 1024), dk0 = ptx::sdesc_sw128(ka, 16, 1024);
#pragma unroll
              for (int kk = 0; kk < C::kQKSteps; ++kk) {
                const uint32_t qoff = (kk / 4) * (128 * 128) + (kk % 4) * 32;  // Q: 128 rows per box
                const uint32_t koff = (kk / 4) * (64 * 128) + (kk % 4) * 32;   // K half: 64 rows per box
                // descriptors: the start address field is addr >> 4 in the low bits, offsets add
                if constexpr (F8)  // (the idesc's E4M3 format codes are the f16 kind's F16 codes: 0)
                  ptx::mma_ss_2cta_f8(tmem + kColS + sb * 128, dq0 + (qoff >> 4), dk0 + (koff >> 4), C::kIdescQK,
                                      kk > 0);
                else
                  ptx::mma_ss_2cta(tmem + kColS + sb * 128, dq0 + (qoff >> 4), dk0 + (koff >> 4), C::kIdescQK, kk > 0);
                if (tr && j == 9) trace[kTraceSteps * 8 + hh * 8 + kk] = (uint32_t)clock();
              }
              ptx::tc_commit_2cta(bar(bars->s_full[sb]), kBoth);
              if (hh == kHalves - 1) {
                ptx::tc_commit_2cta(bar(bars->kv_empty[k_st]), kBoth);
                if (last) ptx::tc_commit_2cta(bar(bars->q_empty), kBoth);
              }
            }
            __syncwarp();
          }
        } else {
          uint32_t v_st, v_ph;
          vslot(gs, v_st, v_ph);
          ptx::mbar_wait(bar(bars->kv_full[v_st]), v_ph);
          if (tr) trace[j * 8 + 2] = (uint32_t)clock();
          const int pb = PP ? (gs & 1) : 0;  // P buffer read
          if constexpr (PP) {
            ptx::mbar_wait(bar(bars->p_full[pb]), (gs >> 1) & 1);
          } else {
            ptx::mbar_wait(bar(bars->p_full[0]), pf_phase);
            pf_phase ^= 1;
          }
          if (first) {  // the previous piece's epilogue has read O
            ptx::mbar_wait(bar(bars->o_empty), oe_phase ^ 1);
            oe_phase ^= 1;
          }
          if (tr) trace[j * 8 + 3] = (uint32_t)clock();
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t va = sKV + v_st * C::kStageBytes;
            const uint64_t dv0 = D == 128 ? ptx::sdesc_sw128(va, 16, 1024) : ptx::sdesc_sw64(va, 16, 512);
#pragma unroll
            for (int kk = 0; kk < BN / 16; ++kk) {
              ptx::mma_ts_2cta(tmem + kColO, tmem + kColP + pb * 64 + kk * 8, dv0 + ((kk * 16 * C::kVRowBytes) >> 4),
                               C::kIdescPV, (!first || kk > 0) ? 1u : 0u);
              if (tr && j == 9) trace[kTraceSteps * 8 + 16 + kk] = (uint32_t)clock();
            }
            ptx::tc_commit_2cta(bar(bars->p_empty[pb]), kBoth);              // P may be overwritten
            if (last) ptx::tc_commit_2cta(bar(bars->o_full), kBoth);
            ptx::tc_commit_2cta(bar(bars->kv_empty[v_st]), kBoth);
          }
          __syncwarp();
        }
        ++gs;
      }
      first_seg = false;
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(regs_softmax<PP>()));
    // ---------------------------------------------- softmax + epilogue --
    const int quad = warp % 4;                  // TMEM lane quadrant (query rows)
    const int hc = warp / 4;                    // key half of S / column half of O
    const int row = quad * 32 + lane;
    const uint32_t lane_bits = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_bits + kColS + hc * 128;
    const uint32_t tP = tmem + lane_bits + kColP + hc * 64;
    const uint32_t tO = tmem + lane_bits + kColO + hc * (D / 2);
    const uint32_t pair_bar = 1 + quad;         // named barrier: the two warps of these rows
    constexpr uint32_t kSoftmaxBar = 5;         // named barrier: all 8 softmax warps
    const bool online = m_static <= 0.f;
    // Epilogue store of this thread's row (D/2 bf16 = D/4 packed pairs, this warp's column half):
    // through the warp's swizzled shared-memory staging tile and one TMA tensor store per warp
    // (32 rows x D bytes), so the output leaves in whole 128-byte lines; rows past nq are clipped.
    const uint32_t sOw = base + C::kOOff + warp * 32 * D;
    auto store_o = [&](const uint32_t* pk, int b_, int h_, int qt_) {
      constexpr int NC = D / 16;  // 16-byte chunks per staged row (D/2 bf16)
      if (lane == 0) ptx::bulk_wait_read_all();  // the previous store has read the staging tile
      __syncwarp();
#pragma unroll
      for (int c = 0; c < NC; ++c)
        ptx::st_shared_v4(sOw + lane * D + ((c ^ ((lane * D >> 7) & (NC - 1))) * 16), pk[4 * c], pk[4 * c + 1],
                          pk[4 * c + 2], pk[4 * c + 3]);
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int r0 = qt_ * BM + quad * 32;
        if (pm.n == 0) {
          ptx::tma_store_4d(&tm_o, sOw, hc * (D / 2), h_, r0, b_);
        } else {
          // peer stores: the 32 rows go to their owners' receive buffers as 4 boxes of 8 rows (owner
          // boundaries n_loc are multiples of 8, so a box never straddles two owners; an 8-row slice
          // of the SW128 staging tile is one 1024-byte swizzle atom)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = r0 + 8 * i;
            if (rr < nq) {
              const int p = rr / pm.n_loc;
              ptx::tma_store_4d(&pm.m[p], sOw + i * 8 * D, hc * (D / 2), h_, rr - p * pm.n_loc, b_);
            }
          }
        }
        ptx::bulk_commit_group();
      }
    };
    uint32_t s_phase = 0, pe_phase = 0, of_phase = 0;
    int gsm = 0;  // executed steps so far (PP: this warp group takes the steps with gsm % 2 == hc)
    Sched sc = sched0;
    Seg sg;
    bool first_seg = true;
    const bool tl = kTrace && g_dz_trace_on != 0 && threadIdx.x == 0 && blockIdx.x < kTimelineCtas;
    uint32_t* const tline = g_dz_timeline + blockIdx.x * kTimelineWords;
    int n_seg = 0, n_comb = 0, n_part = 0;
    if (tl) {
      tline[0] = gtime();
      tline[2] = (uint32_t)clock();
    }
    while (next_seg<BN, kTab>(sc, gpre, n_groups, n_units, H, st, nq, kv_len, nkv, sg)) {
      const int b = sg.b, h = sg.h, g = sg.g;
      const int qt = 2 * g + (int)rank;
      if (tl && n_seg < kTlSegs) tline[8 + 4 * n_seg] = (uint32_t)clock();
      float m_used = online ? -INFINITY : 0.f;   // softmax base, log2 units (fixed base: 0)
      float l = 0.f;                              // partial row sum over this warp's keys
      const int s_row = qt * BM + row;            // this thread's query (row of the new tokens)
      const int qs = st.n == 1 ? 0 : span_at(st, min(s_row, nq - 1));  // its span (rows past nq: never stored)
      const bool map_thread = tile_map != nullptr && b == 0 && h == 0 && rank == 0 && row == 0 && hc == 0;
      int j = step_of<BN, kTab>(st, g, sg.k0, nq, kv_len, nkv);
      // fast walk (PP, one span, no tile map): every step executes, so this group's steps
      // are every other one -- no per-step bookkeeping for the other group's steps
      const int gsm0 = gsm;
      const bool fast = PP && st.n == 1 && tile_map == nullptr;
      const int kstep = fast ? 2 : 1;
      const int k_start = sg.k0 + (fast ? ((hc - gsm0) & 1) : 0);
      j += k_start - sg.k0;
      for (int k = k_start; k < sg.k1; k += kstep, j += kstep) {
        const bool first = k == sg.k0;
        int my_u;                                     // PP: use count of this group's S / P buffer
        if (fast) {
          my_u = (gsm0 + (k - sg.k0)) >> 1;
        } else {
          if (st.n != 1)
            while (cls_get<BN, kTab>(st, g, j, nq, kv_len, nkv) == kSkip) ++j;
          // executed steps only; the host zeroes (SKIP) the map
          if (map_thread) tile_map[g * nkv + j] = step_class<BN>(st, g, j, nq, kv_len);
          my_u = gsm >> 1;
          if (PP && (gsm++ & 1) != hc) continue;      // the other warp group's step
        }
        // mask needed iff an in-bounds row of the tile misses a key of the step (Fig. 10 or key
        // bounds); one span (attend_chunk): only a ragged last key step
        const bool masked = st.n == 1 ? (j == nkv - 1 && kv_len % BN != 0)
                                      : cls_get<BN, kTab>(st, g, j, nq, kv_len, nkv) == kPartial;
        if constexpr (PP) {
          ptx::mbar_wait(bar(bars->s_full[hc]), my_u & 1);
        } else {
          ptx::mbar_wait(bar(bars->s_full[hc]), s_phase);
          s_phase ^= 1;
        }
        const bool tr = trace_on && first_seg && j < kTraceSteps && row == 0 && hc == 0;
        if (tr) trace[j * 8 + 4] = (uint32_t)clock();
        SCHED_POINT();
        ptx::tc_fence_after();
        float s[128];
        {
          uint32_t r[128];
#pragma unroll
          for (int c = 0; c < 4; ++c) ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[c * 32]));
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 128; ++i) s[i] = __uint_as_float(r[i]);
        }
        // S is in registers: the next QK may overwrite it now
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->s_free[hc]));
        if (tr) trace[j * 8 + 6] = (uint32_t)clock();
        SCHED_POINT();
        if (masked) {  // Fig. 10 mask and key bounds for this warp's 128 keys
          uint32_t vm[4];
          visible_bits(st, qs, j * BN + (PP ? 0 : 128 * hc), kv_len, vm);
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (!((vm[i / 32] >> (i % 32)) & 1u)) s[i] = -INFINITY;
        }
        if (!PP && online) {  // (the host selects !PP whenever the softmax base is online)
          // Online softmax with lazy rescaling: a row moves its base only when its max
          // grew by more than 2^8; both warps of a row take the same decision from the
          // exchanged maxima.  O may be rescaled only when no PV into it is in flight:
          // wait for PV(j-1) (p_empty) first.  tcgen05.ld/st are warp-collective, so
          // the decision is warp-uniform.
          // row max as 8 independent chains (the single 128-long chain was 64 dependent
          // FMNMX3 on the critical path of every step); max is exact in any order
          float m8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = s[k];
#pragma unroll
          for (int i = 8; i < 128; i += 8)
#pragma unroll
            for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], s[i + k]);
          float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          red[hc * BM + row] = mx;
          ptx::named_bar_sync(pair_bar, 64);
          mx = fmaxf(mx, red[(hc ^ 1) * BM + row]);
          ptx::named_bar_sync(pair_bar, 64);  // both read before the next exchange
          const bool grow = mx > m_used + kRescaleLog2;
          const bool rescale = grow && !first && m_used != -INFINITY;
          if (__any_sync(0xffffffffu, rescale)) {
            ptx::mbar_wait(bar(bars->p_empty[0]), pe_phase ^ 1);  // PV(j-1) done
            ptx::tc_fence_after();
            const float alpha = rescale ? ptx::ex2(m_used - mx) : 1.f;
            l *= alpha;
#pragma unroll
            for (int c = 0; c < D / 64; ++c) {
              uint32_t r[32];
              ptx::tmem_ld32(tO + c * 32, r);
              ptx::tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              ptx::tmem_st32(tO + c * 32, r);
            }
            ptx::tmem_wait_st();
          }
          if (grow) m_used = mx;
        }
        // Scores are in log2 units (Q' was pre-scaled by scale*log2e).  Fixed base (QK-norm
        // bound, m_static <= 60): p = 2^s directly, every p in [2^-60, 2^60], so neither an
        // offset nor a clamp is needed; online base: p = 2^(s - m).
        const float nbase = (!online || m_used == -INFINITY) ? 0.f : -m_used;
        const uint64_t nb2 = ptx::f2_pack(nbase, nbase);
        const bool plain = !online && !masked;
        __syncwarp();
        uint64_t acc[4] = {0, 0, 0, 0};
        // two halves of 64 keys: exponentials of half h, then its P store (the first store
        // waits until PV(j-1) has read P), so only 32 packed registers are live at a time
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t pk[32];
#ifdef DZ_DIAG_NOEXP  // diagnostics build only: P = packed scores, no exponentials (results are garbage)
          if (true) {
#pragma unroll
            for (int i = 0; i < 32; ++i) pk[i] = ptx::pack_bf16x2(s[64 * half + 2 * i], s[64 * half + 2 * i + 1]);
          } else
#endif
          if (plain)
            exp_half<true>(s + 64 * half, nb2, pk, acc);
          else
            exp_half<false>(s + 64 * half, nb2, pk, acc);
          if (half == 0) {
            if (tr) trace[j * 8 + 7] = (uint32_t)clock();
        SCHED_POINT();
            // P may be overwritten once the PV that last read it is done (PP: PV(j-2), own buffer)
            if constexpr (PP) {
              ptx::mbar_wait(bar(bars->p_empty[hc]), (my_u & 1) ^ 1);
            } else {
              ptx::mbar_wait(bar(bars->p_empty[0]), pe_phase ^ 1);
              pe_phase ^= 1;
            }
            ptx::tc_fence_after();
          }
          ptx::tmem_st32(tP + 32 * half, pk);
        }
        {
          const uint64_t a = ptx::f2_add(ptx::f2_add(acc[0], acc[1]), ptx::f2_add(acc[2], acc[3]));
          float a0, a1;
          ptx::f2_unpack(a, a0, a1);
          l += a0 + a1;
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->p_full[PP ? hc : 0]));
        if (tr) trace[j * 8 + 5] = (uint32_t)clock();
        SCHED_POINT();
      }
      if (fast) gsm = gsm0 + (sg.k1 - sg.k0);
      first_seg = false;
      if (tl && n_seg < kTlSegs) tline[9 + 4 * n_seg] = (uint32_t)clock();
      // total row sum over both key halves
      red[hc * BM + row] = l;
      ptx::named_bar_sync(pair_bar, 64);
      const float lt = l + red[(hc ^ 1) * BM + row];
      ptx::named_bar_sync(pair_bar, 64);  // the buffer is reused by the next exchange
      ptx::mbar_wait(bar(bars->o_full), of_phase);
      of_phase ^= 1;
      ptx::tc_fence_after();
      if (tl && n_seg < kTlSegs) tline[10 + 4 * n_seg] = (uint32_t)clock();
      const int s_idx = qt * BM + row;
      if (sg.k0 == 0 && sg.k1 == sg.cnt) {
        // whole unit: O / l -> bf16 -> HBM (this warp's D/2 columns).  O leaves TMEM first and is
        // released at once, so the next unit's first PV does not wait for the global stores.
        const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
        uint32_t r[D / 2];
#pragma unroll
        for (int c = 0; c < D / 64; ++c) ptx::tmem_ld32(tO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&r[c * 32]));
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->o_empty));
        {
          uint32_t pk[D / 4];
#pragma unroll
          for (int i = 0; i < D / 4; ++i)
            pk[i] = ptx::pack_bf16x2(__uint_as_float(r[2 * i]) * inv_l, __uint_as_float(r[2 * i + 1]) * inv_l);
          store_o(pk, b, h, qt);
        }
        if (lse != nullptr && hc == 0 && s_idx < nq)
          lse[((int64_t)b * H + h) * nq + s_idx] =
              (lt > 0.f) ? (m_used + __log2f(lt)) * 0.69314718055994530942f : -INFINITY;
        if (tl && n_seg < kTlSegs) tline[11 + 4 * n_seg] = (uint32_t)clock();
        ++n_seg;
        continue;
      }
      // ---- a piece of a unit split across pairs (stream-K): publish (O, l, base) ----
      // workspace slot: the pair's head piece (starts mid-unit) or tail piece (ends mid-unit);
      // layout per (slot, rank): O [D][128] fp32 column-major (coalesced per column), l [128], m [128]
      constexpr int kSlotFloats = (D + 2) * BM;
      float* mine = ws + ((size_t)(2 * cid + (sg.k0 > 0 ? 0 : 1)) * 2 + rank) * kSlotFloats;
      const int ustart = (b * H + h) * sched0.wbh + gpre[g];
      const int pf = pair_of(sched0, ustart), pl = pair_of(sched0, ustart + sg.cnt - 1);
      // pieces = pairs in [pf, pl] with a non-empty range (a pair's range may be empty when W < P)
      int n_pieces = 0;
      for (int q = pf; q <= pl; ++q) n_pieces += pair_lo(sched0, q) < pair_lo(sched0, q + 1);
      int* cnt_ptr = ws_cnt + (((int64_t)b * H + h) * n_groups + g) * 2 + rank;
      // Every other piece already published (the usual case for the piece finishing last, e.g. a
      // unit's head piece at the end of a pair's range): combine straight from TMEM, no publish.
      if (threadIdx.x == 0) bars->last_piece = ptx::ld_acquire_gpu(cnt_ptr) == n_pieces - 1 ? 2 : 0;
      ptx::named_bar_sync(kSoftmaxBar, 256);
      const bool direct = bars->last_piece == 2;  // (O leaves TMEM inside the combine loop below)
#pragma unroll 1
      for (int c = 0; c < D / 64 && !direct; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(tO + c * 32, r);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) __stcg(mine + (hc * (D / 2) + c * 32 + i) * BM + row, __uint_as_float(r[i]));
      }
      if (!direct) {
        if (hc == 0) {
          __stcg(mine + D * BM + row, lt);
          __stcg(mine + (D + 1) * BM + row, m_used);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->o_empty));  // TMEM O has been read
        if (tl && n_part < 2) tline[50 + 5 * n_part] = (uint32_t)clock();
        // publish: every thread's stores precede the barrier; one thread fences (cumulative) and counts
        ptx::named_bar_sync(kSoftmaxBar, 256);
        if (threadIdx.x == 0) {
          // acq_rel RMW at GPU scope: releases this CTA's piece (the barrier above made every
          // softmax thread's stores precede it; release is cumulative) and, for the last
          // piece, acquires the others' before the barrier below releases the readers
          const bool last_piece = ptx::atom_add_acq_rel_gpu(cnt_ptr, 1) == n_pieces - 1;
          bars->last_piece = last_piece;
        }
        ptx::named_bar_sync(kSoftmaxBar, 256);
      }
      if (tl && n_part < 2) tline[51 + 5 * n_part] = (uint32_t)clock();
      if (!bars->last_piece) {
        if (tl && n_seg < kTlSegs) tline[11 + 4 * n_seg] = (uint32_t)clock();
        ++n_seg;
        ++n_part;
        continue;
      }
      // last piece to finish: combine all pieces of this unit in key order.  Each piece's
      // D/2 columns of this row are loaded in one batch (64 loads in flight per thread), so
      // a combine costs about one L2 round trip per piece.
      // own piece (direct path): O from TMEM; base and total row sum are this thread's (both warps
      // of a row hold the same m_used and lt)
      const float m_own = m_used, l_own = lt;
      float mmax = -INFINITY;
#pragma unroll 1
      for (int q = pf; q <= pl; ++q) {
        if (pair_lo(sched0, q) == pair_lo(sched0, q + 1)) continue;
        const float* pc = ws + ((size_t)(2 * q + (q == pf ? 1 : 0)) * 2 + rank) * kSlotFloats;
        mmax = fmaxf(mmax, (direct && q == cid) ? m_own : __ldcg(pc + (D + 1) * BM + row));
      }
      float wsum = 0.f;
      float acc[D / 2];
#pragma unroll
      for (int i = 0; i < D / 2; ++i) acc[i] = 0.f;
#pragma unroll 1
      for (int q = pf; q <= pl; ++q) {
        if (pair_lo(sched0, q) == pair_lo(sched0, q + 1)) continue;
        const float* pc = ws + ((size_t)(2 * q + (q == pf ? 1 : 0)) * 2 + rank) * kSlotFloats;
        float v[D / 2];
        float mq, lq;
        if (direct && q == cid) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) ptx::tmem_ld32(tO + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[c * 32]));
          ptx::tmem_wait_ld();
          mq = m_own;
          lq = l_own;
        } else {
#pragma unroll
          for (int i = 0; i < D / 2; ++i) v[i] = __ldcg(pc + (hc * (D / 2) + i) * BM + row);
          mq = __ldcg(pc + (D + 1) * BM + row);
          lq = __ldcg(pc + D * BM + row);
        }
        const float wq = mq == -INFINITY ? 0.f : ptx::ex2(mq - mmax);  // fixed base: every mq = 0, wq = 1
        wsum += wq * lq;
#pragma unroll
        for (int i = 0; i < D / 2; ++i) acc[i] = fmaf(wq, v[i], acc[i]);
      }
      if (direct) {  // TMEM O has been read
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(lbar(bars->o_empty));
      }
      const float inv_l = wsum > 0.f ? 1.f / wsum : 0.f;
      if (tl && n_part < 2) tline[52 + 5 * n_part] = (uint32_t)clock();
      {
        uint32_t pk[D / 4];
#pragma unroll
        for (int i = 0; i < D / 4; ++i) pk[i] = ptx::pack_bf16x2(acc[2 * i] * inv_l, acc[2 * i + 1] * inv_l);
        store_o(pk, b, h, qt);
      }
      if (lse != nullptr && hc == 0 && s_idx < nq)
        lse[((int64_t)b * H + h) * nq + s_idx] =
            (wsum > 0.f) ? (mmax + __log2f(wsum)) * 0.69314718055994530942f : -INFINITY;
      if (threadIdx.x == 0) *cnt_ptr = 0;  // ready for the next launch
      if (tl && n_seg < kTlSegs) tline[11 + 4 * n_seg] = (uint32_t)clock();
      if (tl && n_part < 2) tline[53 + 5 * n_part] = (uint32_t)clock();
      ++n_seg;
      ++n_comb;
      ++n_part;
    }
    if (lane == 0) ptx::bulk_wait_all();  // the last epilogue stores have completed
    if (tl) {
      tline[1] = gtime();
      tline[3] = (uint32_t)clock();
      tline[4] = n_seg;
      tline[5] = n_comb;
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();  // no remote arrives / multicast commits may target an exited CTA
  ptx::tc_fence_after();
  if (warp == kWarpTmem) ptx::tmem_dealloc_2cta<512>(tmem);
  if (threadIdx.x == 0) {
    atomicAdd(&g_dz_k2clk[0], (unsigned long long)(clock64() - bars->clk0));
    atomicAdd(&g_dz_k2clk[1], (unsigned long long)(gtime64() - bars->ns0));
  }
}

template <int D, bool PP, bool F8 = false>
cudaError_t launch_t(const AttnArgs& a, cudaStream_t s) {
  using C = Cfg<D, PP, F8>;
  auto k = attn_fwd_kernel<D, PP, F8>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::kSmem + (C::kTab ? kClsWords * 4 : 0));
  if (e != cudaSuccess) return e;
  const int n_groups = ((a.nq + BM - 1) / BM + 1) / 2, nkv = (a.kv_len + C::kBN - 1) / C::kBN;
  const int smem = C::kSmem + cls_tab_bytes(C::kTab, a.spans.n, n_groups, nkv);
  return launch_pdl(k, dim3(a.grid), dim3(kThreads), (size_t)smem, s, a.tm_q, a.tm_k, a.tm_v, a.tm_k2, a.tm_v2, a.tm_o,
                    a.cur_step,
                    static_cast<__nv_bfloat16*>(a.out), a.o_bstride, a.o_tstride, a.lse, a.tile_map, a.B, a.H, a.nq,
                    a.kv_len, a.m_static, a.debug_flags, a.ws, a.ws_cnt, a.spans, a.pm);
}

}  // namespace

cudaError_t k2_clock(uint64_t* host2, int reset) {
  cudaError_t e = host2 ? cudaMemcpyFromSymbol(host2, g_dz_k2clk, sizeof(uint64_t) * 2) : cudaSuccess;
  if (e != cudaSuccess || !reset) return e;
  const unsigned long long z[2] = {0, 0};
  return cudaMemcpyToSymbol(g_dz_k2clk, z, sizeof(z));
}
cudaError_t read_watchdog(uint32_t* host8) {
  return cudaMemcpyFromSymbol(host8, ptx::g_dz_watchdog, sizeof(uint32_t) * 8);
}
cudaError_t trace_control(int enable, uint32_t* host, size_t n) {
  cudaError_t e = cudaMemcpyToSymbol(g_dz_trace_on, &enable, sizeof(int));
  if (e != cudaSuccess || host == nullptr) return e;
  const size_t bytes = std::min(n, (size_t)kTraceSteps * 32) * sizeof(uint32_t);
  e = cudaMemcpyFromSymbol(host, g_dz_trace, bytes);
  if (e != cudaSuccess || n <= (size_t)kTraceSteps * 32) return e;
  // words past the step trace: the per-CTA timeline
  const size_t tl = std::min(n - kTraceSteps * 32, (size_t)kTimelineCtas * kTimelineWords) * sizeof(uint32_t);
  return cudaMemcpyFromSymbol(host + kTraceSteps * 32, g_dz_timeline, tl);
}
cudaError_t reset_watchdog() {
  static const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return cudaMemcpyToSymbol(ptx::g_dz_watchdog, zero, sizeof zero);
}

int attention_units(int32_t B, int32_t H, int32_t nq) {
  const int n_qtiles = (nq + BM - 1) / BM;
  return B * H * ((n_qtiles + 1) / 2);  // cluster units (pairs of CTAs, one query tile each)
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s) {
  const bool pp = attention_step_keys(a.m_static) == 128;
  if (a.fp8) return (a.D == 128 && pp) ? launch_t<128, true, true>(a, s) : cudaErrorInvalidValue;
  if (a.D == 128) return pp ? launch_t<128, true>(a, s) : launch_t<128, false>(a, s);
  if (a.D == 64) return pp ? launch_t<64, true>(a, s) : launch_t<64, false>(a, s);
  return cudaErrorInvalidValue;
}

int attention_step_keys(float m_static) { return m_static > 0.f ? 128 : 256; }

bool attention_has_step_table(int32_t D, float m_static) {
  return D == 128 ? Cfg<128, true>::kTab && m_static > 0.f : true;  // Cfg<D, PP>::kTab
}

}  // namespace dz
