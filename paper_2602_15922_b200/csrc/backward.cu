// backward.cu -- NEXT-1 backward: gradients of the teacher-forced path (Fig. 10(a) spans, empty cache)
//   L = sum(dO * O),  O = softmax_masked(q' k'^T * scale) V,  x' = RoPE(RMSNorm(x) * g)
// ("trajectory-level updates", Alg. 1 l.512-553).
//
// Three kernels, run after the forward prologue (K1) has recomputed Q' (pre-scaled by
// scale * log2e, fp16) and K' (fp16):
//   B1 delta_kernel     delta_s = <dO_s, O_s> and lse2_s = lse_s * log2(e), per (b, h, query)
//   B2 attn_bwd_kernel  one CTA per (b, h, 128-key tile), looping over the query tiles that see any of
//                       its keys (SKIP tiles never loaded); five tcgen05 MMAs per query tile, all
//                       operands in shared memory (SW128, 64-column TMA boxes), accumulators in TMEM:
//                         S^T = K' Q'^T          (M = keys, N = queries, K = D)      cols [0,128)
//                         dP^T = V dO^T          (M = keys, N = queries, K = D)      cols [128,256)
//                         -- 4 warps (thread = key row): P^T = 2^(S^T - lse2), masked (Fig. 10);
//                            dS^T = P^T (dP^T - delta), written bf16 / fp16 to shared memory --
//                         dV += P^T dO           (B = dO read MN-major)              cols [256,384)
//                         dK += dS^T Q'          (B = Q' read MN-major)              cols [384,512)
//                         dQ^T = K'^T dS^T       (A = K', B = dS^T read MN-major)    cols [0,128)
//                       dQ^T leaves TMEM (thread = d row) as fp32 atomics into dQ' (coalesced over d);
//                       dV (bf16) and dK' (fp32) are written once per key tile.
//   B3 prologue_bwd_kernel  dx = RMSNorm/RoPE backward of dx' for q and k, and the gain gradients.
// First version: correct by construction, not pipelined (each stage waits for the previous one).
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
constexpr int kBwdThreads = 320;     // warps 0..7 compute (quadrant w % 4, query half w / 4), 8 TMA producer, 9 MMA issuer
constexpr int kWarpProd = 8, kWarpMma = 9;
constexpr int kKTile = 128 * 128 * 2;      // [128 keys][128 d] 16-bit as two [128][64] SW128 boxes
constexpr int kKBox = 128 * 128;
constexpr int kQTile = 64 * 128 * 2;       // [64 q][128 d] as two [64][64] boxes
constexpr int kQBox = 64 * 128;
constexpr int kPTile = 128 * 64 * 2;       // [128 keys][64 q]: one box

// shared-memory map: K', V (whole launch), Q'[2], dO[2] (per step, double-buffered), P^T, dS^T,
// lse2 / delta of the step's queries [2][2][64]
constexpr int kOffK = 0, kOffV = kKTile, kOffQ = 2 * kKTile, kOffDO = kOffQ + 2 * kQTile, kOffPT = kOffDO + 2 * kQTile,
              kOffDST = kOffPT + kPTile, kOffVec = kOffDST + kPTile, kOffDQ = kOffVec + 1024,
              kDQTile = kQStep * 128 * 4,                    // dQ staging [64 q][128 d] fp32, double-buffered
              kOffBar = kOffDQ + 2 * kDQTile, kBwdSmem = kOffBar + 1024 + 1024;
static_assert(kBwdSmem <= 232448, "backward shared memory");

struct BwdBars {
  uint64_t kv_full, q_full[2], q_empty[2], s_full, s_read, dq_free[2], p_ready, mma_done;
  uint32_t tmem_base;
};

__device__ __forceinline__ bool span_vis(const SpanTable& st, int qs, int ks) {
  return qs == ks || st.kc[ks] < st.qth[qs];
}
__device__ __forceinline__ int span_of(const SpanTable& st, int x) {
  int i = 0;
  while (i + 1 < st.n && st.start[i + 1] <= x) ++i;
  return i;
}
// any visible (query, key) pair between queries [q0, q0 + kQStep) and keys [k0, k0 + 128) (both < n)
__device__ __forceinline__ bool step_visible(const SpanTable& st, int q0, int k0, int n) {
  const int q1 = min(q0 + kQStep, n), k1 = min(k0 + kBwdTile, n);
  for (int ks = span_of(st, k0); ks < st.n && st.start[ks] < k1; ++ks)
    for (int qs = span_of(st, q0); qs < st.n && st.start[qs] < q1; ++qs)
      if (span_vis(st, qs, ks)) return true;
  return false;
}
// visible queries of key span ks among [q0, q0 + 64): 64-bit mask (two words)
__device__ __forceinline__ void visible_queries(const SpanTable& st, int ks, int q0, int n, uint32_t (&m)[2]) {
  m[0] = m[1] = 0u;
  const int q1 = min(q0 + kQStep, n);
  for (int qs = span_of(st, q0); qs < st.n && st.start[qs] < q1; ++qs) {
    if (!span_vis(st, qs, ks)) continue;
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
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bar(bars->q_full[i]), 1);
      ptx::mbar_init(bar(bars->q_empty[i]), 1);
      ptx::mbar_init(bar(bars->dq_free[i]), 8);
    }
    ptx::mbar_init(bar(bars->s_full), 1);
    ptx::mbar_init(bar(bars->s_read), 8);
    ptx::mbar_init(bar(bars->p_ready), 8);
    ptx::mbar_init(bar(bars->mma_done), 1);
    ptx::fence_mbar_init();
  }
  if (warp == kWarpProd) ptx::tmem_alloc<512>(ptx::smem_u32(&bars->tmem_base));
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::pdl_wait();
  const uint32_t tmem = bars->tmem_base;
  // TMEM: S^T [0, 64), dP^T [64, 128) (one step at a time: the next step's are computed once these are in
  // registers), dQ^T of step i in [128 + 64 (i & 1), +64) (drained while later steps run), dV [256, 384),
  // dK [384, 512)
  constexpr uint32_t kS = 0, kDP = 64, kDQ = 128, kDV = 256, kDK = 384;
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
      for (int qs = 0; qs < n_qsteps; ++qs) {
        if (!step_visible(st, qs * kQStep, k0, n)) continue;
        const uint32_t bi = i & 1, u = i >> 1;
        ptx::mbar_wait(bar(bars->q_empty[bi]), (u & 1) ^ 1);
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
    if (lane == 0) {
      constexpr uint32_t iS = ptx::idesc_f16(0, 0, 0, 0, 128, 64), iDP = ptx::idesc_f16(1, 1, 0, 0, 128, 64),
                         iDV = ptx::idesc_f16(1, 1, 0, 1, 128, 128), iDK = ptx::idesc_f16(0, 0, 0, 1, 128, 128),
                         iDQ = ptx::idesc_f16(0, 0, 1, 1, 128, 64);
      ptx::mbar_wait(bar(bars->kv_full), 0);
      // Software-pipelined: S^T / dP^T of step i + 1 are issued before waiting for step i's P^T / dS^T,
      // so the tensor pipe computes them while the softmax-gradient warps work on step i (and they
      // complete before step i's dV / dK / dQ^T MMAs, which are issued after them).
      auto issue_sdp = [&](uint32_t i) {
        const uint32_t bi = i & 1, u = i >> 1;
        const uint32_t qb = base + kOffQ + bi * kQTile, ob = base + kOffDO + bi * kQTile;
        ptx::mbar_wait(bar(bars->q_full[bi]), u & 1);
        if (i >= 1) ptx::mbar_wait(bar(bars->s_read), (i - 1) & 1);  // S^T / dP^T of step i - 1 are in registers
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kS, desc_k(base + kOffK, kk, kKBox), desc_k(qb, kk, kQBox), iS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDP, desc_k(base + kOffV, kk, kKBox), desc_k(ob, kk, kQBox), iDP, kk > 0);
        ptx::tc_commit(bar(bars->s_full));
      };
      auto next_visible = [&](int qs) {
        while (qs < n_qsteps && !step_visible(st, qs * kQStep, k0, n)) ++qs;
        return qs;
      };
      int qs = next_visible(0);
      if (qs < n_qsteps) issue_sdp(0);
      uint32_t i = 0;
      while (qs < n_qsteps) {
        const uint32_t bi = i & 1, u = i >> 1;
        const int qn = next_visible(qs + 1);
        if (qn < n_qsteps) issue_sdp(i + 1);  // (waits until step i's S^T / dP^T have been read)
        const uint32_t qb = base + kOffQ + bi * kQTile, ob = base + kOffDO + bi * kQTile;
        ptx::mbar_wait(bar(bars->p_ready), i & 1);  // P^T and dS^T of step i are in shared memory
        if (i >= 2) ptx::mbar_wait(bar(bars->dq_free[bi]), (u - 1) & 1);  // dQ^T(i - 2) drained
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_ss(tmem + kDV, desc_k(base + kOffPT, kk, kPTile), desc_mn(ob, kk, kQBox), iDV,
                      (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma_ss(tmem + kDK, desc_k(base + kOffDST, kk, kPTile), desc_mn(qb, kk, kQBox), iDK,
                      (i > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDQ + bi * 64, desc_mn(base + kOffK, kk, kKBox), desc_mn(base + kOffDST, kk, kPTile),
                      iDQ, kk > 0);
        ptx::tc_commit(bar(bars->mma_done));
        ptx::tc_commit(bar(bars->q_empty[bi]));
        qs = qn;
        ++i;
      }
    }
    __syncwarp();
  } else {  // warps 0..7
    // ------------------------------------- softmax-gradient, dQ drain and epilogue --
    // warp w: TMEM lane quadrant w % 4 (key rows, or d rows for dQ^T), query half hq = w / 4 of each step
    const int quad = warp % 4, hq = warp / 4;
    const int r = quad * 32 + lane;
    const uint32_t lb = (uint32_t)(quad * 32) << 16;
    const int key = k0 + r;
    const int ks = span_of(st, min(key, n - 1));
    // dQ^T of a step (thread = d row r, its warp's 32 queries): transposed into the staging tile
    // [64 q][128 d] fp32 (thread r writes column r: conflict-free), then one TMA bulk reduce-add into
    // dQ'[b][q0 .. q0 + 63][h][:] (rows past n clipped).  Staging alternates; its previous reduce must
    // have read it.
    uint32_t n_drain = 0;
    auto drain = [&](uint32_t bi, int q0) {
      const uint32_t sb = base + kOffDQ + (n_drain & 1) * kDQTile;
      if (threadIdx.x == 0) ptx::bulk_wait_read_all();  // (keeps at most one reduce in flight)
      ptx::named_bar_sync(1, 256);
      uint32_t qr[32];
      ptx::tmem_ld32(tmem + lb + kDQ + bi * 64 + hq * 32, qr);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sb + ((hq * 32 + j) * 128 + r) * 4),
                     "f"(__uint_as_float(qr[j]) * scale_q)
                     : "memory");
      ptx::fence_proxy_async_smem();
      ptx::named_bar_sync(1, 256);
      if (threadIdx.x == 0) {
        ptx::tma_reduce_add_4d(&tm_dq, sb, 0, h, q0, b);
        ptx::bulk_commit_group();
      }
      ++n_drain;
    };
    uint32_t i = 0;
    int prev_q0 = 0;
    for (int qs = 0; qs < n_qsteps; ++qs) {
      const int q0 = qs * kQStep;
      if (!step_visible(st, q0, k0, n)) continue;
      const uint32_t bi = i & 1, u = i >> 1;
      uint32_t vm2[2];
      visible_queries(st, ks, q0, n, vm2);
      const uint32_t vm = key < n ? vm2[hq] : 0u;
      ptx::mbar_wait(bar(bars->q_full[bi]), u & 1);    // this step's lse2 / delta are in shared memory
      ptx::mbar_wait(bar(bars->s_full), i & 1);
      ptx::tc_fence_after();
      uint32_t sr[32], dr[32];
      ptx::tmem_ld32(tmem + lb + kS + hq * 32, sr);
      ptx::tmem_ld32(tmem + lb + kDP + hq * 32, dr);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->s_read));  // the next step's S^T / dP^T may be computed
      const float* lv = vec + bi * 128 + hq * 32;
      uint32_t pk[16], dk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float p2[2], d2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int qi = 2 * j + e;
          const bool vis = (vm >> qi) & 1u;
          // (lse2 / delta past n are unwritten workspace: select, never multiply, masked entries)
          const float p = vis ? ptx::ex2(__uint_as_float(sr[qi]) - lv[qi]) : 0.f;
          p2[e] = p;
          d2[e] = vis ? p * (__uint_as_float(dr[qi]) - lv[64 + qi]) : 0.f;
        }
        pk[j] = ptx::pack_bf16x2(p2[0], p2[1]);
        __half2 hh = __floats2half2_rn(d2[0], d2[1]);
        dk[j] = *reinterpret_cast<uint32_t*>(&hh);
      }
      if (i >= 1) {  // the previous step's MMAs have read P^T / dS^T
        ptx::mbar_wait(bar(bars->mma_done), (i - 1) & 1);
        ptx::tc_fence_after();
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // row r of the [128][64] tiles: this warp's 4 chunks of 8 queries, SW128
        const uint32_t o = r * 128 + (((hq * 4 + j) ^ (r & 7)) << 4);
        ptx::st_shared_v4(base + kOffPT + o, pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        ptx::st_shared_v4(base + kOffDST + o, dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
      }
      ptx::fence_proxy_async_smem();  // generic stores -> the tensor core's reads
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->p_ready));
      if (i >= 1) {  // dQ^T of step i - 1 leaves TMEM while step i's MMAs run
        drain((i - 1) & 1, prev_q0);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar(bars->dq_free[(i - 1) & 1]));
      }
      prev_q0 = q0;
      ++i;
    }
    if (i >= 1) {  // the last step's dQ^T (and the final dV / dK)
      ptx::mbar_wait(bar(bars->mma_done), (i - 1) & 1);
      ptx::tc_fence_after();
      drain((i - 1) & 1, prev_q0);
    }
    if (threadIdx.x == 0) ptx::bulk_wait_all();  // the dQ reduces have completed
    // dV (bf16) and dK' (fp32) of this thread's key row, columns [64 hq, 64 hq + 64) (tcgen05.ld is
    // warp-collective: every lane loads, only rows < n store)
    const int64_t row = (((int64_t)b * n + min(key, n - 1)) * H + h) * 128;
    const bool store = key < n;
    if (i == 0) {  // no query sees these keys: zero gradients
      if (store)
        for (int d = hq * 64; d < hq * 64 + 64; d += 8) {
          *reinterpret_cast<uint4*>(dv_out + row + d) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<float4*>(dk_out + row + d) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(dk_out + row + d + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
#pragma unroll 1
      for (int c = 2 * hq; c < 2 * hq + 2; ++c) {
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
}

// B1: delta = <dO, O> per (b, h, s) row and lse2 = lse * log2(e); one warp per row of D = 128
__global__ void delta_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                             const float* __restrict__ lse, float* __restrict__ delta, float* __restrict__ lse2, int B,
                             int n, int H, int n_pad) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (wid >= (int64_t)B * n * H) return;
  const int h = (int)(wid % H), s = (int)((wid / H) % n), b = (int)(wid / ((int64_t)H * n));
  const int64_t row = wid * 128 + lane * 4;  // [b][s][h][d], 4 elements per lane
  const uint2 o = *reinterpret_cast<const uint2*>(out + row), g = *reinterpret_cast<const uint2*>(dout + row);
  const float o4[4] = {__uint_as_float(o.x << 16), __uint_as_float(o.x & 0xFFFF0000u), __uint_as_float(o.y << 16),
                       __uint_as_float(o.y & 0xFFFF0000u)};
  const float g4[4] = {__uint_as_float(g.x << 16), __uint_as_float(g.x & 0xFFFF0000u), __uint_as_float(g.y << 16),
                       __uint_as_float(g.y & 0xFFFF0000u)};
  float acc = 0.f;
#pragma unroll
  for (int e = 0; e < 4; ++e) acc = fmaf(o4[e], g4[e], acc);
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (lane == 0) {  // rows of n_pad (a multiple of 64: the attention backward reads whole 64-query steps)
    const int64_t i = ((int64_t)b * H + h) * n_pad + s;
    delta[i] = acc;
    lse2[i] = lse[((int64_t)b * H + h) * n + s] * 1.4426950408889634f;
  }
}

// B3: prologue backward for one tensor (blockIdx.z: 0 q, 1 k) -- per (token, head) row of D = 128,
// one warp per row, 4 elements (2 rotation pairs) per lane:
//   dy = R(-phi) dx';  dgain += dy * x^;  dx^ = dy * g;  dx = (dx^ - x^ mean(dx^ x^)) / r
// A CTA handles one head and a run of tokens; its gain gradient is reduced in shared memory and
// added once (fp32 atomics).
struct ProBwdArgs {
  const __nv_bfloat16* x[2];  // raw q, k [B][n][H][D]
  const float* dxp[2];        // dq', dk' fp32 [B][n][H][D]
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

__global__ void __launch_bounds__(256) prologue_bwd_kernel(const __grid_constant__ ProBwdArgs a) {
  constexpr int D = 128;
  const int w = blockIdx.z, h = blockIdx.y;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int j0 = 2 * lane;  // this lane's rotation pairs j0, j0 + 1 (elements 4 lane .. 4 lane + 3)
  const float* gp = a.gain[w] + h * D + 4 * lane;
  const float g4[4] = {gp[0], gp[1], gp[2], gp[3]};
  float dg[4] = {0.f, 0.f, 0.f, 0.f};
  const int ax0 = a.axis[j0], ax1 = a.axis[j0 + 1];
  const int items = a.B * a.n;
  for (int it = blockIdx.x * kProBwdTokens + warp; it < min(items, (int)(blockIdx.x + 1) * kProBwdTokens); it += 8) {
    const int b = it / a.n, t = it - b * a.n;
    const int64_t row = (((int64_t)b * a.n + t) * a.H + h) * D + 4 * lane;
    const uint2 xr = *reinterpret_cast<const uint2*>(a.x[w] + row);
    const float x4[4] = {__uint_as_float(xr.x << 16), __uint_as_float(xr.x & 0xFFFF0000u),
                         __uint_as_float(xr.y << 16), __uint_as_float(xr.y & 0xFFFF0000u)};
    float ss = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) ss = fmaf(x4[e], x4[e], ss);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
    const float inv = rsqrtf(ss * (1.0f / D) + a.eps);
    const float4 d4 = *reinterpret_cast<const float4*>(a.dxp[w] + row);
    const int p0 = a.pos[3 * t + ax0], p1 = a.pos[3 * t + ax1];
    const float2 c0 = (unsigned)p0 < (unsigned)a.tab_len ? a.tab[(size_t)p0 * (D / 2) + j0]
                                                         : make_float2((float)cos(p0 * a.omega[j0]), (float)sin(p0 * a.omega[j0]));
    const float2 c1 = (unsigned)p1 < (unsigned)a.tab_len ? a.tab[(size_t)p1 * (D / 2) + j0 + 1]
                                                         : make_float2((float)cos(p1 * a.omega[j0 + 1]), (float)sin(p1 * a.omega[j0 + 1]));
    // dy = R(-phi) dx' per pair
    const float dy[4] = {d4.x * c0.x + d4.y * c0.y, -d4.x * c0.y + d4.y * c0.x,
                         d4.z * c1.x + d4.w * c1.y, -d4.z * c1.y + d4.w * c1.x};
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
    *reinterpret_cast<uint2*>(a.dx[w] + row) = make_uint2(ptx::pack_bf16x2(dx[0], dx[1]), ptx::pack_bf16x2(dx[2], dx[3]));
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
    const int64_t warps = (int64_t)a.B * a.n * a.H;
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
    prologue_bwd_kernel<<<dim3(blocks, (unsigned)a.H, 2), 256, 0, s>>>(p);
    return cudaGetLastError();
  }
}

}  // namespace dz
