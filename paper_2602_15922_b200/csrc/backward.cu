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

constexpr int kBwdTile = 128;        // keys per CTA, queries per step
constexpr int kBwdThreads = 192;     // warps 0..3 compute (TMEM lane quadrants), warp 4 TMA + MMA, warp 5 idle
constexpr int kTileBytes = 128 * 128 * 2;  // one [128][128] 16-bit tile as two [128][64] SW128 boxes
constexpr int kBoxBytes = 128 * 128;       // one [128 rows][64 cols] box

// shared-memory map
constexpr int kOffK = 0, kOffV = kTileBytes, kOffQ = 2 * kTileBytes, kOffDO = 3 * kTileBytes,
              kOffPT = 4 * kTileBytes, kOffDST = 5 * kTileBytes, kOffVec = 6 * kTileBytes,  // lse2[128], delta[128]
              kOffBar = kOffVec + 1024, kBwdSmem = kOffBar + 1024 + 1024;

struct BwdBars {
  uint64_t kv_full, q_full, s_full, p_ready, mma_done, dq_free;
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
// any visible (query, key) pair between query tile [q0, q0+128) and key tile [k0, k0+128) (both < n)
__device__ __forceinline__ bool tile_visible(const SpanTable& st, int q0, int k0, int n) {
  const int q1 = min(q0 + kBwdTile, n), k1 = min(k0 + kBwdTile, n);
  for (int ks = span_of(st, k0); ks < st.n && st.start[ks] < k1; ++ks)
    for (int qs = span_of(st, q0); qs < st.n && st.start[qs] < q1; ++qs)
      if (span_vis(st, qs, ks)) return true;
  return false;
}
// visible queries of key span ks among [q0, q0 + 128): 128-bit mask
__device__ __forceinline__ void visible_queries(const SpanTable& st, int ks, int q0, int n, uint32_t (&m)[4]) {
  m[0] = m[1] = m[2] = m[3] = 0u;
  const int q1 = min(q0 + kBwdTile, n);
  for (int qs = span_of(st, q0); qs < st.n && st.start[qs] < q1; ++qs) {
    if (!span_vis(st, qs, ks)) continue;
    const int a = max(st.start[qs], q0) - q0, b = min(st.start[qs + 1], q1) - q0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int lo = min(max(a - 32 * w, 0), 32), hi = min(max(b - 32 * w, 0), 32);
      if (hi > lo) m[w] |= (hi == 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~(lo == 32 ? 0xffffffffu : ((1u << lo) - 1u));
    }
  }
}

// element (r, c) of a [128][128] 16-bit tile stored as two SW128 boxes: byte offset of its 16-byte chunk
__device__ __forceinline__ uint32_t chunk_off(int r, int c8) {  // c8 = column / 8 (0..15)
  return (c8 / 8) * kBoxBytes + r * 128 + (((c8 % 8) ^ (r & 7)) << 4);
}
// descriptors: K-major (rows = M or N, K along the 128-byte rows) and MN-major (rows = K) views of a tile
__device__ __forceinline__ uint64_t desc_k(uint32_t tile, int kk) {  // K-step kk of 16 elements
  return ptx::sdesc_sw128(tile + (kk / 4) * kBoxBytes + (kk % 4) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t desc_mn(uint32_t tile, int kk) {  // K-step kk = 16 rows; 64-col blocks at LBO
  return ptx::sdesc_sw128(tile + kk * 16 * 128, kBoxBytes, 1024);
}

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const float* __restrict__ lse2, const float* __restrict__ delta, float* __restrict__ dq_acc,
                    float* __restrict__ dk_out, __nv_bfloat16* __restrict__ dv_out, int B, int H, int n,
                    float scale_q, float scale_k, const __grid_constant__ SpanTable st) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  BwdBars* bars = reinterpret_cast<BwdBars*>(smem + kOffBar);
  float* vec = reinterpret_cast<float*>(smem + kOffVec);  // lse2[128], delta[128] of the current query tile
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tiles = (n + kBwdTile - 1) / kBwdTile;
  const int kt = blockIdx.x % n_tiles, bh = blockIdx.x / n_tiles, h = bh % H, b = bh / H;
  const int k0 = kt * kBwdTile;
  auto bar = [&](uint64_t& x) { return ptx::smem_u32(&x); };

  if (threadIdx.x == 0) {
    ptx::mbar_init(bar(bars->kv_full), 1);
    ptx::mbar_init(bar(bars->q_full), 1);
    ptx::mbar_init(bar(bars->s_full), 1);
    ptx::mbar_init(bar(bars->p_ready), 4);
    ptx::mbar_init(bar(bars->mma_done), 1);
    ptx::mbar_init(bar(bars->dq_free), 4);
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc<512>(ptx::smem_u32(&bars->tmem_base));
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  ptx::pdl_wait();
  const uint32_t tmem = bars->tmem_base;
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 384, kDQ = 0;


  if (warp == 4) {
    // ------------------------------------------------------ TMA + MMA (one thread) --
    if (lane == 0) {
      const uint64_t pol = ptx::l2_policy_evict_last();
      ptx::mbar_arrive_expect_tx(bar(bars->kv_full), 2 * kTileBytes);
      for (int x = 0; x < 2; ++x) {
        ptx::tma_load_4d(base + kOffK + x * kBoxBytes, &tm_k, bar(bars->kv_full), x * 64, h, k0, b, pol);
        ptx::tma_load_4d(base + kOffV + x * kBoxBytes, &tm_v, bar(bars->kv_full), x * 64, h, k0, b, pol);
      }
      ptx::mbar_wait(bar(bars->kv_full), 0);
      constexpr uint32_t iS = ptx::idesc_f16(0, 0, 0, 0, 128, 128), iDP = ptx::idesc_f16(1, 1, 0, 0, 128, 128),
                         iDV = ptx::idesc_f16(1, 1, 0, 1, 128, 128), iDK = ptx::idesc_f16(0, 0, 0, 1, 128, 128),
                         iDQ = ptx::idesc_f16(0, 0, 1, 1, 128, 128);
      uint32_t it = 0;
      for (int qt = 0; qt < n_tiles; ++qt) {
        if (!tile_visible(st, qt * kBwdTile, k0, n)) continue;
        const uint32_t ph = it & 1;
        if (it > 0) ptx::mbar_wait(bar(bars->dq_free), ph ^ 1);  // dQ^T (cols 0..127) has been read
        ptx::mbar_arrive_expect_tx(bar(bars->q_full), 2 * kTileBytes);
        for (int x = 0; x < 2; ++x) {
          ptx::tma_load_4d(base + kOffQ + x * kBoxBytes, &tm_q, bar(bars->q_full), x * 64, h, qt * kBwdTile, b, pol);
          ptx::tma_load_4d(base + kOffDO + x * kBoxBytes, &tm_do, bar(bars->q_full), x * 64, h, qt * kBwdTile, b,
                           pol);
        }
        ptx::mbar_wait(bar(bars->q_full), ph);
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) ptx::mma_ss(tmem + kS, desc_k(base + kOffK, kk), desc_k(base + kOffQ, kk), iS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDP, desc_k(base + kOffV, kk), desc_k(base + kOffDO, kk), iDP, kk > 0);
        ptx::tc_commit(bar(bars->s_full));
        ptx::mbar_wait(bar(bars->p_ready), ph);  // P^T and dS^T are in shared memory
        ptx::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDV, desc_k(base + kOffPT, kk), desc_mn(base + kOffDO, kk), iDV, (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDK, desc_k(base + kOffDST, kk), desc_mn(base + kOffQ, kk), iDK, (it > 0 || kk > 0) ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma_ss(tmem + kDQ, desc_mn(base + kOffK, kk), desc_mn(base + kOffDST, kk), iDQ, kk > 0);
        ptx::tc_commit(bar(bars->mma_done));
        ++it;
      }
    }
    __syncwarp();
  } else if (warp < 4) {
    // ------------------------------------------ softmax-gradient and epilogue warps --
    const int r = warp * 32 + lane;                         // TMEM lane: key row r (S^T, dP^T, dV, dK) / d (dQ^T)
    const uint32_t lb = (uint32_t)(warp * 32) << 16;
    const int key = k0 + r;
    const int ks = span_of(st, min(key, n - 1));
    uint32_t it = 0;
    for (int qt = 0; qt < n_tiles; ++qt) {
      const int q0 = qt * kBwdTile;
      if (!tile_visible(st, q0, k0, n)) continue;
      const uint32_t ph = it & 1;
      {  // this tile's lse2 / delta into shared memory (the previous tile's reads ended with dq_free)
        const int q = min(q0 + r, n - 1);
        vec[r] = lse2[((int64_t)b * H + h) * n + q];
        vec[128 + r] = delta[((int64_t)b * H + h) * n + q];
      }
      ptx::named_bar_sync(1, 128);
      uint32_t vm[4];
      visible_queries(st, ks, q0, n, vm);
      if (key >= n) vm[0] = vm[1] = vm[2] = vm[3] = 0u;
      ptx::mbar_wait(bar(bars->s_full), ph);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {  // 32 queries at a time
        uint32_t sr[32], dr[32];
        ptx::tmem_ld32(tmem + lb + kS + c * 32, sr);
        ptx::tmem_ld32(tmem + lb + kDP + c * 32, dr);
        ptx::tmem_wait_ld();
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float p2[2], d2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int qi = c * 32 + 2 * i + e;
            const bool vis = (vm[c] >> (2 * i + e)) & 1u;
            const float p = vis ? ptx::ex2(__uint_as_float(sr[2 * i + e]) - vec[qi]) : 0.f;
            p2[e] = p;
            d2[e] = p * (__uint_as_float(dr[2 * i + e]) - vec[128 + qi]);
          }
          pk[i] = ptx::pack_bf16x2(p2[0], p2[1]);
          __half2 hh = __floats2half2_rn(d2[0], d2[1]);
          dk[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t o = chunk_off(r, c * 4 + j);
          ptx::st_shared_v4(base + kOffPT + o, pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          ptx::st_shared_v4(base + kOffDST + o, dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
        }
      }
      ptx::fence_proxy_async_smem();  // generic stores -> the tensor core's reads
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->p_ready));
      // dQ^T (thread = d row r) -> fp32 atomics into dQ'[b][q][h][r], coalesced over d
      ptx::mbar_wait(bar(bars->mma_done), ph);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t qr[32];
        ptx::tmem_ld32(tmem + lb + kDQ + c * 32, qr);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int q = q0 + c * 32 + i;
          if (q < n) atomicAdd(dq_acc + (((int64_t)b * n + q) * H + h) * 128 + r, __uint_as_float(qr[i]) * scale_q);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->dq_free));
      ++it;
    }
    // dV (bf16) and dK' (fp32) of this thread's key row (tcgen05.ld is warp-collective: every lane
    // loads, only rows < n store)
    const int64_t row = (((int64_t)b * n + min(key, n - 1)) * H + h) * 128;
    const bool store = key < n;
    if (it == 0) {  // no query sees these keys: zero gradients
      if (store)
        for (int d = 0; d < 128; d += 8) {
          *reinterpret_cast<uint4*>(dv_out + row + d) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<float4*>(dk_out + row + d) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(dk_out + row + d + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
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
  if (warp == 4) ptx::tmem_dealloc<512>(tmem);
}

// B1: delta = <dO, O> per (b, h, s) row and lse2 = lse * log2(e); one warp per row of D = 128
__global__ void delta_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
                             const float* __restrict__ lse, float* __restrict__ delta, float* __restrict__ lse2, int B,
                             int n, int H) {
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
  if (lane == 0) {
    const int64_t i = ((int64_t)b * H + h) * n + s;
    delta[i] = acc;
    lse2[i] = lse[i] * 1.4426950408889634f;
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
        a.B, a.n, a.H);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // B2
  {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.n + kBwdTile - 1) / kBwdTile;
    e = launch_pdl(attn_bwd_kernel, dim3((unsigned)(a.B * a.H * tiles)), dim3(kBwdThreads), (size_t)kBwdSmem, s,
                   a.tm_k, a.tm_v, a.tm_q, a.tm_do, a.lse2, a.delta, a.dq_acc, a.dk, static_cast<__nv_bfloat16*>(a.dv),
                   a.B, a.H, a.n, a.scale_q, a.scale_k, a.spans);
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
