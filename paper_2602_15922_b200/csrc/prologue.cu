// prologue.cu -- K1 (attend) / K4 (append): fused per-head RMSNorm + 3D RoPE.
//
//   x'_i = RoPE_3D( x_i / sqrt(mean_j x_j^2 + eps) * g_{h,i} )   for Q and K,
//   V copied unchanged,
// per (token, head) row of D elements (BJ:5 "per-head RMSNorm on Q/K and 3D
// (frame, height, width) RoPE"; readings A1-A9 in DESIGN.md: interleaved pairs
// (2i, 2i+1) inside the axis slices [t | h | w], omega_i = theta^(-2i/d_a)).
// fp32 math; Q' and K' stored fp16 (reading A13), V stays bf16.  Q' is stored
// multiplied by softmax_scale * log2(e), so the attention kernel's scores come
// out of the tensor core already in log2 units (one FMA per score saved).
//
// Two kernels.  H <= 48 at D = 128 (the paper's 40 heads): prologue_loop_kernel, see there.
// More heads: prologue_kernel, a persistent grid (2 CTAs per SM) that walks the (batch, token) items.
// Each item's Q, K, V rows are contiguous H x D blocks in the [B][n][H][D]
// input, so one thread issues three 1D bulk copies (cp.async.bulk, TMA) per
// item into a kStages-deep shared-memory ring, kStages - 1 items ahead of the
// one being processed: HBM reads stay in flight while the CTA computes.  The
// token's D/2 rotation angles (fp64 sincos of p_a * omega_j) go to shared
// memory.  A row of D elements is handled by D/8 threads with one 16-byte
// shared load and one 16-byte global store each; its sum of squares is reduced
// with __shfl_xor inside that thread group.  HBM-bound by design: per token it
// moves (read + write) 2 B x D x H for each of Q, K, V.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"
#include "rmsrope.cuh"

namespace dz {
namespace {

constexpr int kThreads = 256;
#ifndef DZ_PRO_CTAS
#define DZ_PRO_CTAS 2
#endif
#ifndef DZ_PRO_RING_KB
#define DZ_PRO_RING_KB 96
#endif
#ifndef DZ_PRO_LOOP_MINB
#define DZ_PRO_LOOP_MINB 2
#endif
#ifndef DZ_PRO_LOOP_WAVES
#define DZ_PRO_LOOP_WAVES 1
#endif
constexpr int kCtasPerSm = DZ_PRO_CTAS;
constexpr int kMaxStageBytes = DZ_PRO_RING_KB * 1024;  // ring size cap per CTA

using rr::bf16x8_to_f32;
using rr::rope_cs;

// shared-memory carve-up for H heads, nt tensors present, S stages
struct ProSmem {
  int row_bytes, stage_bytes, S;
  __host__ __device__ ProSmem(int H, int D, int nt) {
    row_bytes = H * D * 2;
    stage_bytes = nt * row_bytes;
    S = kMaxStageBytes / stage_bytes;
    S = S < 2 ? 2 : (S > 6 ? 6 : S);
  }
  __host__ __device__ int cs_off() const { return S * stage_bytes; }           // float2 [S][D/2]
  __host__ __device__ int row_off(int D) const { return cs_off() + S * (D / 2) * 8; }  // int64 [H]
  __host__ __device__ int bar_off(int D, int H) const { return (row_off(D) + H * 8 + 7) / 8 * 8; }
  __host__ __device__ int total(int D, int H) const { return bar_off(D, H) + S * 8 + 16; }
};

template <int D>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) prologue_kernel(const PrologueArgs a) {
  constexpr int G = D / 8;               // threads per row (one 16-byte vector each)
  constexpr int kGroups = kThreads / G;  // rows processed side by side
  constexpr int kPer = 3;                // heads per thread in one pass (H <= 48 at D = 128: one pass)
  ptx::pdl_launch_dependents();  // the next kernel may take SMs as our CTAs finish (it waits for us)
  extern __shared__ __align__(128) uint8_t sm[];
  const int H = a.H, tid = threadIdx.x;
  const int g = tid / G, li = tid % G;
  int nt = 0, slot_of[3];
#pragma unroll
  for (int w = 0; w < 3; ++w) slot_of[w] = a.x[w] != nullptr ? nt++ : -1;
  const ProSmem L(H, D, nt);
  float2* cs = reinterpret_cast<float2*>(sm + L.cs_off());
  int64_t* rowoff = reinterpret_cast<int64_t*>(sm + L.row_off(D));
  const uint32_t bar0 = ptx::smem_u32(sm + L.bar_off(D, H));
  const uint32_t ring = ptx::smem_u32(sm);
  // output row offset of head h (destination rank block, local head): one division per head, here only
  for (int h = tid; h < H; h += kThreads) {
    const int dest = h / a.heads_per_dest;
    rowoff[h] = (int64_t)dest * a.y[0].dstride + (int64_t)(h - dest * a.heads_per_dest) * D;
  }
  if (tid == 0) {
    for (int s = 0; s < L.S; ++s) ptx::mbar_init(bar0 + 8 * s, 1);
    ptx::fence_mbar_init();
  }
  const int n_items = a.B * a.n;
  const uint64_t pol = ptx::l2_policy_evict_first();  // activations are read once
  auto issue = [&](int k) {  // bulk loads of this CTA's k-th item into stage k % S
    const int item = blockIdx.x + k * gridDim.x;
    if (item >= n_items) return;
    const int b = item / a.n, t = item - b * a.n;
    const uint32_t st = (uint32_t)(k % L.S), bar = bar0 + 8 * st;
    ptx::mbar_arrive_expect_tx(bar, (uint32_t)L.stage_bytes);
    const int64_t src = ((int64_t)b * a.x_bstride + (int64_t)t * H * D) * 2;
#pragma unroll
    for (int w = 0; w < 3; ++w)
      if (slot_of[w] >= 0)
        ptx::bulk_load(ring + st * L.stage_bytes + slot_of[w] * L.row_bytes,
                       static_cast<const uint8_t*>(a.x[w]) + src, (uint32_t)L.row_bytes, bar, pol);
  };
  // the token's D/2 rotation angles, one per 4th thread so every warp takes a share of the fp64 sincos
  // (the position is loaded one item ahead of its use, so the angle computation never waits on it)
  const int ai = tid >> 2;  // 0 .. 63 >= D/2 - 1
  const bool angle_thread = (tid & 3) == 0 && ai < D / 2;
  auto load_pos = [&](int k) -> int {
    const int item = blockIdx.x + k * gridDim.x;
    if (item >= n_items || !angle_thread) return 0;
    return __ldg(a.pos + 3 * (item % a.n) + a.axis[ai]);
  };
  auto angles = [&](int k, int p) {
    const int item = blockIdx.x + k * gridDim.x;
    if (item >= n_items || !angle_thread) return;
    double sn, cn;
    sincos((double)p * a.omega[ai], &sn, &cn);
    cs[(k % L.S) * (D / 2) + ai] = make_float2((float)cn, (float)sn);
  };
  __syncthreads();  // barriers initialised, row offsets visible
  // the previous kernel of the stream is done and its writes are visible before any input is read:
  // that kernel may be the one that produced q/k/v or the positions
  ptx::pdl_wait();
  if (tid == 0)
    for (int k = 0; k < L.S - 1; ++k) issue(k);
  // gains of this thread's heads (h = g + kGroups * i) and column slice, kept in registers
  const bool gains_in_regs = H <= kGroups * kPer;
  float gq[kPer][8], gk[kPer][8];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int h = g + kGroups * i;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      gq[i][e] = (gains_in_regs && h < H && a.gain[0]) ? __ldg(a.gain[0] + h * D + li * 8 + e) : 0.f;
      gk[i][e] = (gains_in_regs && h < H && a.gain[1]) ? __ldg(a.gain[1] + h * D + li * 8 + e) : 0.f;
    }
  }
  angles(0, load_pos(0));
  int pos_next = load_pos(1);

  for (int k = 0;; ++k) {
    const int item = blockIdx.x + k * gridDim.x;
    if (item >= n_items) break;
    const int b = item / a.n, t = item - b * a.n;
    const int st = k % L.S;
    const int pos_k1 = pos_next;
    pos_next = load_pos(k + 2);
    if (tid == 0) issue(k + L.S - 1);  // its stage was released by the __syncthreads ending item k - 1
    ptx::mbar_wait(bar0 + 8 * st, (uint32_t)((k / L.S) & 1));
    __syncthreads();  // angles of item k visible (written before the barrier that ended item k - 1)
    const uint8_t* stage = sm + st * L.stage_bytes;
    float2 csr[4];  // this thread's 4 rotation pairs (the same for every head and tensor of the item)
    {
      const float4* c4 = reinterpret_cast<const float4*>(cs + st * (D / 2) + li * 4);
      const float4 c0 = c4[0], c1 = c4[1];
      csr[0] = make_float2(c0.x, c0.y);
      csr[1] = make_float2(c0.z, c0.w);
      csr[2] = make_float2(c1.x, c1.y);
      csr[3] = make_float2(c1.z, c1.w);
    }
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      if (slot_of[w] < 0) continue;  // block-uniform
      const OutSlot& o = a.y[w];
      const int64_t base = (int64_t)b * o.bstride + (int64_t)t * o.tstride;
      const uint8_t* src = stage + slot_of[w] * L.row_bytes;
      for (int h0 = 0; h0 < H; h0 += kGroups * kPer) {  // block-uniform trip count (one pass for H <= 48)
        uint4 v[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int h = h0 + g + kGroups * i;
          v[i] = h < H ? *reinterpret_cast<const uint4*>(src + (h * D + li * 8) * 2) : make_uint4(0, 0, 0, 0);
        }
        if (w == 2) {  // V: unchanged bf16 copy into the cache / send slot
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            const int h = h0 + g + kGroups * i;
            if (h < H) reinterpret_cast<uint4*>(o.base)[(base + rowoff[h]) / 8 + li] = v[i];
          }
          continue;
        }
        float f[kPer][8], ss[kPer];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          bf16x8_to_f32(v[i], f[i]);
          ss[i] = rr::chunk_ss(f[i]);
        }
        // butterfly within each half-row, then across the halves (rmsrope.cuh)
#pragma unroll
        for (int m = G / 4; m >= 1; m >>= 1)
#pragma unroll
          for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], m));
#pragma unroll
        for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], G / 2));
        const float sc = w == 0 ? a.q_scale : 1.f;  // Q' leaves pre-scaled by softmax_scale*log2(e)
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          const int h = h0 + g + kGroups * i;
          if (h >= H) continue;
          const float inv = rr::inv_rms(ss[i], D, a.eps);
          float gg[8];
          if (gains_in_regs) {
#pragma unroll
            for (int e = 0; e < 8; ++e) gg[e] = w == 0 ? gq[i][e] : gk[i][e];
          } else {
            const float4* gp = reinterpret_cast<const float4*>(a.gain[w] + h * D + li * 8);
            const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1);
            gg[0] = g0.x; gg[1] = g0.y; gg[2] = g0.z; gg[3] = g0.w;
            gg[4] = g1.x; gg[5] = g1.y; gg[6] = g1.z; gg[7] = g1.w;
          }
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) pk[e] = rr::rot_pair(f[i][2 * e], f[i][2 * e + 1], inv, gg[2 * e], gg[2 * e + 1], csr[e], sc);
          reinterpret_cast<uint4*>(o.base)[(base + rowoff[h]) / 8 + li] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
    angles(k + 1, pos_k1);  // next item's angles into its own slot, off the critical path of the copies
    __syncthreads();  // stage and angles of item k may be refilled
  }
}

// ---- token loop: registers instead of a ring --------------------------------------------
// Thread (g, li) owns column slice li (8 elements) of heads g, g + G', g + 2G' of every present
// tensor.  The persistent ring above (its per-item barriers, 4.5 items per CTA at C1) and a
// one-token-per-CTA variant both left the kernel latency- or instruction-bound.
// Token loop (H <= 48 at D = 128, the default): the per-row arithmetic of prologue_kernel
// with a row per D/8 threads straight from registers; a CTA walks tokens item, item + grid,
// ... and keeps the next token's loads and rotation angles in flight while it processes the
// current one.  The tensors present are a template
// mask (bit w: x[w] given), so only their registers exist; the per-thread head offsets
// (including the SP destination split h / heads_per_dest) are computed once per CTA.
// (It replaced a one-token-per-CTA kernel that ncu showed instruction-bound -- 7060 warp
// instructions per token, mostly per-token address and division arithmetic: attend prologue
// 24.2 -> 22.4 us, append 19.7 -> 17.1 us at C1.)
// DUAL: a second token set (a.j1, one GPU) follows the first in the item sequence; MASK is then the
// union of both sets' tensors and a tensor absent from an item's set (x[w] == nullptr) is skipped.
// PEER: rows go straight to the destination ranks' buffers (a.peer_y, DZ_FLAG_PEER_STORE).
// F8: Q' and K' are stored as E4M3 (DZ_FLAG_FP8_QK; one byte per element, rows of D bytes).
// NT threads, KP head passes per CTA (as prologue_dual2_kernel: 256 x 3, or 320 x 2 for H <= 40 at D = 128)
template <int D, int MASK, bool DUAL, bool PEER = false, bool F8 = false, int NT = 256, int KP = 3>
__global__ void __launch_bounds__(NT, DZ_PRO_LOOP_MINB) prologue_loop_kernel(const PrologueArgs a) {
  constexpr int G = D / 8, kRows = NT / G, kPer = KP;
  ptx::pdl_launch_dependents();
  const int tid = threadIdx.x, g = tid / G, li = tid % G;
  const int H = a.H, items0 = a.B * a.n, items = items0 + (DUAL ? a.B * a.j1.n : 0);
  // item -> (set, batch element, token)
  auto locate = [&](int item, int& b, int& t) -> bool {
    const bool s1 = DUAL && item >= items0;
    const int it = s1 ? item - items0 : item, nn = s1 ? a.j1.n : a.n;
    b = it / nn;
    t = it - b * nn;
    return s1;
  };
  const int64_t tokD = (int64_t)H * D;
  // per (tensor, head slot): output offset inside the token's block, in elements
  int64_t ooff[3][kPer];
  void* pbase[3][kPer];  // PEER: the destination rank's buffer of (tensor, head slot)
  bool hv[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int h = g + kRows * i;
    hv[i] = h < H;
    const int dest = h / a.heads_per_dest;
#pragma unroll
    for (int w = 0; w < 3; ++w)
      if (MASK >> w & 1) {
        ooff[w][i] = (PEER ? 0 : (int64_t)dest * a.y[w].dstride) + (int64_t)(h - dest * a.heads_per_dest) * D + li * 8;
        pbase[w][i] = PEER && hv[i] ? a.peer_y[w][dest] : nullptr;
      }
  }
  auto load = [&](int item, uint4 (&v)[3][kPer]) {
    int b, t;
    const bool s1 = locate(item, b, t);
    const int64_t src = (int64_t)b * (s1 ? a.j1.x_bstride : a.x_bstride) + (int64_t)t * tokD + g * D + li * 8;
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      const void* xw = s1 ? a.j1.x[w] : a.x[w];
      if ((MASK >> w & 1) && (!DUAL || xw != nullptr))
#pragma unroll
        for (int i = 0; i < kPer; ++i)
          if (hv[i])
            v[w][i] = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(xw) + src +
                                                          (int64_t)kRows * i * D));
    }
  };
  // this thread's 4 rotation pairs j = 4 li + e: their axis is fixed, their angle depends on the
  // token's position on that axis; (cos, sin) come from the table (positions two tokens ahead,
  // table entries one token ahead of their use), or are computed for untabulated positions
  int ax[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) ax[e] = a.axis[li * 4 + e];
  auto positions = [&](int item, int (&p)[4]) {
    if (item >= items) return;
    int b, t;
    const int32_t* pos = locate(item, b, t) ? a.j1.pos : a.pos;
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = __ldg(pos + 3 * t + ax[e]);
  };
  auto angles = [&](const int (&p)[4], float2 (&c)[4]) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      c[e] = (unsigned)p[e] < (unsigned)a.rope_len ? __ldg(a.rope_tab + (size_t)p[e] * (D / 2) + li * 4 + e)
                                                   : rope_cs(p[e], a.omega[li * 4 + e]);
  };
  ptx::pdl_wait();  // before the first read of an input (its producer may be the previous kernel)
  uint4 v[3][kPer], vn[3][kPer];
  float2 csr[4], csn[4];
  int pn[4] = {0, 0, 0, 0};
  int item = blockIdx.x;
  if (item < items) {
    load(item, v);
    positions(item, pn);
    angles(pn, csr);
    positions(item + gridDim.x, pn);
  }
  for (; item < items; item += gridDim.x) {
    const int nxt = item + gridDim.x;
    if (nxt < items) {  // in flight while this token is processed
      load(nxt, vn);
      angles(pn, csn);
      positions(nxt + gridDim.x, pn);
    }
    int b, t;
    const bool s1 = locate(item, b, t);
#pragma unroll
    for (int w = 0; w < 3; ++w) {
      if (!(MASK >> w & 1)) continue;
      if (DUAL && (s1 ? a.j1.x[w] : a.x[w]) == nullptr) continue;  // (uniform per item)
      const OutSlot& o = s1 ? a.j1.y[w] : a.y[w];
      const int64_t base = (int64_t)b * o.bstride + (int64_t)t * o.tstride;
      if (w == 2) {
#pragma unroll
        for (int i = 0; i < kPer; ++i)
          if (hv[i])
            reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(PEER ? pbase[w][i] : o.base) + base + ooff[w][i])[0] =
                v[w][i];
        continue;
      }
      float ss[kPer];
      float f[kPer][8];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        bf16x8_to_f32(v[w][i], f[i]);
        ss[i] = rr::chunk_ss(f[i]);
      }
      // butterfly within each half-row, then across the halves (rmsrope.cuh)
#pragma unroll
      for (int m = G / 4; m >= 1; m >>= 1)
#pragma unroll
        for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], m));
#pragma unroll
      for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], G / 2));
      const float sc = w == 0 ? a.q_scale : 1.f;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (!hv[i]) continue;
        const int h = g + kRows * i;
        const float inv = rr::inv_rms(ss[i], D, a.eps);
        const float4* gp = reinterpret_cast<const float4*>(a.gain[w] + h * D + li * 8);
        const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        if constexpr (F8) {  // E4M3 rows of D bytes: this thread's 8 elements are 8 bytes
          uint16_t q8[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            q8[e] = rr::rot_pair_e4m3(f[i][2 * e], f[i][2 * e + 1], inv, gg[2 * e], gg[2 * e + 1], csr[e], sc,
                                      a.f8_mul[w]);
          uint8_t* dst = static_cast<uint8_t*>(PEER ? pbase[w][i] : o.base) + base + ooff[w][i];
          *reinterpret_cast<uint2*>(dst) = make_uint2((uint32_t)q8[0] | ((uint32_t)q8[1] << 16),
                                                      (uint32_t)q8[2] | ((uint32_t)q8[3] << 16));
        } else {
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pk[e] = rr::rot_pair(f[i][2 * e], f[i][2 * e + 1], inv, gg[2 * e], gg[2 * e + 1], csr[e], sc);
          reinterpret_cast<uint4*>(static_cast<__half*>(PEER ? pbase[w][i] : o.base) + base + ooff[w][i])[0] =
              make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
#pragma unroll
    for (int w = 0; w < 3; ++w)
#pragma unroll
      for (int i = 0; i < kPer; ++i) v[w][i] = vn[w][i];
#pragma unroll
    for (int e = 0; e < 4; ++e) csr[e] = csn[e];
  }
}

// The fused append + attend prologue (one GPU, bf16) with two tensor slots per item instead of three:
// an item of the attend set (j0) carries (q, k), an item of the appended set (j1) carries (k, v), so
// slot 0 is q or k and slot 1 is k or v (v: a copy).  Same arithmetic and order as
// prologue_loop_kernel; two thirds of its load registers (no spills at two CTAs per SM).
// NT threads per CTA (NT / (D / 8) head rows per pass), KP passes: 256 x 3 covers 48 heads at D = 128,
// 320 x 2 covers 40 with no idle head slots and two thirds of the load registers (two CTAs per SM
// either way: 20 warps instead of 16)
template <int D, bool F8 = false, int NT = 256, int KP = 3>
__global__ void __launch_bounds__(NT, DZ_PRO_LOOP_MINB) prologue_dual2_kernel(const PrologueArgs a) {
  constexpr int G = D / 8, kRows = NT / G, kPer = KP;
  ptx::pdl_launch_dependents();
  const int tid = threadIdx.x, g = tid / G, li = tid % G;
  const int H = a.H, items0 = a.B * a.n, items = items0 + a.B * a.j1.n;
  // item cursor (set, batch element, token), advanced by gridDim.x without a division except
  // when it crosses into the appended set
  struct Cur {
    int item, b, t;
    bool s1;
  };
  auto at = [&](int item) {
    Cur c;
    c.item = item;
    c.s1 = item >= items0;
    const int it = c.s1 ? item - items0 : item, nn = c.s1 ? a.j1.n : a.n;
    c.b = it / nn;
    c.t = it - c.b * nn;
    return c;
  };
  auto adv = [&](const Cur& c) {
    if (!c.s1 && c.item + (int)gridDim.x >= items0) return at(c.item + (int)gridDim.x);
    Cur d = c;
    const int nn = c.s1 ? a.j1.n : a.n;
    d.item += gridDim.x;
    d.t += gridDim.x;
    while (d.t >= nn) {
      d.t -= nn;
      ++d.b;
    }
    return d;
  };
  const int64_t tokD = (int64_t)H * D;
  int64_t ooff[kPer];  // one GPU: every tensor's row of head h sits at h * D in the token's block
  bool hv[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int h = g + kRows * i;
    hv[i] = h < H;
    ooff[i] = (int64_t)h * D + li * 8;
  }
  auto load = [&](const Cur& c, uint4 (&v)[2][kPer]) {
    const int b = c.b, t = c.t;
    const bool s1 = c.s1;
    const int64_t src = (int64_t)b * (s1 ? a.j1.x_bstride : a.x_bstride) + (int64_t)t * tokD + g * D + li * 8;
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const void* xw = s1 ? a.j1.x[sl + 1] : a.x[sl];
#pragma unroll
      for (int i = 0; i < kPer; ++i)
        if (hv[i])
          v[sl][i] = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(xw) + src + (int64_t)kRows * i * D));
    }
  };
  int ax[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) ax[e] = a.axis[li * 4 + e];
  auto positions = [&](const Cur& c, int (&p)[4]) {
    if (c.item >= items) return;
    const int32_t* pos = c.s1 ? a.j1.pos : a.pos;
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = __ldg(pos + 3 * c.t + ax[e]);
  };
  auto angles = [&](const int (&p)[4], float2 (&c)[4]) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      c[e] = (unsigned)p[e] < (unsigned)a.rope_len ? __ldg(a.rope_tab + (size_t)p[e] * (D / 2) + li * 4 + e)
                                                   : rope_cs(p[e], a.omega[li * 4 + e]);
  };
  ptx::pdl_wait();  // before the first read of an input (its producer may be the previous kernel)
  uint4 v[2][kPer], vn[2][kPer];
  float2 csr[4], csn[4];
  int pn[4] = {0, 0, 0, 0};
  Cur cur = at(blockIdx.x), nxt = adv(cur), nn2 = adv(nxt);  // this item, the next, the one after
  if (cur.item < items) {
    load(cur, v);
    positions(cur, pn);
    angles(pn, csr);
    positions(nxt, pn);
  }
  for (; cur.item < items; cur = nxt, nxt = nn2, nn2 = adv(nn2)) {
    if (nxt.item < items) {  // in flight while this token is processed
      load(nxt, vn);
      angles(pn, csn);
      positions(nn2, pn);
    }
    const int b = cur.b, t = cur.t;
    const bool s1 = cur.s1;
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int w = s1 ? sl + 1 : sl;  // the tensor in this slot: 0 q, 1 k, 2 v (uniform per item)
      const OutSlot& o = s1 ? a.j1.y[w] : a.y[w];
      const int64_t base = (int64_t)b * o.bstride + (int64_t)t * o.tstride;
      if (w == 2) {
#pragma unroll
        for (int i = 0; i < kPer; ++i)
          if (hv[i]) reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(o.base) + base + ooff[i])[0] = v[sl][i];
        continue;
      }
      float ss[kPer];
      float f[kPer][8];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        bf16x8_to_f32(v[sl][i], f[i]);
        ss[i] = rr::chunk_ss(f[i]);
      }
#pragma unroll
      for (int m = G / 4; m >= 1; m >>= 1)
#pragma unroll
        for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], m));
#pragma unroll
      for (int i = 0; i < kPer; ++i) ss[i] = __fadd_rn(ss[i], __shfl_xor_sync(0xffffffffu, ss[i], G / 2));
      const float sc = w == 0 ? a.q_scale : 1.f;
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        if (!hv[i]) continue;
        const int h = g + kRows * i;
        const float inv = rr::inv_rms(ss[i], D, a.eps);
        const float4* gp = reinterpret_cast<const float4*>(a.gain[w] + h * D + li * 8);
        const float4 g0 = __ldg(gp), g1 = __ldg(gp + 1);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        if constexpr (F8) {  // E4M3 rows of D bytes: this thread's 8 elements are 8 bytes
          uint16_t q8[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            q8[e] = rr::rot_pair_e4m3(f[i][2 * e], f[i][2 * e + 1], inv, gg[2 * e], gg[2 * e + 1], csr[e], sc,
                                      a.f8_mul[w]);
          *reinterpret_cast<uint2*>(static_cast<uint8_t*>(o.base) + base + ooff[i]) =
              make_uint2((uint32_t)q8[0] | ((uint32_t)q8[1] << 16), (uint32_t)q8[2] | ((uint32_t)q8[3] << 16));
        } else {
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            pk[e] = rr::rot_pair(f[i][2 * e], f[i][2 * e + 1], inv, gg[2 * e], gg[2 * e + 1], csr[e], sc);
          reinterpret_cast<uint4*>(static_cast<__half*>(o.base) + base + ooff[i])[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
#pragma unroll
    for (int sl = 0; sl < 2; ++sl)
#pragma unroll
      for (int i = 0; i < kPer; ++i) v[sl][i] = vn[sl][i];
#pragma unroll
    for (int e = 0; e < 4; ++e) csr[e] = csn[e];
  }
}

template <int D>
__global__ void rope_table_kernel(float2* __restrict__ tab, int32_t len, const PrologueArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)len * (D / 2)) return;
  const int p = (int)(i / (D / 2)), j = (int)(i % (D / 2));
  tab[i] = rope_cs(p, a.omega[j]);
}

}  // namespace

#ifndef DZ_PRO_NT320
#define DZ_PRO_NT320 1
#endif
// persistent grid of a token-loop kernel: SMs x resident CTAs per SM x DZ_PRO_LOOP_WAVES
template <typename K>
int grid_of(K kernel, int threads) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  return sms * std::max(1, per_sm) * DZ_PRO_LOOP_WAVES;
}

template <int D, int MASK, bool DUAL = false, bool PEER = false, bool F8 = false>
cudaError_t launch_loop(const PrologueArgs& a, cudaStream_t s) {
  const int items = a.B * (a.n + (DUAL ? a.j1.n : 0));
  if (DZ_PRO_NT320 && D == 128 && a.H <= 2 * (320 / (D / 8))) {
    auto k = prologue_loop_kernel<D, MASK, DUAL, PEER, F8, 320, 2>;
    static int grid_cap = 0;
    if (grid_cap == 0) grid_cap = grid_of(k, 320);
    return launch_pdl(k, dim3((unsigned)std::min(items, grid_cap)), dim3(320), 0, s, a);
  }
  auto k = prologue_loop_kernel<D, MASK, DUAL, PEER, F8>;
  static int grid_cap = 0;
  if (grid_cap == 0) grid_cap = grid_of(k, 256);
  return launch_pdl(k, dim3((unsigned)std::min(items, grid_cap)), dim3(256), 0, s, a);
}

// the two-slot fused prologue when the sets are (q, k) and (k, v); false: use the three-slot loop
template <int D, bool F8>
bool launch_dual2(const PrologueArgs& a, cudaStream_t s, cudaError_t& err) {
  static const bool dual3 = getenv("DZ_PRO_DUAL3") != nullptr;  // A/B switch (diagnostics)
  if (dual3 || !(a.x[0] && a.x[1] && !a.x[2] && !a.j1.x[0] && a.j1.x[1] && a.j1.x[2])) return false;
  const int items = a.B * (a.n + a.j1.n);
  if (DZ_PRO_NT320 && D == 128 && a.H <= 2 * (320 / (D / 8))) {
    static int grid_cap = 0;
    if (grid_cap == 0) grid_cap = grid_of(prologue_dual2_kernel<D, F8, 320, 2>, 320);
    err = launch_pdl(prologue_dual2_kernel<D, F8, 320, 2>, dim3((unsigned)std::min(items, grid_cap)), dim3(320), 0, s, a);
    return true;
  }
  static int grid_cap = 0;
  if (grid_cap == 0) grid_cap = grid_of(prologue_dual2_kernel<D, F8>, 256);
  err = launch_pdl(prologue_dual2_kernel<D, F8>, dim3((unsigned)std::min(items, grid_cap)), dim3(256), 0, s, a);
  return true;
}

template <int D>
cudaError_t launch_pro(const PrologueArgs& a, cudaStream_t s) {
  if (a.fp8) {  // E4M3 Q'/K' (one GPU, token loop): attend (q, k [, v]), append (k, v), both in one launch
    if (a.peer || a.H > 3 * (256 / (D / 8))) return cudaErrorInvalidValue;
    if (a.j1.n > 0) {
      cudaError_t e;
      if (launch_dual2<D, true>(a, s, e)) return e;
      return launch_loop<D, 7, true, false, true>(a, s);
    }
    const int mask = (a.x[0] ? 1 : 0) | (a.x[1] ? 2 : 0) | (a.x[2] ? 4 : 0);
    switch (mask) {
      case 3: return launch_loop<D, 3, false, false, true>(a, s);
      case 6: return launch_loop<D, 6, false, false, true>(a, s);
      case 7: return launch_loop<D, 7, false, false, true>(a, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (a.peer) {  // peer stores (Ulysses, one node): q, k, v (attend) or k, v (append); token loop only
    if (a.H > 3 * (256 / (D / 8))) return cudaErrorInvalidValue;
    if (a.x[0]) return launch_loop<D, 7, false, true>(a, s);
    return launch_loop<D, 6, false, true>(a, s);
  }
  if (a.j1.n > 0) {  // two token sets in one launch (one GPU, H within one pass of the token loop)
    if (a.H > 3 * (256 / (D / 8))) return cudaErrorInvalidValue;
    cudaError_t e;
    if (launch_dual2<D, false>(a, s, e)) return e;
    return launch_loop<D, 7, true>(a, s);
  }
  static const bool force_ring = getenv("DZ_PRO_RING") != nullptr;  // diagnostics: the TMA-ring kernel
  if (a.H <= 3 * (256 / (D / 8)) && !force_ring) {
    const int mask = (a.x[0] ? 1 : 0) | (a.x[1] ? 2 : 0) | (a.x[2] ? 4 : 0);
    switch (mask) {
      case 1: return launch_loop<D, 1>(a, s);
      case 2: return launch_loop<D, 2>(a, s);
      case 3: return launch_loop<D, 3>(a, s);
      case 4: return launch_loop<D, 4>(a, s);
      case 5: return launch_loop<D, 5>(a, s);
      case 6: return launch_loop<D, 6>(a, s);
      case 7: return launch_loop<D, 7>(a, s);
      default: return cudaSuccess;
    }
  }
  // more heads than one pass of the CTA: the persistent ring
  int nt = 0;
  for (int w = 0; w < 3; ++w) nt += a.x[w] != nullptr;
  const ProSmem L(a.H, D, nt);
  const int smem = L.total(D, a.H);
  if (L.stage_bytes > 2 * kMaxStageBytes) return cudaErrorInvalidValue;  // heads beyond the ring's reach
  auto k = prologue_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int items = a.B * a.n;
  const int grid = items < kCtasPerSm * sms ? items : kCtasPerSm * sms;
  return launch_pdl(k, dim3(grid), dim3(kThreads), (size_t)smem, s, a);
}

cudaError_t launch_rope_table(float2* tab, int32_t len, const PrologueArgs& a, cudaStream_t s) {
  const int64_t n = (int64_t)len * (a.D / 2);
  const unsigned grid = (unsigned)((n + 255) / 256);
  if (a.D == 128) rope_table_kernel<128><<<grid, 256, 0, s>>>(tab, len, a);
  else if (a.D == 64) rope_table_kernel<64><<<grid, 256, 0, s>>>(tab, len, a);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_prologue(const PrologueArgs& a, cudaStream_t s) {
  if (a.n == 0 || a.B == 0) return cudaSuccess;
  if (a.D == 128) return launch_pro<128>(a, s);
  if (a.D == 64) return launch_pro<64>(a, s);
  return cudaErrorInvalidValue;
}

// K5: [N src][B][n_loc][Hl][D] -> [B][n_loc][H = N*Hl][D], one 16-byte vector per thread.
__global__ void sp_unpack_kernel(const uint4* __restrict__ recv, uint4* __restrict__ out, int N, int B, int n_loc,
                                 int Hl, int vec_per_row) {
  const int64_t total = (int64_t)N * B * n_loc * Hl * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i;
    const int v = r % vec_per_row; r /= vec_per_row;
    const int hl = r % Hl; r /= Hl;
    const int t = r % n_loc; r /= n_loc;
    const int b = r % B; r /= B;
    const int src = (int)r;
    const int64_t o = (((int64_t)b * n_loc + t) * (N * Hl) + (int64_t)src * Hl + hl) * vec_per_row + v;
    out[o] = recv[i];
  }
}

cudaError_t launch_sp_unpack(const void* recv, void* out, int32_t N, int32_t B, int32_t n_loc, int32_t Hl, int32_t D,
                             cudaStream_t s) {
  const int vpr = D / 8;
  const int64_t total = (int64_t)N * B * n_loc * Hl * vpr;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
  sp_unpack_kernel<<<(unsigned)blocks, threads, 0, s>>>(static_cast<const uint4*>(recv), static_cast<uint4*>(out), N,
                                                        B, n_loc, Hl, vpr);
  return cudaGetLastError();
}

}  // namespace dz
