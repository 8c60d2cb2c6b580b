// attention.cu -- K2: block-causal chunk attention on tcgen05 tensor cores.
//
// Computes, for every (b, h, query s) of the current chunk,
//     O_s = sum_j softmax_j(<q'_s, k'_j> * scale) v_j
// over the visible keys j = the committed clean chunks plus the current chunk
// (Fig. 10 / l.505; Alg. 2 l.584-585; BJ:5).  For attend_chunk every
// committed key and every own-chunk key is visible, so the only masked pairs
// are out-of-bounds columns of the last KV tile.
//
// Structure (one persistent CTA per SM, 12 warps):
//   warp 0       TMA producer: Q tile pair once per unit, then K_j, V_j into a
//                ring of 32 KB stages (cp.async.bulk.tensor, SW128).
//   warp 1       MMA issuer (one thread): S_t = Q_t K_j^T (SS, f16 x f16 -> f32
//                in TMEM), O_t += P_t V_j (TS, P bf16 from TMEM, V bf16 smem).
//   warp 2       TMEM allocator (512 columns: S0 S1 O0 O1).
//   warps 4..7   softmax for Q tile 0, warps 8..11 for Q tile 1: one thread per
//                query row (TMEM lane), register-resident online softmax with
//                lazy rescaling (only when the running max grows by > 2^8),
//                P written back over S in TMEM, epilogue O / l -> bf16 -> HBM.
// Two Q tiles of the same head share every K/V stage; while one tile's
// softmax runs, the tensor core works on the other tile (ping-pong).
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace dz {
namespace {

constexpr int BM = 128;        // query rows per tile (MMA M)
constexpr int BN = 128;        // keys per KV tile (MMA N of QK^T, K of PV)
constexpr int kThreads = 384;  // 12 warps
constexpr float kRescaleLog2 = 8.0f;

template <int D>
struct Cfg {
  static constexpr int kBoxes = D / 64;                   // 64-element (128 B) SW128 boxes per row
  static constexpr int kTileBytes = BM * D * 2;           // Q / K / V tile (fp16 / bf16)
  static constexpr int kStages = D == 128 ? 4 : 8;
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kTileBytes;
  static constexpr int kBarOff = kKVOff + kStages * kTileBytes;
  static constexpr int kSmem = kBarOff + 256 + 1024;      // + barriers + 1 KB alignment slack
  static constexpr uint32_t kIdescQK = ptx::idesc_f16(0, 0, 0, 0, BM, BN);  // f16 x f16, K-major both
  static constexpr uint32_t kIdescPV = ptx::idesc_f16(1, 1, 0, 1, BM, D);   // bf16 P (TMEM) x bf16 V (MN-major)
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t s_full[2], p_full[2], o_full[2], o_empty[2];
  uint64_t kv_full[8], kv_empty[8];
  uint32_t tmem_base;
};

__device__ __forceinline__ void decode_unit(int u, int n_qpairs, int H, int& b, int& h, int& qp) {
  qp = u % n_qpairs;
  const int bh = u / n_qpairs;
  h = bh % H;
  b = bh / H;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, __nv_bfloat16* __restrict__ out, int64_t o_bstride,
                    int64_t o_tstride, float* __restrict__ lse, uint8_t* __restrict__ tile_map, int B, int H,
                    int nq, int kv_len, float scale_log2) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  // SW128 operands need 1024-byte aligned tiles.
  const uint32_t raw = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kBarOff);
  const uint32_t sQ = base + C::kQOff;
  const uint32_t sKV = base + C::kKVOff;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_qtiles = (nq + BM - 1) / BM;
  const int n_qpairs = (n_qtiles + 1) / 2;
  const int n_units = B * H * n_qpairs;
  const int nkv = (kv_len + BN - 1) / BN;

  auto bar = [&](uint64_t& b) { return ptx::smem_u32(&b); };

  if (warp == 0 && lane == 0) {
    ptx::mbar_init(bar(bars->q_full), 1);
    ptx::mbar_init(bar(bars->q_empty), 1);
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(bar(bars->s_full[t]), 1);
      ptx::mbar_init(bar(bars->p_full[t]), 4);
      ptx::mbar_init(bar(bars->o_full[t]), 1);
      ptx::mbar_init(bar(bars->o_empty[t]), 4);
    }
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(bar(bars->kv_full[s]), 1);
      ptx::mbar_init(bar(bars->kv_empty[s]), 1);
    }
    ptx::fence_mbar_init();
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) ptx::tmem_alloc<512>(ptx::smem_u32(&bars->tmem_base));
  if (blockIdx.x == 0 && threadIdx.x == 0) ptx::g_dz_watchdog[6] = ptx::smem_u32(bars);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer --
    const uint64_t pol_q = ptx::l2_policy_evict_first();
    const uint64_t pol_kv = ptx::l2_policy_evict_last();
    uint32_t stage = 0, phase = 0, q_phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int b, h, qp;
      decode_unit(u, n_qpairs, H, b, h, qp);
      ptx::mbar_wait(bar(bars->q_empty), q_phase ^ 1);
      q_phase ^= 1;
      if (lane == 0) {
        // the second tile of the last pair may lie wholly past nq: do not load it
        // (its rows are computed on stale data and never stored).
        const int tiles = (2 * qp + 1 < n_qtiles) ? 2 : 1;
        ptx::mbar_arrive_expect_tx(bar(bars->q_full), tiles * C::kTileBytes);
        for (int t = 0; t < tiles; ++t)
          for (int x = 0; x < C::kBoxes; ++x)
            ptx::tma_load_4d(sQ + t * C::kTileBytes + x * BM * 128, &tm_q, bar(bars->q_full), x * 64, h,
                             (2 * qp + t) * BM, b, pol_q);
      }
      for (int j = 0; j < nkv; ++j) {
        for (int kv = 0; kv < 2; ++kv) {  // K_j then V_j
          ptx::mbar_wait(bar(bars->kv_empty[stage]), phase ^ 1);
          if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bar(bars->kv_full[stage]), C::kTileBytes);
            for (int x = 0; x < C::kBoxes; ++x)
              ptx::tma_load_4d(sKV + stage * C::kTileBytes + x * BN * 128, kv == 0 ? &tm_k : &tm_v,
                               bar(bars->kv_full[stage]), x * 64, h, j * BN, b, pol_kv);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer --
    uint32_t stage = 0, phase = 0, q_phase = 0;
    uint32_t p_phase[2] = {0, 0}, oe_phase[2] = {0, 0};
    const uint32_t tS[2] = {tmem + 0, tmem + 128};
    const uint32_t tO[2] = {tmem + 256, tmem + 384};
    auto qk = [&](int t, uint32_t kst) {
      const uint32_t qa = sQ + t * C::kTileBytes, ka = sKV + kst * C::kTileBytes;
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = (kk / 4) * (BM * 128) + (kk % 4) * 32;
        ptx::mma_ss(tS[t], ptx::sdesc_sw128(qa + off, 16, 1024), ptx::sdesc_sw128(ka + off, 16, 1024),
                    C::kIdescQK, kk > 0);
      }
    };
    auto pv = [&](int t, uint32_t vst, bool acc) {
      const uint32_t va = sKV + vst * C::kTileBytes;
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk)
        ptx::mma_ts(tO[t], tS[t] + kk * 8, ptx::sdesc_sw128(va + kk * 16 * 128, BN * 128, 1024), C::kIdescPV,
                    (acc || kk > 0) ? 1u : 0u);
    };
    auto next = [&](uint32_t& st) {
      st = stage;
      if (++stage == C::kStages) { stage = 0; phase ^= 1; }
    };
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      ptx::mbar_wait(bar(bars->q_full), q_phase);
      q_phase ^= 1;
      uint32_t k_st, v_st;
      ptx::mbar_wait(bar(bars->kv_full[stage]), phase);
      next(k_st);
      ptx::tc_fence_after();
      if (lane == 0) {
        for (int t = 0; t < 2; ++t) {
          qk(t, k_st);
          ptx::tc_commit(bar(bars->s_full[t]));
        }
        ptx::tc_commit(bar(bars->kv_empty[k_st]));
        if (nkv == 1) ptx::tc_commit(bar(bars->q_empty));
      }
      __syncwarp();
      for (int j = 1; j < nkv; ++j) {
        ptx::mbar_wait(bar(bars->kv_full[stage]), phase);  // V_{j-1}
        next(v_st);
        ptx::mbar_wait(bar(bars->kv_full[stage]), phase);  // K_j
        next(k_st);
        for (int t = 0; t < 2; ++t) {
          ptx::mbar_wait(bar(bars->p_full[t]), p_phase[t]);
          p_phase[t] ^= 1;
          if (j == 1) {
            ptx::mbar_wait(bar(bars->o_empty[t]), oe_phase[t] ^ 1);
            oe_phase[t] ^= 1;
          }
          ptx::tc_fence_after();
          if (lane == 0) {
            pv(t, v_st, j > 1);
            qk(t, k_st);
            ptx::tc_commit(bar(bars->s_full[t]));
          }
          __syncwarp();
        }
        if (lane == 0) {
          ptx::tc_commit(bar(bars->kv_empty[v_st]));
          ptx::tc_commit(bar(bars->kv_empty[k_st]));
          if (j == nkv - 1) ptx::tc_commit(bar(bars->q_empty));
        }
        __syncwarp();
      }
      ptx::mbar_wait(bar(bars->kv_full[stage]), phase);  // V_{nkv-1}
      next(v_st);
      for (int t = 0; t < 2; ++t) {
        ptx::mbar_wait(bar(bars->p_full[t]), p_phase[t]);
        p_phase[t] ^= 1;
        if (nkv == 1) {
          ptx::mbar_wait(bar(bars->o_empty[t]), oe_phase[t] ^ 1);
          oe_phase[t] ^= 1;
        }
        ptx::tc_fence_after();
        if (lane == 0) {
          pv(t, v_st, nkv > 1);
          ptx::tc_commit(bar(bars->o_full[t]));
        }
        __syncwarp();
      }
      if (lane == 0) ptx::tc_commit(bar(bars->kv_empty[v_st]));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------------------------------------- softmax + epilogue --
    const int t = (warp - 4) / 4;
    const int quad = warp % 4;
    const int row = quad * 32 + lane;
    const uint32_t lane_bits = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_bits + t * 128;
    const uint32_t tO = tmem + lane_bits + 256 + t * 128;
    uint32_t s_phase = 0, of_phase = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      int b, h, qp;
      decode_unit(u, n_qpairs, H, b, h, qp);
      float m_used = -INFINITY;  // running max in log2 units of scaled scores
      float l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        ptx::mbar_wait(bar(bars->s_full[t]), s_phase);
        s_phase ^= 1;
        ptx::tc_fence_after();
        float s[BN];
        {
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            ptx::tmem_ld32(tS + c * 32, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
          }
        }
        const int kv_valid = kv_len - j * BN;
        if (tile_map != nullptr && u < n_qpairs && row == 0) {
          // debug: the kernel's own per-tile decision for unit (b=0, h=0):
          // 2 FULL (no column masked, all rows in bounds), 1 PARTIAL (masked).
          const int qt = 2 * qp + t;
          if (qt < n_qtiles) tile_map[qt * nkv + j] = (kv_valid >= BN && nq - qt * BM >= BM) ? 2 : 1;
        }
        if (kv_valid < BN) {
#pragma unroll
          for (int i = 0; i < BN; ++i)
            if (i >= kv_valid) s[i] = -INFINITY;
        }
        float mx = s[0];
#pragma unroll
        for (int i = 1; i < BN; ++i) mx = fmaxf(mx, s[i]);
        const float mx_s = mx * scale_log2;
        // Lazy rescale: a row moves its softmax base only when its max grew by
        // more than 2^8.  The decision is made per row, but the TMEM traffic it
        // needs (tcgen05.ld/st are warp-collective) is issued by the whole warp.
        const bool grow = mx_s > m_used + kRescaleLog2;
        const bool rescale = grow && j > 0 && m_used != -INFINITY;
        if (__any_sync(0xffffffffu, rescale)) {
          // O_t is quiescent here: PV_t(j-1) completed before S_t(j) was committed.
          const float alpha = rescale ? ptx::ex2(m_used - mx_s) : 1.f;
          l *= alpha;
          uint32_t r[32];
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            ptx::tmem_ld32(tO + c * 32, r);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            ptx::tmem_st32(tO + c * 32, r);
          }
          ptx::tmem_wait_st();
        }
        if (grow) m_used = mx_s;
        const float nbase = (m_used == -INFINITY) ? 0.f : -m_used;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float p0 = ptx::ex2(fmaf(s[c * 32 + 2 * i], scale_log2, nbase));
            const float p1 = ptx::ex2(fmaf(s[c * 32 + 2 * i + 1], scale_log2, nbase));
            l += p0 + p1;
            pk[i] = ptx::pack_bf16x2(p0, p1);
          }
          ptx::tmem_st16(tS + c * 16, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bar(bars->p_full[t]));
      }
      // epilogue: O_t / l -> bf16 -> HBM
      ptx::mbar_wait(bar(bars->o_full[t]), of_phase);
      of_phase ^= 1;
      ptx::tc_fence_after();
      const int s_idx = (2 * qp + t) * BM + row;
      const float inv_l = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = out + b * o_bstride + (int64_t)s_idx * o_tstride + (int64_t)h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        __syncwarp();  // reconverge after the row-dependent store below
        ptx::tmem_ld32(tO + c * 32, r);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pk[i] = ptx::pack_bf16x2(__uint_as_float(r[2 * i]) * inv_l, __uint_as_float(r[2 * i + 1]) * inv_l);
        if (s_idx < nq) {
#pragma unroll
          for (int v = 0; v < 4; ++v)
            ptx::st_global_v4(orow + c * 32 + v * 8, pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
        }
      }
      if (lse != nullptr && s_idx < nq)
        lse[((int64_t)b * H + h) * nq + s_idx] =
            (l > 0.f) ? (m_used + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bar(bars->o_empty[t]));
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<512>(tmem);
}

template <int D>
cudaError_t launch_t(const AttnArgs& a, cudaStream_t s) {
  using C = Cfg<D>;
  auto k = attn_fwd_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return e;
  k<<<a.grid, kThreads, C::kSmem, s>>>(a.tm_q, a.tm_k, a.tm_v, static_cast<__nv_bfloat16*>(a.out), a.o_bstride,
                                       a.o_tstride, a.lse, a.tile_map, a.B, a.H, a.nq, a.kv_len,
                                       a.scale_log2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t read_watchdog(uint32_t* host8) {
  return cudaMemcpyFromSymbol(host8, ptx::g_dz_watchdog, sizeof(uint32_t) * 8);
}
cudaError_t reset_watchdog() {
  static const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return cudaMemcpyToSymbol(ptx::g_dz_watchdog, zero, sizeof zero);
}

int attention_units(int32_t B, int32_t H, int32_t nq) {
  const int n_qtiles = (nq + BM - 1) / BM;
  return B * H * ((n_qtiles + 1) / 2);
}

cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s) {
  if (a.D == 128) return launch_t<128>(a, s);
  if (a.D == 64) return launch_t<64>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace dz
