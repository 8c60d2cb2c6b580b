// kernels.h -- internal launcher interface between the C-ABI layer (dz.cpp)
// and the sm_100a kernels (*.cu).  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dz {

constexpr int kMaxHeadDim = 128;

// Launch with programmatic stream serialization (PDL): the kernel may start while the previous
// kernel of the stream drains; it calls griddepcontrol.wait before touching global memory.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- K1 / K4: fused per-head RMSNorm + 3D RoPE (+ V copy) -----------------
// One output tensor slot.  Address of output row (b, t, h):
//   base + b*bstride + (h / heads_per_dest)*dstride + t*tstride + (h % heads_per_dest)*D
struct OutSlot {
  void* base = nullptr;
  int64_t bstride = 0, tstride = 0, dstride = 0;
};

// A second token set processed in the same launch (dz_append_attend: the ground-truth chunk's
// append next to the noisy chunk's prologue; one GPU).  Tensors with x[w] == nullptr are absent.
struct PrologueJob {
  const void* x[3] = {nullptr, nullptr, nullptr};
  int64_t x_bstride = 0;
  const int32_t* pos = nullptr;
  OutSlot y[3];
  int32_t n = 0;
};

constexpr int kMaxPeers = 8;  // Ulysses ranks of one node

struct PrologueArgs {
  PrologueJob j1;                                  // optional second token set (j1.n > 0)
  // peer stores (DZ_FLAG_PEER_STORE): output rows of destination rank p go to peer_y[w][p] +
  // b*bstride + t*tstride + (h % heads_per_dest)*D (y[w].dstride unused); null: y[w].base as usual
  void* peer_y[3][kMaxPeers] = {};
  int32_t peer = 0;
  const void* x[3] = {nullptr, nullptr, nullptr};  // raw bf16 q, k, v: [B][n][H][D]
  int64_t x_bstride = 0;                           // elements between batch elements
  const int32_t* pos = nullptr;                    // [n][3] (t, h, w)
  const float* gain[2] = {nullptr, nullptr};       // q, k gains [H*D]
  OutSlot y[3];                                    // q' fp16, k' fp16, v bf16
  int32_t B = 0, n = 0, H = 0, D = 0, heads_per_dest = 0;
  float eps = 1e-6f;
  float q_scale = 1.f;                             // extra factor on Q' (softmax_scale * log2e)
  // FP8 QK (DZ_FLAG_FP8_QK): Q' and K' are stored as E4M3 (1 byte) after multiplying by the
  // power-of-two factors f8_mul[0] (Q') and f8_mul[1] (K'), whose product is 1 (scores unchanged)
  int32_t fp8 = 0;
  float f8_mul[2] = {1.f, 1.f};
  const float2* rope_tab = nullptr;                // [rope_len][D/2] (cos, sin) of p * omega_j, or null
  int32_t rope_len = 0;                            // positions 0 .. rope_len-1 tabulated (others computed)
  double omega[kMaxHeadDim / 2];                   // per pair j: theta^(-2i/d_a), fp64 (host)
  int8_t axis[kMaxHeadDim / 2];                    // per pair j: 0 t, 1 h, 2 w
};
cudaError_t launch_prologue(const PrologueArgs& a, cudaStream_t s);
// RoPE table: tab[p][j] = (cos, sin)(p * omega_j) for p < len, fp64 sincos rounded to fp32
// (the same values the prologue would compute per token)
constexpr int kRopeLen = 4096;
cudaError_t launch_rope_table(float2* tab, int32_t len, const PrologueArgs& a, cudaStream_t s);

// ---- K2: block-causal flash attention (tcgen05 + TMEM + TMA) --------------
// Fig. 10 visibility in span form (R3).  Queries are
// the nq new tokens, split into n spans [start[i], start[i+1]); keys are the
// `valid` committed tokens (visible to every query: every span id exceeds the
// last committed id) followed by the same nq new tokens.  A query of span qs
// sees a new key of span ks iff qs == ks (own span, bidirectional) or
// kc[ks] < qth[qs] (kc: the key span's chunk id if CLEAN, else INT32_MAX; qth:
// the query span's chunk id if NOISY, chunk id + 1 if CLEAN).
constexpr int kMaxSpans = 64;
struct SpanTable {
  int32_t n = 1;
  int32_t valid = 0;
  int32_t start[kMaxSpans + 1] = {};
  int32_t kc[kMaxSpans] = {};
  int32_t qth[kMaxSpans] = {};
};

// K2 epilogue stores to the owners of the query rows (DZ_FLAG_PEER_STORE): rows [p*n_loc, (p+1)*n_loc)
// of this rank's head shard go to rank p's receive buffer through m[p], dims (D, H/N, n_loc, B).
struct PeerMaps {
  CUtensorMap m[kMaxPeers];
  int32_t n = 0;       // 0: O goes to tm_o
  int32_t n_loc = 0;
};

struct AttnArgs {
  SpanTable spans;
  PeerMaps pm;
  int32_t fp8 = 0;  // 1: Q' and K' are E4M3 (QK^T by tcgen05.mma kind::f8f6f4)
  CUtensorMap tm_q;   // Q' fp16, dims (D, H, nq, B), box (64, 1, 128, 1), SW128
  CUtensorMap tm_k;   // K' fp16 cache, dims (D, H, kv_len, B)
  CUtensorMap tm_v;   // V  bf16 cache, dims (D, H, kv_len, B)
  CUtensorMap tm_k2;  // K' of the new tokens in the current-chunk buffer, dims (D, H, nq, B) (see cur_step)
  CUtensorMap tm_v2;  // V of the new tokens straight from the caller's input, dims (D, H, nq, B) (see cur_step)
  CUtensorMap tm_o;   // O  bf16 output, dims (D, H, nq, B), box (64, 1, 32, 1), SW128 (epilogue TMA stores)
  void* out = nullptr;            // bf16, row (b, s, h) at out + b*o_bstride + s*o_tstride + h*D
  int64_t o_bstride = 0, o_tstride = 0;
  float* lse = nullptr;           // optional fp32 [B][H][nq] natural-log LSE
  uint8_t* tile_map = nullptr;    // optional debug [n_groups][n_steps] (256 x 256 tiles) for (b, h) = (0, 0)
  int32_t B = 0, H = 0, D = 0, nq = 0, kv_len = 0;
  float scale_log2 = 0.f;         // unused by the kernel: Q' is pre-scaled by softmax_scale * log2(e)
  float m_static = 0.f;           // > 0: fixed softmax base (log2 units) bounding every logit; 0: online max
  int32_t debug_flags = 0;        // diagnostics only (DZ_DEBUG_KERNEL env): 1 no K/V TMA (results are garbage)
  int32_t grid = 0;               // persistent CTAs (<= #SMs)
  float* ws = nullptr;            // stream-K piece workspace: [2 * pairs][2 ranks][(D + 2) * 128] fp32 (nullptr: no split)
  int32_t* ws_cnt = nullptr;      // per (unit, rank) piece counters, zero between launches
  int32_t cur_step = 0x7fffffff;  // key steps >= cur_step read K'/V from tm_k2/tm_v2 (row (j - cur_step) * step)
};
cudaError_t launch_attention(const AttnArgs& a, cudaStream_t s);
constexpr int kMaxPairs = 80;  // CTA pairs of the persistent grid (B200: 74)
int attention_units(int32_t B, int32_t H, int32_t nq);
constexpr int kTileQ = 256;  // skip / mask decision granularity: query rows of a CTA pair x the keys of a step
// stream-K balances cost-weighted steps: a step of a full 256-row unit weighs kStepWeight, a step of a
// half unit (a last query group of <= 128 rows, run as M = 128 pair MMAs) less (attention.cu)
constexpr int kStepWeight = 8;
// keys per K2 step: 128 with the fixed softmax base (ping-pong kernel), 256 with the online base
int attention_step_keys(float m_static);
// span layouts (several spans): the kernel's step-class table holds at most kMaxStepTiles
// (256-row query group, key step) tiles when attention_has_step_table(D, m_static)
constexpr int kMaxStepTiles = 65536;
bool attention_has_step_table(int32_t D, float m_static);
cudaError_t k2_clock(uint64_t* host2, int reset);  // {SM cycles, globaltimer ns} summed over K2 CTAs
cudaError_t read_watchdog(uint32_t* host8);   // {fired, block, warp, bar addr, parity, smid, bars base, 0}
cudaError_t reset_watchdog();
cudaError_t trace_control(int enable, uint32_t* host, size_t n);  // K2 cycle trace (CTA 0, first unit)  // work units (b, h, q-tile pair)

// ---- NEXT-1 backward (backward.cu): gradients of the teacher-forced path, one GPU, empty cache ----
struct BwdArgs {
  CUtensorMap tm_k, tm_v, tm_q, tm_do;  // K' fp16, V bf16 (box (64, 1, 128, 1)); Q' fp16 (pre-scaled), dO bf16 (64 rows)
  CUtensorMap tm_dq;                    // dL/dq' fp32 [B][n][H][D], box (128, 1, 64, 1), no swizzle (TMA reduce-add)
  const void* dout = nullptr;           // bf16 [B][n][H][D]
  const void* out = nullptr;            // bf16 [B][n][H][D], the forward's output
  const float* lse = nullptr;           // fp32 [B][H][n], the forward's natural-log LSE
  float* delta = nullptr;               // workspace fp32 [B][H][n]
  float* lse2 = nullptr;                // workspace fp32 [B][H][n]
  float* dq_acc = nullptr;              // workspace fp32 [B][n][H][D] (zeroed by the caller): dL/dq'
  float* dk = nullptr;                  // workspace fp32 [B][n][H][D]: dL/dk'
  void* dv = nullptr;                   // bf16 [B][n][H][D] out
  const void* q_raw = nullptr;
  const void* k_raw = nullptr;
  void* dq = nullptr;                   // bf16 [B][n][H][D] out
  void* dk_raw = nullptr;               // bf16 [B][n][H][D] out
  const float* gain[2] = {nullptr, nullptr};
  float* dgain[2] = {nullptr, nullptr};  // fp32 [H][D] out (zeroed by the caller)
  const int32_t* pos = nullptr;
  const float2* tab = nullptr;
  int32_t tab_len = 0;
  float eps = 1e-6f;
  int32_t B = 0, n = 0, H = 0, D = 0;
  int32_t n_pad = 0;                    // row length of delta / lse2 (n rounded up to 64)
  float scale_q = 1.f;                  // dq' = scale_q * (dS K')
  float scale_k = 1.f;                  // dk' = scale_k * (dS^T Q'), Q' pre-scaled by scale * log2e
  SpanTable spans;
  double omega[kMaxHeadDim / 2];
  int8_t axis[kMaxHeadDim / 2];
};
cudaError_t launch_attention_backward(const BwdArgs& a, cudaStream_t s);

// ---- K5: Ulysses receive unpack [N][B][n_loc][Hl][D] -> [B][n_loc][H][D] ---
cudaError_t launch_sp_unpack(const void* recv, void* out, int32_t N, int32_t B, int32_t n_loc, int32_t Hl,
                             int32_t D, cudaStream_t s);

// ---- benchmark helper: invalidate a buffer's L2 lines without write-back (l2.cu) ---
cudaError_t launch_l2_discard(void* p, size_t bytes, cudaStream_t s);

}  // namespace dz
