// dz.cpp -- the C ABI (include/dz.h): validation, cache bookkeeping, tensor
// maps, Ulysses exchange plan and NCCL calls, kernel launches.
//
// Cache bookkeeping follows Alg. 2 of PAPER.md (l.558-607): committed clean
// chunks occupy slots [start, start + valid) of a token-major buffer; the
// chunk being denoised is staged right after them so that one contiguous KV
// range [start, start + valid + n) is what the attention kernel reads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <cstdlib>
#include <deque>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/dz.h"
#include "kernels.h"

namespace {

constexpr size_t kAlign = 256;
std::atomic<int64_t> g_launches{0};  // kernels this library enqueued (dz_kernel_launches)
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Layout {  // byte offsets inside the caller's storage
  int64_t slots = 0;
  size_t k_off = 0, v_off = 0, q_off = 0, kc_off = 0, lse_off = 0, sq_off = 0, sk_off = 0, sv_off = 0, ol_off = 0,
         or_off = 0, map_off = 0, ws_off = 0, cnt_off = 0, cnt_bytes = 0, rope_off = 0, bar_off = 0, bq_off = 0,
         bk_off = 0, bd_off = 0, bl_off = 0, total = 0;
};

bool basic_cfg_ok(const dz_config* c) {
  if (!c) return false;
  if (c->batch <= 0 || c->heads <= 0) return false;
  if (c->head_dim != 64 && c->head_dim != 128) return false;
  if (c->world_size <= 0 || c->rank < 0 || c->rank >= c->world_size) return false;
  if (c->heads % c->world_size) return false;
  if (c->max_chunk_tokens <= 0 || c->max_chunk_tokens % c->world_size) return false;
  if (c->cache_capacity_tokens < 0 || c->window_slack_tokens < 0) return false;
  int s = 0;
  for (int a = 0; a < 3; ++a) {
    if (c->rope_dims[a] < 0 || c->rope_dims[a] % 2) return false;
    s += c->rope_dims[a];
  }
  return s == c->head_dim;
}

// debug tile map: [query groups of kTileQ rows][key steps] (sized for the smallest step, 128 keys)
size_t map_bytes(const dz_config* c) {
  const int64_t mc = c->max_chunk_tokens;
  const int64_t keys = c->cache_capacity_tokens + mc + c->window_slack_tokens;
  return 256 + (size_t)((mc + dz::kTileQ - 1) / dz::kTileQ) * ((keys + 127) / 128);
}

Layout make_layout(const dz_config* c) {
  Layout L;
  const int64_t B = c->batch, Hl = c->heads / c->world_size, D = c->head_dim, N = c->world_size;
  const int64_t mc = c->max_chunk_tokens;
  L.slots = c->cache_capacity_tokens + mc + c->window_slack_tokens;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += align_up(bytes);
    return o;
  };
  L.k_off = take((size_t)B * L.slots * Hl * D * 2);
  L.v_off = take((size_t)B * L.slots * Hl * D * 2);
  L.q_off = take((size_t)B * mc * Hl * D * 2);                       // Q' fp16
  L.kc_off = take(N == 1 ? (size_t)B * mc * Hl * D * 2 : 0);         // K' fp16 of a noisy chunk (not staged)
  L.lse_off = take((c->flags & DZ_FLAG_WRITE_LSE) ? (size_t)B * Hl * mc * 4 : 0);
  L.map_off = take((c->flags & DZ_FLAG_TILE_MAP) ? map_bytes(c) : 0);
  // K2 stream-K workspace: per pair a head and a tail piece, per CTA rank (D + 2) x 128 fp32
  L.ws_off = take((size_t)2 * dz::kMaxPairs * 2 * (D + 2) * 128 * 4);
  L.cnt_bytes = (size_t)B * Hl * ((mc + dz::kTileQ - 1) / dz::kTileQ) * 2 * 4;
  L.cnt_off = take(L.cnt_bytes);
  L.rope_off = take((size_t)dz::kRopeLen * (D / 2) * 8);             // RoPE (cos, sin) table, fp32
  if (c->flags & DZ_FLAG_BACKWARD) {                                  // NEXT-1 backward workspace
    L.bq_off = take((size_t)B * mc * Hl * D * 4);                     // dL/dq' fp32 (atomic accumulation)
    L.bk_off = take((size_t)B * mc * Hl * D * 4);                     // dL/dk' fp32
    L.bd_off = take((size_t)B * Hl * ((mc + 63) / 64 * 64) * 4);      // delta = <dO, O> (rows padded to 64)
    L.bl_off = take((size_t)B * Hl * ((mc + 63) / 64 * 64) * 4);      // lse * log2(e)
  }
  if (N > 1) {
    const size_t sb = (size_t)B * (mc / N) * c->heads * D * 2;       // [N][B][n_loc][Hl][D]
    L.sq_off = take(sb);
    L.sk_off = take(sb);
    L.sv_off = take(sb);
    L.ol_off = take((size_t)B * mc * Hl * D * 2);                    // O local [B][n][Hl][D]
    L.or_off = take(sb);                                              // O recv [N][B][n_loc][Hl][D]
    L.bar_off = take(256);                                            // barrier scratch (peer stores)
  }
  L.total = off;
  return L;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 4D token-major tensor [B][tokens][H][D] (16-bit elements) as TMA dims (D, H, tokens, B),
// box (box_d, 1, box_t, 1); swizzle = box_d * 2 bytes (128 or 64); out-of-bounds elements read as zero.
// dt: 0 fp16, 1 bf16 (2-byte elements), 2 E4M3 as uint8 (1-byte elements)
bool make_tmap(CUtensorMap* m, const void* base, int dt, int64_t D, int64_t H, int64_t tokens, int64_t B,
               int64_t batch_stride_elems, uint32_t box_d, uint32_t box_t) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int64_t es = dt == 2 ? 1 : 2;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)tokens, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)(D * es), (cuuint64_t)(H * D * es), (cuuint64_t)(batch_stride_elems * es)};
  cuuint32_t box[4] = {box_d, 1, box_t, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle sw = box_d * es == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const CUtensorMapDataType ty = dt == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : dt == 1 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUresult r = fn(m, ty, 4,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

struct dz_ctx {
  dz_config cfg{};
  Layout L;
  int B = 0, H = 0, Hl = 0, D = 0, N = 1, rank = 0;
  float theta = 1e4f, eps = 1e-6f, scale = 0.f;
  float m_static = 0.f;  // QK-norm logit bound used as a fixed softmax base (0: online max)
  int num_sms = 148;
  // committed state
  int64_t start = 0, valid = 0;
  std::deque<std::pair<int32_t, int64_t>> chunks;  // (id, tokens)
  int32_t last_id = -1;
  // staged chunk (written by the last attend)
  bool staged = false;
  // the last attention read the new tokens' K'/V from the staging slots after the committed ones
  // (they are only staged there when the chunk may be committed, under SP, or unaligned)
  bool staging_read = false;
  int32_t staged_id = 0, staged_kind = 0;
  int64_t staged_n = 0;
  // last attend geometry (tile map / lse)
  int32_t last_nq = 0, last_nkv_tiles = 0, last_nq_tiles = 0, last_step_keys = 256;
  bool have_map = false;
  // device pointers into the caller's storage
  char* base = nullptr;
  dz::PrologueArgs pro;  // RoPE frequencies, axes, gains
  ncclComm_t comm = nullptr;
  bool poisoned = false;
  bool ws_zeroed = false;  // stream-K piece counters initialised
  bool rope_ready = false;  // RoPE table written (first prologue)
  // DZ_FLAG_PROFILE: events e[0..4] around the attend phases, a[0..1] around the append
  cudaEvent_t ev[5] = {}, ev_app[2] = {};
  bool have_attend_ev = false, have_append_ev = false;
  bool prof_on = true;  // dz_profile_enable: events are recorded only while on
  bool external_x = false;  // DZ_FLAG_EXTERNAL_EXCHANGE: the caller runs the all-to-all transfers
  bool host_only = false;   // DZ_FLAG_HOST_ONLY: planning context, never touches the device
  bool peer_mode = false;   // DZ_FLAG_PEER_STORE: stores into the peers' storages instead of exchanges
  bool peers_set = false;
  char* peers[dz::kMaxPeers] = {};  // every rank's cache_storage base (dz_sp_set_peers)
  float max_gain = 0.f;     // max |g| over q_gain and k_gain (read from the device at create)
  // An operation suspended at an exchange point (DZ_FLAG_EXTERNAL_EXCHANGE): the caller runs
  // `plan` (dz_sp_pending), then dz_sp_resume enqueues the rest.
  struct Pending {
    int op = 0;          // 0 none, 1 attend, 2 append
    int phase = -1;      // exchange phase of `plan` (0 attend pre, 1 append pre, 2 attend post)
    int64_t n = 0;
    dz::SpanTable spans;
    void* out = nullptr;
    bool prof = false;
    bool stage_chunk = false;  // attend_chunk: record the staged chunk when the call completes
    int32_t chunk_id = 0, kind = 0;
    std::vector<dz_xfer> plan;
  } pend;
  std::string err;

  bool f8 = false;          // DZ_FLAG_FP8_QK: Q' and K' (cache and current chunk) are E4M3
  float f8_mul[2] = {1.f, 1.f};  // power-of-two factors on Q' and K' (product 1)
  int64_t krow() const { return (int64_t)Hl * D * (f8 ? 1 : 2); }  // bytes of one slot of K'
  void* kslot(int b, int64_t slot) const {
    return base + L.k_off + ((size_t)b * L.slots + slot) * krow();
  }
  void* vslot(int b, int64_t slot) const {
    return base + L.v_off + ((size_t)b * L.slots + slot) * Hl * D * 2;
  }
};

namespace {

dz_status fail(dz_ctx* c, dz_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
    if (s == DZ_ECUDA || s == DZ_ENCCL) c->poisoned = true;
  }
  return s;
}

dz_status cuda_check(dz_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DZ_OK;
  return fail(c, DZ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

dz_status nccl_check(dz_ctx* c, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return DZ_OK;
  return fail(c, DZ_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Ulysses exchange plan: per (tensor, peer p, batch element b),
// the block this rank sends to p and where the block it receives from p lands,
// as byte offsets into the caller's storage.  One source of truth for the NCCL
// calls below and for dz_sp_plan (host-side tests of the plan).
//   phase 0 (attend) / 1 (append): seq shard [n_loc, H] -> head shard [n, Hl] for
//     Q' (phase 0 only), K', V; the send layout is [N][B][n_loc][Hl][D] (written by
//     K1), Q' lands in the Q' scratch [B][n][Hl][D], K'/V in the cache staging slots
//     [start + valid + p * n_loc, ...) of batch element b;
//   phase 2 (post): O head shard [B][n][Hl][D] -> the receive buffer [N][B][n_loc][Hl][D]
//     (K5 then unpacks it to [B][n_loc][H][D]).
std::vector<dz_xfer> make_plan(const dz_ctx* c, int phase, int64_t n) {
  std::vector<dz_xfer> v;
  const int64_t n_loc = n / c->N;
  const int64_t row = (int64_t)c->Hl * c->D * 2;  // one token of one rank's heads
  const int64_t blk = n_loc * row;
  if (phase == 0 || phase == 1) {
    for (int which = phase == 0 ? 0 : 1; which < 3; ++which) {
      const int64_t so = (int64_t)(which == 0 ? c->L.sq_off : which == 1 ? c->L.sk_off : c->L.sv_off);
      for (int p = 0; p < c->N; ++p)
        for (int b = 0; b < c->B; ++b) {
          dz_xfer x;
          x.peer = p;
          x.tensor = which;
          x.bytes = blk;
          x.send_off = so + ((int64_t)p * c->B + b) * blk;
          const int64_t slot = c->start + c->valid + (int64_t)p * n_loc;
          if (which == 0)
            x.recv_off = (int64_t)c->L.q_off + ((int64_t)b * n + (int64_t)p * n_loc) * row;
          else
            x.recv_off = (int64_t)(which == 1 ? c->L.k_off : c->L.v_off) + ((int64_t)b * c->L.slots + slot) * row;
          v.push_back(x);
        }
    }
  } else {
    for (int p = 0; p < c->N; ++p)
      for (int b = 0; b < c->B; ++b) {
        dz_xfer x;
        x.peer = p;
        x.tensor = 3;
        x.bytes = blk;
        x.send_off = (int64_t)c->L.ol_off + ((int64_t)b * n + (int64_t)p * n_loc) * row;
        x.recv_off = (int64_t)c->L.or_off + ((int64_t)p * c->B + b) * blk;
        v.push_back(x);
      }
  }
  return v;
}

dz_status check_ready(dz_ctx* c) {
  if (!c) return DZ_EINVAL;
  if (c->poisoned) return fail(c, DZ_ESTATE, "context poisoned by an earlier CUDA/NCCL error: %s", c->err.c_str());
  if (c->pend.op != 0)
    return fail(c, DZ_ESTATE, "exchange phase %d pending: run dz_sp_pending's transfers, then dz_sp_resume",
                c->pend.phase);
  return DZ_OK;
}

// a planning context (DZ_FLAG_HOST_ONLY) validates a compute call, then refuses to enqueue it
dz_status check_device(dz_ctx* c) {
  if (c->host_only) return fail(c, DZ_ESTATE, "host-only (planning) context: nothing is enqueued");
  if (c->peer_mode && !c->peers_set) return fail(c, DZ_ESTATE, "DZ_FLAG_PEER_STORE: dz_sp_set_peers first");
  return DZ_OK;
}

dz_status check_span(dz_ctx* c, const dz_span* s) {
  if (!s || !s->pos_thw) return fail(c, DZ_EINVAL, "null span or positions");
  if (s->kind != DZ_CLEAN && s->kind != DZ_NOISY) return fail(c, DZ_EINVAL, "bad span kind %d", s->kind);
  if (s->n_tokens <= 0 || s->n_tokens % c->N) return fail(c, DZ_ESHAPE, "n_tokens %d not a positive multiple of world_size %d", s->n_tokens, c->N);
  if (c->peer_mode && (s->n_tokens / c->N) % 8)
    return fail(c, DZ_ESHAPE, "DZ_FLAG_PEER_STORE: n_tokens / world_size = %d is not a multiple of 8", s->n_tokens / c->N);
  if (s->n_tokens > c->cfg.max_chunk_tokens)
    return fail(c, DZ_ECAPACITY, "chunk of %d tokens exceeds max_chunk_tokens %d", s->n_tokens, c->cfg.max_chunk_tokens);
  if (s->chunk_id <= c->last_id)
    return fail(c, DZ_ESTATE, "chunk id %d must exceed the last committed id %d", s->chunk_id, c->last_id);
  return DZ_OK;
}

// Keep [start, start + valid + max_chunk) inside the slot range: compact the
// committed window down to slot 0 when it would run past the end.
dz_status ensure_staging_room(dz_ctx* c, cudaStream_t st, int64_t extra = 0) {
  if (c->start + c->valid + extra + c->cfg.max_chunk_tokens <= c->L.slots) return DZ_OK;
  if (c->host_only) {  // a planning context holds no data: bookkeeping only
    c->start = 0;
    return DZ_OK;
  }
  const int64_t s0 = c->start;
  for (int b = 0; b < c->B; ++b) {
    for (int kv = 0; kv < 2; ++kv) {
      // forward copy in pieces of s0 slots: each piece's source lies above its destination
      for (int64_t done = 0; done < c->valid; done += s0) {
        const int64_t len = std::min<int64_t>(s0, c->valid - done);
        void* dst = kv == 0 ? c->kslot(b, done) : c->vslot(b, done);
        const void* src = kv == 0 ? c->kslot(b, s0 + done) : c->vslot(b, s0 + done);
        const size_t row = kv == 0 ? (size_t)c->krow() : (size_t)c->Hl * c->D * 2;
        dz_status r = cuda_check(c, cudaMemcpyAsync(dst, src, len * row, cudaMemcpyDeviceToDevice, st), "compact");
        if (r) return r;
      }
    }
  }
  c->start = 0;
  return DZ_OK;
}

void fill_prologue_common(dz_ctx* c, dz::PrologueArgs& a, const int32_t* pos, int64_t n_loc) {
  a = c->pro;
  a.B = c->B;
  a.n = (int32_t)n_loc;
  a.H = c->H;
  a.D = c->D;
  a.x_bstride = n_loc * c->H * c->D;
  a.pos = pos;
}

// K1 prologue for the current chunk: Q' and the chunk's K'/V, written either
// straight into the staging slot (N == 1) or into the all-to-all send layout.
// A ground-truth chunk appended in the same prologue launch as an attend (dz_append_attend, one GPU):
// its K'/V go to slots [valid, valid + n) and the attended chunk's staging slots follow them.
struct AppendJob {
  const void* k = nullptr;
  const void* v = nullptr;
  const int32_t* pos = nullptr;
  int64_t n = 0;
};

dz_status run_prologue(dz_ctx* c, const void* q, const void* k, const void* v, const int32_t* pos, int64_t n,
                       cudaStream_t st, bool cur_separate = false, const AppendJob* aj = nullptr) {
  const int64_t n_loc = n / c->N;
  dz::PrologueArgs a;
  fill_prologue_common(c, a, pos, n_loc);
  a.q_scale = c->scale * 1.4426950408889634f;  // scores leave the QK MMA in log2 units
  a.x[0] = q;
  a.x[1] = k;
  a.x[2] = v;
  if (c->N == 1) {
    a.heads_per_dest = c->H;
    a.y[0] = {c->base + c->L.q_off, n * c->H * c->D, (int64_t)c->H * c->D, 0};
    const int64_t slot = c->start + c->valid + (aj ? aj->n : 0);
    if (aj) {  // the ground-truth chunk: K' and V into the slots right after the committed ones
      a.j1.x[1] = aj->k;
      a.j1.x[2] = aj->v;
      a.j1.x_bstride = aj->n * c->H * c->D;
      a.j1.pos = aj->pos;
      a.j1.n = (int32_t)aj->n;
      a.j1.y[1] = {c->kslot(0, c->start + c->valid), c->L.slots * c->H * c->D, (int64_t)c->H * c->D, 0};
      a.j1.y[2] = {c->vslot(0, c->start + c->valid), c->L.slots * c->H * c->D, (int64_t)c->H * c->D, 0};
    }
    if (cur_separate)  // a noisy chunk's K' goes to its own buffer; the committed cache is only read
      a.y[1] = {c->base + c->L.kc_off, n * c->H * c->D, (int64_t)c->H * c->D, 0};
    else
      a.y[1] = {c->kslot(0, slot), c->L.slots * c->H * c->D, (int64_t)c->H * c->D, 0};
    a.y[2] = {c->vslot(0, slot), c->L.slots * c->H * c->D, (int64_t)c->H * c->D, 0};
  } else {
    a.heads_per_dest = c->Hl;
    const int64_t tst = (int64_t)c->Hl * c->D, bst = n_loc * tst, dst = (int64_t)c->B * bst;
    a.y[0] = {c->base + c->L.sq_off, bst, tst, dst};
    a.y[1] = {c->base + c->L.sk_off, bst, tst, dst};
    a.y[2] = {c->base + c->L.sv_off, bst, tst, dst};
    if (c->peer_mode) {
      // straight into rank p's receive locations (the recv_off of dz_sp_plan): Q' scratch rows
      // [rank * n_loc, ...) of [B][n][Hl][D], K'/V staging slots start + valid + rank * n_loc + t
      a.peer = 1;
      const int64_t row = (int64_t)c->Hl * c->D * 2, slot = c->start + c->valid + (int64_t)c->rank * n_loc;
      a.y[0] = {nullptr, n * tst, tst, 0};
      a.y[1] = {nullptr, c->L.slots * tst, tst, 0};
      a.y[2] = {nullptr, c->L.slots * tst, tst, 0};
      for (int p = 0; p < c->N; ++p) {
        a.peer_y[0][p] = c->peers[p] + c->L.q_off + (int64_t)c->rank * n_loc * row;
        a.peer_y[1][p] = c->peers[p] + c->L.k_off + slot * row;
        a.peer_y[2][p] = c->peers[p] + c->L.v_off + slot * row;
      }
    }
  }
  a.rope_tab = reinterpret_cast<const float2*>(c->base + c->L.rope_off);
  a.rope_len = dz::kRopeLen;
  a.fp8 = c->f8 ? 1 : 0;
  a.f8_mul[0] = c->f8_mul[0];
  a.f8_mul[1] = c->f8_mul[1];
  if (!c->rope_ready) {  // first prologue: fill the table; this prologue waits for it before reading
    dz_status r = cuda_check(c, dz::launch_rope_table(reinterpret_cast<float2*>(c->base + c->L.rope_off),
                                                      dz::kRopeLen, a, st), "rope table launch");
    if (r) return r;
    g_launches.fetch_add(1, std::memory_order_relaxed);
    // a fill recorded into a graph being captured has not run yet: fill again on the next eager call
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) c->rope_ready = true;
  }
  dz_status r = cuda_check(c, dz::launch_prologue(a, st), "prologue launch");
  if (!r) g_launches.fetch_add(1, std::memory_order_relaxed);
  return r;
}

// one grouped NCCL send/recv per plan entry (all peers, all tensors) on the caller's stream
dz_status run_exchange(dz_ctx* c, int phase, int64_t n, cudaStream_t st) {
  if (c->peer_mode) {  // peer stores put the data in place: only order the ranks (a 4-byte all-reduce)
    void* flag = c->base + c->L.bar_off;
    return nccl_check(c, ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, c->comm, st), "ncclAllReduce (barrier)");
  }
  const std::vector<dz_xfer> plan = make_plan(c, phase, n);
  dz_status r = nccl_check(c, ncclGroupStart(), "ncclGroupStart");
  if (r) return r;
  for (const dz_xfer& x : plan) {
    r = nccl_check(c, ncclSend(c->base + x.send_off, (size_t)x.bytes, ncclUint8, x.peer, c->comm, st), "ncclSend");
    if (!r) r = nccl_check(c, ncclRecv(c->base + x.recv_off, (size_t)x.bytes, ncclUint8, x.peer, c->comm, st), "ncclRecv");
    if (r) {
      ncclGroupEnd();
      return r;
    }
  }
  return nccl_check(c, ncclGroupEnd(), "ncclGroupEnd");
}
dz_status exchange_pre(dz_ctx* c, bool with_q, int64_t n, cudaStream_t st) { return run_exchange(c, with_q ? 0 : 1, n, st); }
dz_status exchange_post(dz_ctx* c, int64_t n, cudaStream_t st) { return run_exchange(c, 2, n, st); }

// K2 over local heads and the full sequence: committed slots + the staged chunk.
dz_status run_attention(dz_ctx* c, int64_t n, const dz::SpanTable& spans, void* out_local, int64_t o_bstride,
                        int64_t o_tstride, const void* k_new, const void* v_new, cudaStream_t st) {
  dz::AttnArgs a;
  a.spans = spans;
  a.spans.valid = (int32_t)c->valid;
  const int64_t kv_len = c->valid + n;
  const int64_t bs = c->L.slots * c->Hl * c->D;
  // Q: 128-row tiles per CTA; a step is 128 keys (fixed softmax base) or 256 (online base,
  // dz::attention_step_keys): each CTA of a pair loads 64-key boxes of K (half of the step's keys)
  // and D/2 of the columns of all the step's V rows (see attention.cu).
  // FP8 QK: Q' / K' are E4M3 rows of D bytes: one 128-byte SW128 box per row
  const int qk_dt = c->f8 ? 2 : 0;
  const uint32_t qk_box = c->f8 ? (uint32_t)c->D : 64u;
  a.fp8 = c->f8 ? 1 : 0;
  if (!make_tmap(&a.tm_q, c->base + c->L.q_off, qk_dt, c->D, c->Hl, n, c->B, n * c->Hl * c->D, qk_box, 128) ||
      !make_tmap(&a.tm_k, c->kslot(0, c->start), qk_dt, c->D, c->Hl, kv_len, c->B, bs, qk_box, 64) ||
      !make_tmap(&a.tm_v, c->vslot(0, c->start), 1, c->D, c->Hl, kv_len, c->B, bs, (uint32_t)c->D / 2,
                 (uint32_t)dz::attention_step_keys(c->m_static)))
    return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled failed");
  // O rows are token-major with o_tstride == Hl * D (the caller's [B][n][H][D] or the SP local buffer)
  if (o_tstride != (int64_t)c->Hl * c->D ||
      !make_tmap(&a.tm_o, out_local, 1, c->D, c->Hl, n, c->B, o_bstride, (uint32_t)c->D / 2, 32))
    return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled (O) failed");
  if (v_new != nullptr) {  // the new tokens: K' from the current-chunk buffer, V from the caller's input
    const int step_keys = dz::attention_step_keys(c->m_static);
    if (!make_tmap(&a.tm_k2, k_new, qk_dt, c->D, c->Hl, n, c->B, n * c->Hl * c->D, qk_box, 64) ||
        !make_tmap(&a.tm_v2, v_new, 1, c->D, c->Hl, n, c->B, n * c->Hl * c->D, (uint32_t)c->D / 2,
                   (uint32_t)step_keys))
      return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled (new tokens) failed");
    a.cur_step = (int32_t)(c->valid / step_keys);
  }
  if (c->peer_mode && c->N > 1) {  // O rows to their owners' receive buffers ([N][B][n_loc][Hl][D], block `rank`)
    const int64_t n_loc = n / c->N, blk = (int64_t)c->B * n_loc * c->Hl * c->D * 2;
    a.pm.n = c->N;
    a.pm.n_loc = (int32_t)n_loc;
    for (int p = 0; p < c->N; ++p)
      if (!make_tmap(&a.pm.m[p], c->peers[p] + c->L.or_off + (int64_t)c->rank * blk, 1, c->D, c->Hl, n_loc, c->B,
                     n_loc * c->Hl * c->D, (uint32_t)c->D / 2, 8))
        return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled (peer O) failed");
  }
  a.out = out_local;
  a.o_bstride = o_bstride;
  a.o_tstride = o_tstride;
  a.lse = (c->cfg.flags & DZ_FLAG_WRITE_LSE) ? reinterpret_cast<float*>(c->base + c->L.lse_off) : nullptr;
  a.B = c->B;
  a.H = c->Hl;
  a.D = c->D;
  a.nq = (int32_t)n;
  a.kv_len = (int32_t)kv_len;
  a.scale_log2 = c->scale * 1.4426950408889634f;
  a.m_static = c->m_static;
  if (const char* e = getenv("DZ_DEBUG_KERNEL")) a.debug_flags = atoi(e);  // diagnostics: results are garbage
  // persistent grid: one CTA pair per TPC; stream-K spreads the executed steps evenly over the pairs
  a.grid = 2 * std::min(c->num_sms / 2, dz::kMaxPairs);
  // stream-K needs <= 64 query groups and 32-bit step arithmetic (W * pairs < 2^31); else whole units round-robin
  const int step_keys = dz::attention_step_keys(c->m_static);
  const int64_t n_groups = (n + dz::kTileQ - 1) / dz::kTileQ, n_steps = (kv_len + step_keys - 1) / step_keys;
  // DZ_FLAG_WHOLE_UNITS: every unit computed whole by one CTA pair, so a unit's result depends only on
  // its rows and keys, not on the unit count (the same bits at every world size, reading A21)
  static const bool rr_forced = getenv("DZ_SCHED_RR") != nullptr;  // diagnostics: whole units round-robin
  const bool streamk = !rr_forced && !(c->cfg.flags & DZ_FLAG_WHOLE_UNITS) && n_groups <= 64 &&
                       (int64_t)c->B * c->Hl * n_groups * n_steps * dz::kMaxPairs * dz::kStepWeight < (1ll << 31);
  a.ws = streamk ? reinterpret_cast<float*>(c->base + c->L.ws_off) : nullptr;
  a.ws_cnt = reinterpret_cast<int32_t*>(c->base + c->L.cnt_off);
  if (!c->ws_zeroed) {  // piece counters start at zero; every combine resets its own
    dz_status r = cuda_check(c, cudaMemsetAsync(a.ws_cnt, 0, c->L.cnt_bytes, st),
                             "counter init");
    if (r) return r;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;  // (a captured clear runs at replay only)
    if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) c->ws_zeroed = true;
  }
  const int ngr = (int)n_groups, nst = (int)n_steps;
  if ((c->cfg.flags & DZ_FLAG_TILE_MAP) && (size_t)ngr * nst <= map_bytes(&c->cfg)) {
    a.tile_map = reinterpret_cast<uint8_t*>(c->base + c->L.map_off);
    // the kernel writes the executed steps (FULL / PARTIAL); the rest stay SKIP
    dz_status r = cuda_check(c, cudaMemsetAsync(a.tile_map, 0, (size_t)ngr * nst, st), "tile map clear");
    if (r) return r;
    c->last_nq_tiles = ngr;
    c->last_step_keys = step_keys;
    c->last_nkv_tiles = nst;
    c->have_map = true;
  }
  c->last_nq = (int32_t)n;
  dz_status r = cuda_check(c, dz::launch_attention(a, st), "attention launch");
  if (!r) g_launches.fetch_add(1, std::memory_order_relaxed);
  return r;
}

}  // namespace

extern "C" {

size_t dz_cache_bytes(const dz_config* cfg) {
  if (!basic_cfg_ok(cfg)) return 0;
  return make_layout(cfg).total;
}

dz_status dz_create(const dz_config* cfg, dz_ctx** out) {
  if (!out) return DZ_EINVAL;
  *out = nullptr;
  if (!cfg) return DZ_EINVAL;
  if (cfg->head_dim != 64 && cfg->head_dim != 128) return DZ_ESHAPE;
  if (!basic_cfg_ok(cfg)) return DZ_ESHAPE;
  if (!cfg->q_gain || !cfg->k_gain || !cfg->cache_storage) return DZ_EINVAL;
  if ((reinterpret_cast<uintptr_t>(cfg->cache_storage) & (kAlign - 1)) || !aligned16(cfg->q_gain) ||
      !aligned16(cfg->k_gain))
    return DZ_EINVAL;
  const bool host_only = (cfg->flags & DZ_FLAG_HOST_ONLY) != 0;
  const bool external_x = (cfg->flags & DZ_FLAG_EXTERNAL_EXCHANGE) != 0;
  if (cfg->world_size > 1 && !cfg->nccl_comm && !external_x) return DZ_EINVAL;  // SP needs a transport
  // max |g| from the gains themselves (one synchronous read; create is never captured): it sets the
  // fp16 range check and the fixed softmax base below, so it is not taken on the caller's word.
  // A caller bound (max_abs_gain > 0) below the true maximum is rejected.
  double gmax = 0.0;
  if (host_only) {
    gmax = cfg->max_abs_gain;  // a planning context never reads device memory
  } else {
    const size_t ne = (size_t)cfg->heads * cfg->head_dim;
    std::vector<float> h(2 * ne);
    if (cudaMemcpy(h.data(), cfg->q_gain, ne * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(h.data() + ne, cfg->k_gain, ne * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();  // (an invalid pointer is not a sticky error)
      return DZ_EINVAL;
    }
    for (float g : h) {
      if (!std::isfinite(g)) return DZ_ERANGE;
      gmax = std::max(gmax, (double)std::fabs(g));
    }
    if (cfg->max_abs_gain > 0.f && (double)cfg->max_abs_gain < gmax) return DZ_ERANGE;  // under-reported bound
  }
  // fp16 Q'/K' (reading A13): |x'_i| <= sqrt(D) * |g_i| after RMSNorm
  if (!(gmax > 0.0) || std::sqrt((double)cfg->head_dim) * gmax >= 6.0e4) return DZ_ERANGE;
  Layout L = make_layout(cfg);
  if (cfg->cache_bytes < L.total) return DZ_ECAPACITY;

  if (cfg->flags & DZ_FLAG_FP8_QK) {  // E4M3 QK: one GPU, D = 128, the token-loop prologue
    if (cfg->head_dim != 128 || cfg->world_size != 1 || cfg->heads > 48) return DZ_ESHAPE;
  }
  if (cfg->flags & DZ_FLAG_PEER_STORE) {  // one node, the token-loop prologue (H within one pass of it);
    // the epilogue's 8-row O boxes need owner boundaries (n / world_size) on multiples of 8
    if (cfg->world_size < 2 || cfg->world_size > dz::kMaxPeers || cfg->heads > 3 * (256 / (cfg->head_dim / 8)) ||
        (cfg->max_chunk_tokens / cfg->world_size) % 8)
      return DZ_ESHAPE;
  }
  dz_ctx* c = new (std::nothrow) dz_ctx();
  if (!c) return DZ_ECUDA;
  c->cfg = *cfg;
  c->L = L;
  c->B = cfg->batch;
  c->H = cfg->heads;
  c->N = cfg->world_size;
  c->rank = cfg->rank;
  c->Hl = cfg->heads / cfg->world_size;
  c->D = cfg->head_dim;
  c->theta = cfg->rope_theta > 0.f ? cfg->rope_theta : 1e4f;
  c->eps = cfg->rms_eps > 0.f ? cfg->rms_eps : 1e-6f;
  c->scale = cfg->softmax_scale > 0.f ? cfg->softmax_scale : 1.0f / std::sqrt((float)cfg->head_dim);
  c->base = static_cast<char*>(cfg->cache_storage);
  c->comm = static_cast<ncclComm_t>(cfg->nccl_comm);
  c->external_x = external_x;
  c->peer_mode = (cfg->flags & DZ_FLAG_PEER_STORE) != 0;
  c->host_only = host_only;
  c->max_gain = (float)gmax;
  int dev = 0;
  if (!host_only && cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  // RoPE frequencies per pair j (fp64): axis slice [t | h | w], omega = theta^(-2i/d_a)
  int j = 0;
  for (int ax = 0; ax < 3; ++ax)
    for (int i = 0; i < cfg->rope_dims[ax] / 2; ++i, ++j) {
      c->pro.omega[j] = std::pow((double)c->theta, -2.0 * i / cfg->rope_dims[ax]);
      c->pro.axis[j] = (int8_t)ax;
    }
  c->pro.gain[0] = cfg->q_gain;
  c->pro.gain[1] = cfg->k_gain;
  c->pro.eps = c->eps;
  // RMSNorm gives ||q'|| <= sqrt(D) max|g|, ||k'|| <= sqrt(D) max|g| (RoPE keeps norms), so
  // |score| * log2e <= D * max|g|^2 * scale * log2e (+0.5% for the fp16 rounding of Q'/K').
  // When that bound is <= 60 the kernel uses base 0 instead of a running row max: every
  // p = 2^s lies in [2^-60, 2^60], normal in fp32 and bf16, and no running max is needed.
  {
    const double bound = (double)cfg->head_dim * gmax * gmax * c->scale * 1.4426950408889634 * 1.005;
    c->m_static = (!(cfg->flags & DZ_FLAG_ONLINE_SOFTMAX) && bound <= 60.0) ? (float)std::max(bound, 1.0) : 0.f;  // > 0 selects the fixed base
  }
  if (cfg->flags & DZ_FLAG_FP8_QK) {
    // the fixed softmax base is required (scores stay in [-60, 60] log2 units); Q' * 2^a and
    // K' * 2^-a as E4M3 with a balancing their bounds (|q'| <= sqrt(D) G scale log2e, |k'| <= sqrt(D) G),
    // both far inside E4M3's +-448, so the MMA's scores need no descale
    if (c->m_static <= 0.f) {
      delete c;
      return DZ_ERANGE;
    }
    const double bq = std::sqrt((double)cfg->head_dim) * gmax * c->scale * 1.4426950408889634;
    const double bk = std::sqrt((double)cfg->head_dim) * gmax;
    const int e = (int)std::lround(0.5 * std::log2(bk / bq));
    c->f8 = true;
    c->f8_mul[0] = std::ldexp(1.f, e);
    c->f8_mul[1] = std::ldexp(1.f, -e);
    if (bq * c->f8_mul[0] > 448.0 || bk * c->f8_mul[1] > 448.0) {
      delete c;
      return DZ_ERANGE;
    }
  }
  if ((cfg->flags & DZ_FLAG_PROFILE) && !host_only) {
    for (auto& e : c->ev)
      if (cudaEventCreate(&e) != cudaSuccess) e = nullptr;
    for (auto& e : c->ev_app)
      if (cudaEventCreate(&e) != cudaSuccess) e = nullptr;
  }
  *out = c;
  return DZ_OK;
}

}  // extern "C"

namespace {

// The append's commit (bookkeeping) once its K'/V are in the slots.
dz_status append_commit(dz_ctx* c, int32_t chunk_id, int64_t n, bool prof, cudaStream_t st) {
  if (prof) cudaEventRecord(c->ev_app[1], st);
  c->have_append_ev = prof;
  c->valid += n;
  c->chunks.emplace_back(chunk_id, n);
  c->last_id = chunk_id;
  c->staged = false;
  return ensure_staging_room(c, st);
}

// Suspend the current operation at an exchange point: the caller runs `phase`'s plan, then
// dz_sp_resume continues (DZ_FLAG_EXTERNAL_EXCHANGE).
void suspend(dz_ctx* c, int op, int phase, int64_t n) {
  c->pend.op = op;
  c->pend.phase = phase;
  c->pend.n = n;
  // peer stores: the data is already in place; the caller only orders the ranks (a barrier)
  if (c->peer_mode) c->pend.plan.clear(); else c->pend.plan = make_plan(c, phase, n);
}

}  // namespace

extern "C" {

dz_status dz_append_kv(dz_ctx* c, const void* k_raw, const void* v_raw, const dz_span* s, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if (!k_raw || !v_raw || !aligned16(k_raw) || !aligned16(v_raw)) return fail(c, DZ_EINVAL, "null/misaligned k or v");
  if ((r = check_span(c, s))) return r;
  if (s->kind != DZ_CLEAN) return fail(c, DZ_ESTATE, "only clean chunks enter the cache (Alg. 2 l.603)");
  if (c->valid + s->n_tokens > c->cfg.cache_capacity_tokens)
    return fail(c, DZ_ECAPACITY, "cache full: %lld + %d > %lld", (long long)c->valid, s->n_tokens,
                (long long)c->cfg.cache_capacity_tokens);
  if ((r = check_device(c))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool prof = c->ev_app[0] != nullptr && c->prof_on;
  if (prof) cudaEventRecord(c->ev_app[0], st);
  // K4 waits for its predecessor on the stream before it reads k_raw / v_raw / positions (that
  // predecessor may be the kernel that produced them); it may still be scheduled early (PDL).
  if ((r = run_prologue(c, nullptr, k_raw, v_raw, s->pos_thw, s->n_tokens, st, false))) return r;
  c->staging_read = false;
  if (c->N > 1) {
    if (c->external_x) {
      suspend(c, 2, 1, s->n_tokens);
      c->pend.prof = prof;
      c->pend.chunk_id = s->chunk_id;
      return DZ_OK;
    }
    if ((r = exchange_pre(c, false, s->n_tokens, st))) return r;
  }
  return append_commit(c, s->chunk_id, s->n_tokens, prof, st);
}

}  // extern "C"

namespace {

// Stages of one attention call under SP: [prologue] -> exchange 0 -> [attention] -> exchange 2 ->
// [unpack].  With DZ_FLAG_EXTERNAL_EXCHANGE the call stops at each exchange and dz_sp_resume
// runs the next stage.
void attend_mark(dz_ctx* c, bool prof, int i, cudaStream_t st) {
  if (prof) cudaEventRecord(c->ev[i], st);
}

void attend_done(dz_ctx* c, bool prof, bool stage_chunk, int32_t chunk_id, int32_t kind, int64_t n) {
  c->have_attend_ev = prof;
  if (stage_chunk) {
    c->staged = true;
    c->staged_id = chunk_id;
    c->staged_kind = kind;
    c->staged_n = n;
  }
}

dz_status attend_unpack(dz_ctx* c, int64_t n, void* out, bool prof, cudaStream_t st) {
  dz_status r = cuda_check(c, dz::launch_sp_unpack(c->base + c->L.or_off, out, c->N, c->B, (int32_t)(n / c->N), c->Hl,
                                                   c->D, st),
                           "unpack launch");
  if (r) return r;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  attend_mark(c, prof, 4, st);
  return DZ_OK;
}

// SP: K2 on this rank's heads over the full sequence, into the local O buffer; then exchange 2.
dz_status attend_sp_attention(dz_ctx* c, int64_t n, const dz::SpanTable& spans, void* out, bool prof,
                              cudaStream_t st) {
  attend_mark(c, prof, 2, st);
  dz_status r = run_attention(c, n, spans, c->base + c->L.ol_off, n * c->Hl * c->D, (int64_t)c->Hl * c->D, nullptr,
                              nullptr, st);
  if (r) return r;
  attend_mark(c, prof, 3, st);
  if (c->external_x) {
    suspend(c, 1, 2, n);
    c->pend.out = out;
    return DZ_OK;
  }
  if ((r = exchange_post(c, n, st))) return r;
  return attend_unpack(c, n, out, prof, st);
}

// One attention call (K1 prologue [+ exchange] + K2 [+ exchange + unpack]) over
// n new tokens described by `spans`; keys = committed chunks + the new tokens.
dz_status attend_impl(dz_ctx* c, const void* q_raw, const void* k_raw, const void* v_raw, const int32_t* pos,
                      int64_t n, const dz::SpanTable& spans, void* out, bool may_commit, int32_t chunk_id,
                      int32_t kind, cudaStream_t st, const AppendJob* aj = nullptr, int32_t aj_id = 0) {
  dz_status r;
  c->staged = false;
  if (aj) {  // room for the appended chunk and the staging slots after it (compaction if needed)
    if ((r = ensure_staging_room(c, st, aj->n))) return r;
  }
  const int64_t valid_new = c->valid + (aj ? aj->n : 0);
  // The new tokens' K'/V are only staged after the committed slots when the chunk may be committed
  // (attend_chunk of a CLEAN chunk), the exchange needs them (SP) or the new keys do not start at a
  // key step; otherwise K' goes to the current-chunk buffer, V is read in place from the caller's
  // input, and the attention only reads the committed cache.
  const bool cur_sep = c->N == 1 && !may_commit && valid_new % dz::attention_step_keys(c->m_static) == 0;
  c->staging_read = !cur_sep;
  const bool prof = c->ev[0] != nullptr && c->prof_on;
  const bool stage_chunk = chunk_id >= 0;
  attend_mark(c, prof, 0, st);
  if ((r = run_prologue(c, q_raw, k_raw, cur_sep ? nullptr : v_raw, pos, n, st, cur_sep, aj))) return r;
  if (aj) {  // the ground-truth chunk is committed: the attention's keys include it
    c->valid += aj->n;
    c->chunks.emplace_back(aj_id, aj->n);
    c->last_id = aj_id;
    c->have_append_ev = false;
  }
  attend_mark(c, prof, 1, st);
  if (c->N == 1) {
    attend_mark(c, prof, 2, st);
    if ((r = run_attention(c, n, spans, out, n * c->H * c->D, (int64_t)c->H * c->D,
                           cur_sep ? c->base + c->L.kc_off : nullptr, cur_sep ? v_raw : nullptr, st)))
      return r;
    attend_mark(c, prof, 3, st);
    attend_mark(c, prof, 4, st);
    attend_done(c, prof, stage_chunk, chunk_id, kind, n);
    return DZ_OK;
  }
  if (c->external_x) {
    suspend(c, 1, 0, n);
    c->pend.spans = spans;
    c->pend.out = out;
    c->pend.prof = prof;
    c->pend.stage_chunk = stage_chunk;
    c->pend.chunk_id = chunk_id;
    c->pend.kind = kind;
    return DZ_OK;
  }
  if ((r = exchange_pre(c, true, n, st))) return r;
  if ((r = attend_sp_attention(c, n, spans, out, prof, st))) return r;
  attend_done(c, prof, stage_chunk, chunk_id, kind, n);
  return DZ_OK;
}

dz_status check_attend_ptrs(dz_ctx* c, const void* q_raw, const void* k_raw, const void* v_raw, const void* out) {
  if (!q_raw || !k_raw || !v_raw || !out) return fail(c, DZ_EINVAL, "null q/k/v/out");
  if (!aligned16(q_raw) || !aligned16(k_raw) || !aligned16(v_raw) || !aligned16(out))
    return fail(c, DZ_EINVAL, "q/k/v/out must be 16-byte aligned");
  return DZ_OK;
}

// span table entry i (Fig. 10 rule, R3)
void set_span(dz::SpanTable& t, int i, int32_t chunk_id, int32_t kind, int32_t start, int32_t n) {
  t.start[i] = start;
  t.start[i + 1] = start + n;
  t.kc[i] = kind == DZ_CLEAN ? chunk_id : INT32_MAX;
  t.qth[i] = kind == DZ_NOISY ? chunk_id : chunk_id + 1;
}

}  // namespace

extern "C" {

dz_status dz_attend_chunk(dz_ctx* c, const void* q_raw, const void* k_raw, const void* v_raw, const dz_span* s,
                          void* out, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if ((r = check_attend_ptrs(c, q_raw, k_raw, v_raw, out))) return r;
  if ((r = check_span(c, s))) return r;
  if ((r = check_device(c))) return r;
  dz::SpanTable t;
  t.n = 1;
  set_span(t, 0, s->chunk_id, s->kind, 0, s->n_tokens);
  return attend_impl(c, q_raw, k_raw, v_raw, s->pos_thw, s->n_tokens, t, out, s->kind == DZ_CLEAN, s->chunk_id,
                     s->kind, static_cast<cudaStream_t>(stream));
}

dz_status dz_attend_spans(dz_ctx* c, const void* q_raw, const void* k_raw, const void* v_raw, const int32_t* pos_thw,
                          const dz_span* spans, int32_t n_spans, void* out, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if ((r = check_attend_ptrs(c, q_raw, k_raw, v_raw, out))) return r;
  if (!pos_thw || !spans) return fail(c, DZ_EINVAL, "null positions or spans");
  if (n_spans <= 0 || n_spans > dz::kMaxSpans)
    return fail(c, DZ_EINVAL, "n_spans %d outside [1, %d]", n_spans, dz::kMaxSpans);
  dz::SpanTable t;
  t.n = n_spans;
  int64_t n = 0;
  for (int i = 0; i < n_spans; ++i) {
    const dz_span& s = spans[i];
    if (s.kind != DZ_CLEAN && s.kind != DZ_NOISY) return fail(c, DZ_EINVAL, "span %d: bad kind %d", i, s.kind);
    if (s.n_tokens <= 0) return fail(c, DZ_ESHAPE, "span %d: n_tokens %d must be positive", i, s.n_tokens);
    if (s.chunk_id <= c->last_id || s.chunk_id == INT32_MAX)
      return fail(c, DZ_ESTATE, "span %d: chunk id %d must exceed the last committed id %d", i, s.chunk_id,
                  c->last_id);
    set_span(t, i, s.chunk_id, s.kind, (int32_t)n, s.n_tokens);
    n += s.n_tokens;
  }
  if (n % c->N) return fail(c, DZ_ESHAPE, "%lld tokens not a multiple of world_size %d", (long long)n, c->N);
  if (c->peer_mode && (n / c->N) % 8)
    return fail(c, DZ_ESHAPE, "DZ_FLAG_PEER_STORE: %lld tokens per rank is not a multiple of 8", (long long)(n / c->N));
  if (n > c->cfg.max_chunk_tokens)
    return fail(c, DZ_ECAPACITY, "%lld span tokens exceed max_chunk_tokens %d", (long long)n, c->cfg.max_chunk_tokens);
  if (n_spans > 1) {  // K2 keeps the (query group, key step) classes of a span layout in a 65536-tile table
    const int step_keys = dz::attention_step_keys(c->m_static);
    const int64_t tiles = ((n + dz::kTileQ - 1) / dz::kTileQ) * ((c->valid + n + step_keys - 1) / step_keys);
    if (dz::attention_has_step_table(c->D, c->m_static) && tiles > dz::kMaxStepTiles)
      return fail(c, DZ_ESHAPE, "span layout of %lld query groups x key steps exceeds %d tiles", (long long)tiles,
                  dz::kMaxStepTiles);
  }
  if ((r = check_device(c))) return r;
  return attend_impl(c, q_raw, k_raw, v_raw, pos_thw, n, t, out, false, -1, 0, static_cast<cudaStream_t>(stream));
}

dz_status dz_append_attend(dz_ctx* c, const void* k_gt, const void* v_gt, const dz_span* gt, const void* q_raw,
                           const void* k_raw, const void* v_raw, const dz_span* s, void* out, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if (!k_gt || !v_gt || !aligned16(k_gt) || !aligned16(v_gt)) return fail(c, DZ_EINVAL, "null/misaligned k_gt or v_gt");
  if ((r = check_attend_ptrs(c, q_raw, k_raw, v_raw, out))) return r;
  if ((r = check_span(c, gt))) return r;
  if (gt->kind != DZ_CLEAN) return fail(c, DZ_ESTATE, "only clean chunks enter the cache (Alg. 2 l.603)");
  if (c->valid + gt->n_tokens > c->cfg.cache_capacity_tokens)
    return fail(c, DZ_ECAPACITY, "cache full: %lld + %d > %lld", (long long)c->valid, gt->n_tokens,
                (long long)c->cfg.cache_capacity_tokens);
  if ((r = check_span(c, s))) return r;
  if (s->chunk_id <= gt->chunk_id)
    return fail(c, DZ_ESTATE, "chunk id %d must exceed the appended chunk's id %d", s->chunk_id, gt->chunk_id);
  if (c->external_x)
    return fail(c, DZ_EINVAL, "with DZ_FLAG_EXTERNAL_EXCHANGE call dz_append_kv and dz_attend_chunk");
  if ((r = check_device(c))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // one launch for both prologues needs the token-loop prologue (one GPU, H within one pass of it)
  static const bool no_fuse = getenv("DZ_NO_FUSED_APPEND") != nullptr;  // diagnostics: the two calls
  const bool fused = c->N == 1 && c->H <= 3 * (256 / (c->D / 8)) && !no_fuse;
  if (!fused) {
    if ((r = dz_append_kv(c, k_gt, v_gt, gt, stream))) return r;
    return dz_attend_chunk(c, q_raw, k_raw, v_raw, s, out, stream);
  }
  dz::SpanTable t;
  t.n = 1;
  set_span(t, 0, s->chunk_id, s->kind, 0, s->n_tokens);
  AppendJob aj;
  aj.k = k_gt;
  aj.v = v_gt;
  aj.pos = gt->pos_thw;
  aj.n = gt->n_tokens;
  return attend_impl(c, q_raw, k_raw, v_raw, s->pos_thw, s->n_tokens, t, out, s->kind == DZ_CLEAN, s->chunk_id,
                     s->kind, st, &aj, gt->chunk_id);
}

dz_status dz_sp_set_peers(dz_ctx* c, void* const* storages, int32_t n) {
  if (!c || !storages) return DZ_EINVAL;
  if (!c->peer_mode) return fail(c, DZ_ESTATE, "created without DZ_FLAG_PEER_STORE");
  if (n != c->N) return fail(c, DZ_EINVAL, "%d peer storages for world_size %d", n, c->N);
  for (int p = 0; p < n; ++p) {
    if (!storages[p] || (reinterpret_cast<uintptr_t>(storages[p]) & (kAlign - 1)))
      return fail(c, DZ_EINVAL, "peer %d storage null or not 256-byte aligned", p);
    c->peers[p] = static_cast<char*>(storages[p]);
  }
  if (c->peers[c->rank] != c->base) return fail(c, DZ_EINVAL, "entry %d must be this rank's cache_storage", c->rank);
  c->peers_set = true;
  return DZ_OK;
}

dz_status dz_attend_spans_backward(dz_ctx* c, const void* q_raw, const void* k_raw, const void* v_raw,
                                   const int32_t* pos_thw, const dz_span* spans, int32_t n_spans, const void* out,
                                   const float* lse, const void* dout, void* dq_raw, void* dk_raw, void* dv_raw,
                                   float* dq_gain, float* dk_gain, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if ((r = check_attend_ptrs(c, q_raw, k_raw, v_raw, out))) return r;
  if (!pos_thw || !spans || !lse || !dout || !dq_raw || !dk_raw || !dv_raw || !dq_gain || !dk_gain ||
      !aligned16(dout) || !aligned16(dq_raw) || !aligned16(dk_raw) || !aligned16(dv_raw) || !aligned16(lse))
    return fail(c, DZ_EINVAL, "null or misaligned backward argument");
  if (!(c->cfg.flags & DZ_FLAG_BACKWARD)) return fail(c, DZ_ESTATE, "created without DZ_FLAG_BACKWARD");
  if (c->N != 1 || c->D != 128 || c->f8) return fail(c, DZ_ESHAPE, "backward: one GPU, head_dim 128, bf16 path");
  if (c->valid != 0) return fail(c, DZ_ESTATE, "backward: the teacher-forced layout has no committed cache");
  if (n_spans <= 0 || n_spans > dz::kMaxSpans)
    return fail(c, DZ_EINVAL, "n_spans %d outside [1, %d]", n_spans, dz::kMaxSpans);
  dz::SpanTable t;
  t.n = n_spans;
  int64_t n = 0;
  for (int i = 0; i < n_spans; ++i) {
    const dz_span& s = spans[i];
    if (s.kind != DZ_CLEAN && s.kind != DZ_NOISY) return fail(c, DZ_EINVAL, "span %d: bad kind %d", i, s.kind);
    if (s.n_tokens <= 0) return fail(c, DZ_ESHAPE, "span %d: n_tokens %d must be positive", i, s.n_tokens);
    set_span(t, i, s.chunk_id, s.kind, (int32_t)n, s.n_tokens);
    n += s.n_tokens;
  }
  if (n > c->cfg.max_chunk_tokens)
    return fail(c, DZ_ECAPACITY, "%lld span tokens exceed max_chunk_tokens %d", (long long)n, c->cfg.max_chunk_tokens);
  t.valid = 0;
  if ((r = check_device(c))) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // recompute Q' (pre-scaled, fp16) and K' (fp16, current-chunk buffer) with the forward's prologue
  if ((r = run_prologue(c, q_raw, k_raw, nullptr, pos_thw, n, st, true))) return r;
  dz::BwdArgs a;
  a.dq_acc = reinterpret_cast<float*>(c->base + c->L.bq_off);
  a.dk = reinterpret_cast<float*>(c->base + c->L.bk_off);
  a.delta = reinterpret_cast<float*>(c->base + c->L.bd_off);
  a.lse2 = reinterpret_cast<float*>(c->base + c->L.bl_off);
  const size_t nel = (size_t)c->B * n * c->H * c->D;
  if ((r = cuda_check(c, cudaMemsetAsync(a.dq_acc, 0, nel * 4, st), "dq clear"))) return r;
  if ((r = cuda_check(c, cudaMemsetAsync(dq_gain, 0, (size_t)c->H * c->D * 4, st), "dgq clear"))) return r;
  if ((r = cuda_check(c, cudaMemsetAsync(dk_gain, 0, (size_t)c->H * c->D * 4, st), "dgk clear"))) return r;
  const int64_t bs = n * c->H * c->D;
  if (!make_tmap(&a.tm_k, c->base + c->L.kc_off, 0, c->D, c->H, n, c->B, bs, 64, 128) ||
      !make_tmap(&a.tm_v, v_raw, 1, c->D, c->H, n, c->B, bs, 64, 128) ||
      !make_tmap(&a.tm_q, c->base + c->L.q_off, 0, c->D, c->H, n, c->B, bs, 64, 64) ||
      !make_tmap(&a.tm_do, dout, 1, c->D, c->H, n, c->B, bs, 64, 64))
    return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled (backward) failed");
  {  // dL/dq' accumulator: fp32, box (D, 1, 64, 1), no swizzle -- the target of TMA reduce-adds
    auto fn = encode_fn();
    cuuint64_t dims[4] = {(cuuint64_t)c->D, (cuuint64_t)c->H, (cuuint64_t)n, (cuuint64_t)c->B};
    cuuint64_t strides[3] = {(cuuint64_t)c->D * 4, (cuuint64_t)c->H * c->D * 4, (cuuint64_t)bs * 4};
    cuuint32_t box[4] = {(cuuint32_t)c->D, 1, 64, 1}, estr[4] = {1, 1, 1, 1};
    if (!fn || fn(&a.tm_dq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.dq_acc, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(c, DZ_ECUDA, "cuTensorMapEncodeTiled (dq) failed");
  }
  a.dout = dout;
  a.out = out;
  a.lse = lse;
  a.dv = dv_raw;
  a.q_raw = q_raw;
  a.k_raw = k_raw;
  a.dq = dq_raw;
  a.dk_raw = dk_raw;
  a.gain[0] = c->cfg.q_gain;
  a.gain[1] = c->cfg.k_gain;
  a.dgain[0] = dq_gain;
  a.dgain[1] = dk_gain;
  a.pos = pos_thw;
  a.tab = reinterpret_cast<const float2*>(c->base + c->L.rope_off);
  a.tab_len = dz::kRopeLen;
  a.eps = c->eps;
  a.B = c->B;
  a.n = (int32_t)n;
  a.n_pad = (int32_t)((n + 63) / 64 * 64);
  a.H = c->H;
  a.D = c->D;
  a.scale_q = c->scale;
  a.scale_k = 0.69314718055994530942f;  // Q' carries scale * log2(e): dk' = scale * dS^T q' = ln 2 * dS^T Q'
  a.spans = t;
  for (int j = 0; j < c->D / 2; ++j) {
    a.omega[j] = c->pro.omega[j];
    a.axis[j] = c->pro.axis[j];
  }
  r = cuda_check(c, dz::launch_attention_backward(a, st), "backward launch");
  if (!r) g_launches.fetch_add(3, std::memory_order_relaxed);
  return r;
}

int32_t dz_sp_pending(const dz_ctx* c, int32_t* phase, dz_xfer* out, int32_t cap) {
  if (!c || cap < 0) return DZ_EINVAL;
  if (phase) *phase = c->pend.op ? c->pend.phase : -1;
  if (!c->pend.op) return 0;
  if (out)
    for (int32_t i = 0; i < (int32_t)c->pend.plan.size() && i < cap; ++i) out[i] = c->pend.plan[i];
  return (int32_t)c->pend.plan.size();
}

dz_status dz_sp_resume(dz_ctx* c, void* stream) {
  if (!c) return DZ_EINVAL;
  if (c->poisoned) return fail(c, DZ_ESTATE, "context poisoned by an earlier CUDA/NCCL error: %s", c->err.c_str());
  if (!c->pend.op) return fail(c, DZ_ESTATE, "no exchange pending");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dz_ctx::Pending p = c->pend;
  c->pend = dz_ctx::Pending();
  dz_status r = DZ_OK;
  if (p.op == 2) return append_commit(c, p.chunk_id, p.n, p.prof, st);  // append: K'/V have landed
  if (p.phase == 0) {  // attend: Q', K', V have landed -> attention (stops again at exchange 2)
    if ((r = attend_sp_attention(c, p.n, p.spans, p.out, p.prof, st))) return r;
    if (c->pend.op) {  // carry the call's finalisation to the last stage
      c->pend.prof = p.prof;
      c->pend.stage_chunk = p.stage_chunk;
      c->pend.chunk_id = p.chunk_id;
      c->pend.kind = p.kind;
      return DZ_OK;
    }
  } else if ((r = attend_unpack(c, p.n, p.out, p.prof, st))) {  // phase 2: O has landed
    return r;
  }
  attend_done(c, p.prof, p.stage_chunk, p.chunk_id, p.kind, p.n);
  return DZ_OK;
}

dz_status dz_commit_staged(dz_ctx* c, int32_t chunk_id, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if (!c->staged || c->staged_id != chunk_id || c->staged_kind != DZ_CLEAN)
    return fail(c, DZ_ESTATE, "no clean chunk %d staged by the last attend", chunk_id);
  if (c->valid + c->staged_n > c->cfg.cache_capacity_tokens)
    return fail(c, DZ_ECAPACITY, "cache full");
  c->valid += c->staged_n;
  c->chunks.emplace_back(chunk_id, c->staged_n);
  c->last_id = chunk_id;
  c->staged = false;
  return ensure_staging_room(c, static_cast<cudaStream_t>(stream));
}

dz_status dz_evict_front(dz_ctx* c, int32_t n_chunks, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if (n_chunks < 0 || (size_t)n_chunks > c->chunks.size())
    return fail(c, DZ_EINVAL, "cannot evict %d of %zu chunks", n_chunks, c->chunks.size());
  for (int i = 0; i < n_chunks; ++i) {
    c->start += c->chunks.front().second;
    c->valid -= c->chunks.front().second;
    c->chunks.pop_front();
  }
  if (c->valid == 0) c->start = 0;
  c->staged = false;
  return ensure_staging_room(c, static_cast<cudaStream_t>(stream));
}

dz_status dz_cache_state(const dz_ctx* c, int64_t* valid, int32_t* n_chunks, int32_t* last_id) {
  if (!c) return DZ_EINVAL;
  if (valid) *valid = c->valid;
  if (n_chunks) *n_chunks = (int32_t)c->chunks.size();
  if (last_id) *last_id = c->last_id;
  return DZ_OK;
}

dz_status dz_cache_view(const dz_ctx* c, int32_t b, void** k0, void** v0, int64_t* stride) {
  if (!c || b < 0 || b >= c->B) return DZ_EINVAL;
  if (k0) *k0 = c->kslot(b, c->start);
  if (v0) *v0 = c->vslot(b, c->start);
  if (stride) *stride = (int64_t)c->Hl * c->D;
  return DZ_OK;
}

dz_status dz_copy_lse(dz_ctx* c, float* dst, size_t elems, void* stream) {
  dz_status r = check_ready(c);
  if (r) return r;
  if (!(c->cfg.flags & DZ_FLAG_WRITE_LSE)) return fail(c, DZ_ESTATE, "created without DZ_FLAG_WRITE_LSE");
  if ((r = check_device(c))) return r;
  const size_t need = (size_t)c->B * c->Hl * c->last_nq;
  if (!dst || elems < need) return fail(c, DZ_EINVAL, "lse buffer too small (%zu < %zu)", elems, need);
  return cuda_check(c, cudaMemcpyAsync(dst, c->base + c->L.lse_off, need * 4, cudaMemcpyDeviceToDevice,
                                       static_cast<cudaStream_t>(stream)),
                    "lse copy");
}

dz_status dz_get_tile_map(const dz_ctx* c, uint8_t* host, size_t cap, int32_t* nq, int32_t* nk, int32_t* bm,
                          int32_t* bn) {
  if (!c) return DZ_EINVAL;
  if (!c->have_map) return DZ_ESTATE;
  const size_t need = (size_t)c->last_nq_tiles * c->last_nkv_tiles;
  if (nq) *nq = c->last_nq_tiles;
  if (nk) *nk = c->last_nkv_tiles;
  if (bm) *bm = dz::kTileQ;
  if (bn) *bn = c->last_step_keys;
  if (!host) return DZ_OK;
  if (cap < need) return DZ_EINVAL;
  // synchronous device read of the kernel-written debug map (tests only)
  if (cudaMemcpy(host, c->base + c->L.map_off, need, cudaMemcpyDeviceToHost) != cudaSuccess) return DZ_ECUDA;
  return DZ_OK;
}

dz_status dz_profile_enable(dz_ctx* c, int32_t on) {
  if (!c) return DZ_EINVAL;
  if (!c->ev[0]) return fail(c, DZ_ESTATE, "created without DZ_FLAG_PROFILE");
  c->prof_on = on != 0;
  if (!c->prof_on) c->have_attend_ev = c->have_append_ev = false;
  return DZ_OK;
}

dz_status dz_profile_last(dz_ctx* c, float* ms) {
  if (!c || !ms) return DZ_EINVAL;
  if (!c->ev[0]) return fail(c, DZ_ESTATE, "created without DZ_FLAG_PROFILE");
  for (int i = 0; i < 6; ++i) ms[i] = 0.f;
  auto el = [&](cudaEvent_t a, cudaEvent_t b, float* o) {
    if (cudaEventSynchronize(b) != cudaSuccess) return false;
    return cudaEventElapsedTime(o, a, b) == cudaSuccess;
  };
  bool ok = true;
  if (c->have_attend_ev) {
    ok &= el(c->ev[0], c->ev[1], &ms[0]);
    ok &= el(c->ev[1], c->ev[2], &ms[1]);
    ok &= el(c->ev[2], c->ev[3], &ms[2]);
    ok &= el(c->ev[3], c->ev[4], &ms[3]);
    ok &= el(c->ev[0], c->ev[4], &ms[4]);
  }
  if (c->have_append_ev) ok &= el(c->ev_app[0], c->ev_app[1], &ms[5]);
  return ok ? DZ_OK : fail(c, DZ_ECUDA, "cudaEventElapsedTime failed");
}

dz_status dz_destroy(dz_ctx* c) {
  if (!c) return DZ_OK;
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_app)
    if (e) cudaEventDestroy(e);
  delete c;
  return DZ_OK;
}

const char* dz_status_string(dz_status s) {
  switch (s) {
    case DZ_OK: return "DZ_OK";
    case DZ_EINVAL: return "DZ_EINVAL: invalid argument";
    case DZ_ESHAPE: return "DZ_ESHAPE: unsupported shape";
    case DZ_ECAPACITY: return "DZ_ECAPACITY: capacity exceeded";
    case DZ_ESTATE: return "DZ_ESTATE: invalid cache state or ordering";
    case DZ_ECUDA: return "DZ_ECUDA: CUDA error";
    case DZ_ENCCL: return "DZ_ENCCL: NCCL error";
    case DZ_ERANGE: return "DZ_ERANGE: gains overflow fp16";
  }
  return "unknown dz_status";
}

const char* dz_last_error(const dz_ctx* c) { return c ? c->err.c_str() : "null context"; }

dz_status dz_nccl_unique_id(void* id128) {
  if (!id128) return DZ_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  return ncclGetUniqueId(static_cast<ncclUniqueId*>(id128)) == ncclSuccess ? DZ_OK : DZ_ENCCL;
}

dz_status dz_nccl_comm_init(int32_t world_size, const void* id128, int32_t rank, void** comm) {
  if (!id128 || !comm || world_size <= 0 || rank < 0 || rank >= world_size) return DZ_EINVAL;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  if (ncclCommInitRank(&c, world_size, id, rank) != ncclSuccess) return DZ_ENCCL;
  *comm = c;
  return DZ_OK;
}

dz_status dz_nccl_comm_destroy(void* comm) {
  if (!comm) return DZ_OK;
  return ncclCommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? DZ_OK : DZ_ENCCL;
}

dz_status dz_debug_watchdog(uint32_t* host8, int32_t reset) {
  if (!host8) return DZ_EINVAL;
  if (dz::read_watchdog(host8) != cudaSuccess) return DZ_ECUDA;
  if (reset && dz::reset_watchdog() != cudaSuccess) return DZ_ECUDA;
  return DZ_OK;
}

dz_status dz_debug_k2_clock(uint64_t* host2, int32_t reset) {
  return dz::k2_clock(host2, reset) == cudaSuccess ? DZ_OK : DZ_ECUDA;
}

dz_status dz_debug_trace(int32_t enable, uint32_t* host, size_t n) {
  return dz::trace_control(enable, host, n) == cudaSuccess ? DZ_OK : DZ_ECUDA;
}

int32_t dz_sp_plan(const dz_ctx* c, int32_t phase, int32_t n_tokens, dz_xfer* out, int32_t cap) {
  if (!c || phase < 0 || phase > 2 || n_tokens <= 0 || n_tokens % c->N || cap < 0) return DZ_EINVAL;
  const std::vector<dz_xfer> plan = make_plan(c, phase, n_tokens);
  if (out)
    for (int32_t i = 0; i < (int32_t)plan.size() && i < cap; ++i) out[i] = plan[i];
  return (int32_t)plan.size();
}

dz_status dz_debug_sp_unpack(const void* recv, void* out, int32_t world_size, int32_t batch, int32_t n_local,
                             int32_t heads_local, int32_t head_dim, void* stream) {
  if (!recv || !out || world_size <= 0 || batch <= 0 || n_local < 0 || heads_local <= 0 || head_dim % 8)
    return DZ_EINVAL;
  return dz::launch_sp_unpack(recv, out, world_size, batch, n_local, heads_local, head_dim,
                              static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? DZ_OK
             : DZ_ECUDA;
}

dz_status dz_debug_l2_discard(void* buf, size_t bytes, void* stream) {
  if (!buf || bytes % 128) return DZ_EINVAL;
  return dz::launch_l2_discard(buf, bytes, static_cast<cudaStream_t>(stream)) == cudaSuccess ? DZ_OK : DZ_ECUDA;
}

int64_t dz_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int32_t dz_attention_units(const dz_ctx* c, int32_t n) {
  if (!c || n <= 0) return 0;
  return dz::attention_units(c->B, c->Hl, n);
}

}  // extern "C"
