/*
 * dz.h -- C ABI of libdz: block-causal chunk attention for DreamZero-style
 * chunk-wise autoregressive video/action diffusion on NVIDIA B200 (sm_100a).
 *
 * The operation (arXiv 2602.15922, PAPER.md):
 *   * A chunk is K latent frames of view-concatenated video tokens plus the
 *     chunk's action tokens (l.94 "concatenate all views into a single frame",
 *     l.99 "each chunk has a fixed number of latent frames K").
 *   * During one denoising step the current noisy chunk attends
 *     bidirectionally to itself and causally to the KV cache of clean previous
 *     chunks (Fig. 10 / l.505; Alg. 2 l.584-585, u_theta(...; KV, ..., update=False)).
 *   * Ground-truth injection appends the clean chunk's keys/values to the cache
 *     (Alg. 2 l.569-570 and l.601-602, update=True); predicted latents are
 *     never cached (l.603).
 *   * Q and K first get per-head RMSNorm and 3D (frame, height, width) RoPE
 *     (BASELINE.json north_star).  Conventions (readings A1-A9):
 *     x' = RoPE(x / sqrt(mean(x^2) + eps) * g); RoPE rotates interleaved pairs
 *     (2i, 2i+1) inside axis slices [t | h | w] of widths rope_dims, by angle
 *     p_axis * theta^(-2i / d_axis).
 *
 * Tensor conventions (all device memory, caller-owned, contiguous):
 *   * activations q_raw, k_raw, v_raw, out: bf16 [batch][n_local][heads][head_dim]
 *     (token-major, what a QKV projection emits); n_local = n / world_size.
 *   * positions: int32 [n_local][3] = (t, h, w) of this rank's tokens, global
 *     coordinates (the same positions for every batch element).
 *   * gains: fp32 [heads * head_dim] (q_gain, k_gain).
 *   * cache storage: one caller-owned device buffer of dz_cache_bytes() bytes;
 *     K' is kept post-norm/post-RoPE in fp16, V as given in bf16, token-major
 *     per rank: [batch][slots][heads/world_size][head_dim].
 *
 * Streams and concurrency: every kernel and NCCL call is enqueued on the given
 * stream (a cudaStream_t passed as void*); no call synchronises the host.
 * Inputs must stay untouched until the stream passes the call.  A context is
 * single-owner: calls on one context must be serialised by the caller;
 * different contexts may be used concurrently.
 *
 * Errors: argument/state validation happens before anything is enqueued and
 * leaves the context unchanged.  A CUDA or NCCL enqueue error returns
 * DZ_ECUDA / DZ_ENCCL and poisons the context (later calls return DZ_ESTATE
 * until dz_destroy).  Device faults surface at the caller's next sync.  The
 * library never throws and never aborts.
 */
#ifndef DZ_H_
#define DZ_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DZ_API __attribute__((visibility("default")))
#else
#define DZ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dz_ctx dz_ctx; /* opaque; one per (layer, batch group) */

typedef enum {
  DZ_OK = 0,
  DZ_EINVAL = -1,    /* null pointer, bad flag, misaligned pointer            */
  DZ_ESHAPE = -2,    /* unsupported shape (head_dim, rope split, n % world)  */
  DZ_ECAPACITY = -3, /* cache or staging capacity exceeded                   */
  DZ_ESTATE = -4,    /* chunk ordering violated, nothing staged, poisoned    */
  DZ_ECUDA = -5,     /* CUDA error while enqueuing (see dz_last_error)       */
  DZ_ENCCL = -6,     /* NCCL error while enqueuing                           */
  DZ_ERANGE = -7     /* sqrt(head_dim)*max|gain| would overflow fp16 Q'/K'    */
} dz_status;

enum { DZ_CLEAN = 0, DZ_NOISY = 1 }; /* dz_span.kind (Fig. 10: C chunks vs Z/Y chunks) */

enum {
  DZ_FLAG_NONE = 0,
  DZ_FLAG_WRITE_LSE = 1, /* keep a per-row log-sum-exp of the last attend (dz_copy_lse) */
  DZ_FLAG_PROFILE = 2,   /* record CUDA events around every kernel/exchange (dz_profile_last) */
  DZ_FLAG_ONLINE_SOFTMAX = 4, /* always track the running row max, even when the QK-norm bound
                                 D*max|g|^2*scale would allow a fixed softmax base (see dz_create) */
  DZ_FLAG_TILE_MAP = 8,       /* record the attention kernel's tile decisions (dz_get_tile_map; tests) */
  DZ_FLAG_EXTERNAL_EXCHANGE = 16, /* world_size > 1 without NCCL: calls stop at each all-to-all, the
                                     caller moves the bytes dz_sp_pending lists, then dz_sp_resume */
  DZ_FLAG_WHOLE_UNITS = 32,   /* no stream-K split: each (batch, head, 256-row query group) is computed
                                 whole by one CTA pair, so its bits do not depend on the unit count
                                 (identical results at every world size, reading A21) */
  DZ_FLAG_HOST_ONLY = 64,     /* planning context: never touches the device (gains unread, the caller's
                                 max_abs_gain is taken as given); compute calls validate, then
                                 return DZ_ESTATE without enqueuing; dz_sp_plan works (host tests) */
  DZ_FLAG_FP8_QK = 256,       /* Q' and K' (cache and current chunk) stored as
                                 FP8 E4M3 (times 2^a and 2^-a, a chosen at create from the gains so
                                 scores need no descale) and QK^T on tcgen05 kind::f8f6f4; PV stays
                                 bf16.  Its own error budget, not BJ:5.  One GPU,
                                 head_dim 128, <= 48 heads (else DZ_ESHAPE) and the fixed softmax
                                 base (else DZ_ERANGE).  dz_cache_view's K' is then E4M3 bytes */
  DZ_FLAG_BACKWARD = 512,     /* allocate the backward workspace (dz_attend_spans_backward) */
  DZ_FLAG_PEER_STORE = 128    /* Ulysses without exchange copies: the prologue
                                 stores each destination rank's Q'/K'/V rows straight into that
                                 rank's storage and the attention's epilogue stores O rows straight
                                 into their owner's receive buffer, through the peer storage
                                 pointers of dz_sp_set_peers (CUDA IPC / NVLink-mapped on a node);
                                 the exchanges become barriers (a 4-byte NCCL all-reduce, or an
                                 empty dz_sp_pending list with DZ_FLAG_EXTERNAL_EXCHANGE).
                                 2 <= world_size <= 8 and at most 48 heads at head_dim 128
                                 (96 at 64), else DZ_ESHAPE */
};

typedef struct {
  int32_t batch;                 /* B: independent sequences (e.g. CFG cond/uncond) */
  int32_t heads;                 /* global heads H (Wan-14B: 40)                            */
  int32_t head_dim;              /* D in {64, 128}                                          */
  int32_t rope_dims[3];          /* (d_t, d_h, d_w), each even, sum == head_dim              */
  float rope_theta;              /* 0 => 10000                                              */
  float rms_eps;                 /* 0 => 1e-6                                               */
  float softmax_scale;           /* 0 => 1/sqrt(head_dim)                                   */
  int64_t cache_capacity_tokens; /* committed tokens per batch element (global sequence)    */
  int32_t max_chunk_tokens;      /* largest chunk n (global), staged after the committed part */
  int32_t window_slack_tokens;   /* extra slots so dz_evict_front rarely compacts; 0 = none */
  const float* q_gain;           /* device fp32 [heads*head_dim]; must outlive the ctx      */
  const float* k_gain;           /* device fp32 [heads*head_dim]; must outlive the ctx      */
  float max_abs_gain;            /* optional bound on |gain|: 0 = none; if > 0 it must be >= the
                                    true max (dz_create reads the gains; else DZ_ERANGE)       */
  void* cache_storage;           /* device buffer of >= dz_cache_bytes(cfg) bytes, 256-B aligned */
  size_t cache_bytes;
  void* nccl_comm;               /* ncclComm_t when world_size > 1 (NULL with DZ_FLAG_EXTERNAL_EXCHANGE) */
  int32_t world_size;            /* Ulysses sequence-parallel ranks (heads % world_size == 0) */
  int32_t rank;
  int32_t flags;                 /* DZ_FLAG_*                                               */
} dz_config;

/* One chunk of the sequence (Fig. 10): id, kind and its global token count. */
typedef struct {
  int32_t chunk_id;        /* chunk index; committed ids must increase                  */
  int32_t kind;            /* DZ_CLEAN or DZ_NOISY                                       */
  int32_t n_tokens;        /* global tokens of the chunk; n_tokens % world_size == 0     */
  const int32_t* pos_thw;  /* device int32 [n_tokens/world_size][3], this rank's tokens  */
} dz_span;

/* Bytes of cache storage the caller must provide for cfg:
 *   2 tensors (K' fp16, V bf16) x batch x (capacity + max_chunk + slack) x
 *   (heads / world_size) x head_dim x 2 B, plus the device workspace below (Q' and
 *   the noisy chunk's K' fp16, the stream-K partials, a 4096 x head_dim/2 fp32 RoPE
 *   (cos, sin) table written by the first prologue, SP buffers), each rounded up to
 *   256 B. 0 if cfg is invalid. */
DZ_API size_t dz_cache_bytes(const dz_config* cfg);

/* Validates cfg and computes the RoPE frequencies (fp64, host).  The device
 * workspace (Q', the RoPE table, the all-to-all buffers under SP, debug maps) lives inside the
 * caller's cache_storage (dz_cache_bytes counts it); the context allocates no
 * device memory.  Reads q_gain and k_gain once (a synchronous device-to-host copy;
 * an unreadable pointer gives DZ_EINVAL, a non-finite gain DZ_ERANGE) and takes
 * G = max |g| from them; a caller bound max_abs_gain > 0 below G is rejected
 * (DZ_ERANGE), and sqrt(head_dim) * G >= 6e4 would overflow fp16 Q'/K' (DZ_ERANGE).
 * Also derives the QK-norm logit bound
 *   |<q',k'>| * scale * log2(e) <= head_dim * G^2 * scale * log2(e)
 * (RMSNorm makes ||x'|| <= sqrt(head_dim) * max|g|); when it is <= 60 the
 * attention uses base 0 (p = 2^s in [2^-60, 2^60]) instead of a running row max
 * (DZ_FLAG_ONLINE_SOFTMAX disables this).  The gains are model weights: the bound
 * is taken at create, so a caller who later enlarges them must recreate the
 * context.  *out is owned by the caller until dz_destroy. */
DZ_API dz_status dz_create(const dz_config* cfg, dz_ctx** out);

/* Cache append of a clean chunk (Alg. 2 l.601-602, update=True): K' =
 * RoPE(RMSNorm(k_raw)) and V are written to slots [valid, valid + n) and
 * committed.  The append kernel may be scheduled while the previous kernel of
 * `stream` drains, but reads k_raw / v_raw / positions only after that kernel
 * (which may have produced them) has completed.  Requires chunk->kind == DZ_CLEAN, chunk_id greater than the last
 * committed id (else DZ_ESTATE) and valid + n <= capacity (else DZ_ECAPACITY).
 * k_raw, v_raw: bf16 [batch][n_local][heads][head_dim]. */
DZ_API dz_status dz_append_kv(dz_ctx* ctx, const void* k_raw, const void* v_raw, const dz_span* chunk, void* stream);

/* One denoising step of the current chunk (Alg. 2 l.584-585, update=False):
 * out = softmax(Q' K'^T * scale) V over keys = committed chunks (all have id <
 * chunk_id) plus the chunk itself (bidirectional, Fig. 10).  Q' and the chunk's
 * K' are computed here (K1 prologue).  A CLEAN chunk (which dz_commit_staged may
 * commit), SP, or new keys not starting at a key step (valid not a multiple of
 * 128 with the fixed softmax base, 256 otherwise): K' and V are staged after the
 * committed slots.  Otherwise (a NOISY chunk on one GPU) K' goes to a
 * current-chunk buffer, V is read in place from v_raw, and the call only reads
 * the cache.  The committed cache is never modified.  chunk_id must exceed every committed
 * id (else DZ_ESTATE); n <= max_chunk_tokens (else DZ_ECAPACITY).
 * out: bf16 [batch][n_local][heads][head_dim].
 * Capture-safe: no host synchronisation, every launch on `stream`, so the
 * denoising steps of one chunk can be recorded once into a CUDA graph and
 * replayed; a replay reads the committed state of the
 * capture, so re-capture after dz_append_kv / dz_evict_front / dz_commit_staged.
 * The context's one-time device setup (stream-K piece counters, RoPE table) runs
 * in the first call; if that call is captured, the setup is part of the graph and
 * the next eager call performs it again. */
DZ_API dz_status dz_attend_chunk(dz_ctx* ctx, const void* q_raw, const void* k_raw, const void* v_raw,
                          const dz_span* chunk, void* out, void* stream);

/* General Fig. 10 form (PAPER.md l.505 caption): the new
 * tokens are n_spans consecutive spans (the token ranges of q_raw/k_raw/v_raw
 * in order), each with its own chunk id and kind; spans[i].pos_thw is ignored
 * and pos_thw holds the positions of all new tokens of this rank, int32
 * [n_local_total][3].  Queries are the new tokens; keys are the committed
 * chunks followed by the new tokens.  A NOISY query of chunk k sees the CLEAN
 * keys of chunks < k and every key of its own span; a CLEAN query of chunk j
 * sees the CLEAN keys of chunks <= j; committed chunks are CLEAN and, because
 * every span id must exceed the last committed id (else DZ_ESTATE), visible to
 * every query.  Examples: the training layout [C0 .. C_{M-1}; Z1 .. Z_M] of
 * Fig. 10(a) with an empty cache; attend_chunk is the one-span case.
 * Key steps (128 keys with the fixed softmax base, 256 with the online one)
 * whose (query group of 256 rows, key step) pairs are all invisible are
 * skipped (never loaded, never multiplied); partially visible ones are masked
 * per element.  1 <= n_spans <= 64; the total token count must be <=
 * max_chunk_tokens (else DZ_ECAPACITY) and a multiple of world_size; with
 * several spans, ceil(n / 256) query groups x key steps over committed + new
 * keys must not exceed 65536 (the kernel's tile-class table; else DZ_ESHAPE).
 * Nothing is staged for dz_commit_staged.
 * out: bf16 [batch][n_local_total][heads][head_dim]. */
DZ_API dz_status dz_attend_spans(dz_ctx* ctx, const void* q_raw, const void* k_raw, const void* v_raw,
                                 const int32_t* pos_thw, const dz_span* spans, int32_t n_spans, void* out,
                                 void* stream);

/* Ground-truth injection of one chunk followed by the denoising step of the next (Alg. 2: the
 * update=True pass of chunk c-1, l.601-602, then u_theta(x_t; KV, ..., update=False) of chunk c,
 * l.584-585): exactly dz_append_kv(k_gt, v_gt, gt) then dz_attend_chunk(q_raw, k_raw, v_raw, chunk,
 * out) -- same results, same cache state -- but on one GPU both prologues (the appended chunk's K'/V
 * and the attended chunk's Q'/K') run in one kernel launch.  Validation as for the two calls, plus
 * chunk->chunk_id > gt->chunk_id (else DZ_ESTATE); nothing is enqueued if either fails.  Under SP
 * (or with more heads than one prologue pass holds) it performs the two calls; not available with
 * DZ_FLAG_EXTERNAL_EXCHANGE (DZ_EINVAL). */
DZ_API dz_status dz_append_attend(dz_ctx* ctx, const void* k_gt, const void* v_gt, const dz_span* gt, const void* q_raw,
                                  const void* k_raw, const void* v_raw, const dz_span* chunk, void* out, void* stream);

/* Backward of dz_attend_spans for teacher-forced training (PAPER.md l.115-119
 * "trajectory-level updates", Fig. 10(a) layout [C0 .. C_{M-1}; Z1 .. Z_M], Alg. 1 l.512-553):
 * given the same q_raw, k_raw, v_raw, positions and spans as the forward, its output `out` and its
 * natural-log LSE rows `lse` (fp32 [batch][heads][n], DZ_FLAG_WRITE_LSE + dz_copy_lse) and dout =
 * dL/dout, writes dq_raw, dk_raw, dv_raw = dL/d{q,k,v}_raw (bf16 [batch][n][heads][head_dim]) and
 * dq_gain, dk_gain = dL/dg (fp32 [heads*head_dim], overwritten), through the RMSNorm, the gains, the
 * 3D RoPE and the Fig. 10-masked attention.  Key tiles no query sees are never loaded against those
 * queries.  Needs DZ_FLAG_BACKWARD, one GPU, head_dim 128, the bf16 path (DZ_ESHAPE) and an empty
 * cache (DZ_ESTATE).  Tolerance against the fp64 oracle: DESIGN.md §4.  dv_raw and dk_raw are bitwise
 * repeatable (one CTA per key tile); dq_raw and the gain gradients sum per-tile contributions with fp32
 * reduce-adds in arrival order, so they repeat to fp32 rounding, not bitwise.  The fp32 dq accumulator
 * lives in the context's workspace (sized at dz_create from max_chunk_tokens). */
DZ_API dz_status dz_attend_spans_backward(dz_ctx* ctx, const void* q_raw, const void* k_raw, const void* v_raw,
                                          const int32_t* pos_thw, const dz_span* spans, int32_t n_spans,
                                          const void* out, const float* lse, const void* dout, void* dq_raw,
                                          void* dk_raw, void* dv_raw, float* dq_gain, float* dk_gain, void* stream);

/* Commit the chunk staged by the last dz_attend_chunk (which must have had
 * kind DZ_CLEAN and this chunk_id): the model-side "attend the clean chunk,
 * then update the cache" form of Alg. 2 l.601-602.  Moves no data.  DZ_ESTATE
 * if nothing matching is staged; DZ_ECAPACITY if the cache is full. */
DZ_API dz_status dz_commit_staged(dz_ctx* ctx, int32_t chunk_id, void* stream);

/* Drop the n_chunks oldest committed chunks (sliding context window, PAPER.md
 * l.510 "maximum context length is 8 latent frames").  RoPE is relative, so the
 * remaining keys need no re-rotation.  Usually bookkeeping only; compacts the
 * storage with a device copy on `stream` when the window reaches its end. */
DZ_API dz_status dz_evict_front(dz_ctx* ctx, int32_t n_chunks, void* stream);

/* Committed state: tokens per batch element, number of chunks, last chunk id (-1 if none). */
DZ_API dz_status dz_cache_state(const dz_ctx* ctx, int64_t* valid_tokens, int32_t* n_chunks, int32_t* last_chunk_id);

/* Device pointers to the K' (fp16) and V (bf16) slot 0 of batch element b, and
 * the element stride between slots (= heads/world_size * head_dim); committed
 * tokens are slots [0, valid).  For tests and checkpoint dumps. */
DZ_API dz_status dz_cache_view(const dz_ctx* ctx, int32_t b, void** k_slot0, void** v_slot0, int64_t* slot_stride);

/* Copy the fp32 log-sum-exp rows [batch][heads/world_size][n] of the last
 * attend (needs DZ_FLAG_WRITE_LSE) into a caller device buffer on stream. */
DZ_API dz_status dz_copy_lse(dz_ctx* ctx, float* dst, size_t dst_elems, void* stream);

/* Tile map of the last attend as decided by the attention kernel for (batch,
 * head) = (0, 0): host uint8 [n_q_tiles][n_kv_tiles] with tiles of *bm = 256
 * query rows (one CTA pair) x *bn keys (one KV step: 128 with the fixed softmax
 * base, 256 with the online one); 0 SKIP (not
 * computed), 1 PARTIAL (masked per element), 2 FULL (unmasked) -- the
 * encoding of the oracle's classifier.  Synchronous device read (tests). */
DZ_API dz_status dz_get_tile_map(const dz_ctx* ctx, uint8_t* host, size_t cap, int32_t* n_q_tiles, int32_t* n_kv_tiles,
                          int32_t* bm, int32_t* bn);

/* Device times in ms of the last calls (needs DZ_FLAG_PROFILE), measured with
 * CUDA events on the caller's stream: ms[0] attend prologue (K1), ms[1]
 * pre-attention all-to-all, ms[2] attention (K2), ms[3] post all-to-all +
 * unpack, ms[4] attend total, ms[5] last append (K4 + exchange).  Waits for the
 * recorded events (host sync).  Entries not yet recorded are 0. */
DZ_API dz_status dz_profile_last(dz_ctx* ctx, float* ms6);

/* Switches the DZ_FLAG_PROFILE event recording on (default) or off.  An event
 * recorded between two kernels ends their programmatic overlap (each kernel
 * is launched with programmatic stream serialization and may start while its
 * predecessor drains), so throughput runs switch it off and measure the
 * kernels in a separate profiled pass.  DZ_ESTATE without DZ_FLAG_PROFILE. */
DZ_API dz_status dz_profile_enable(dz_ctx* ctx, int32_t on);

/* Releases the context's host state and device workspace (not the caller's
 * buffers).  Safe on NULL. */
DZ_API dz_status dz_destroy(dz_ctx* ctx);

DZ_API const char* dz_status_string(dz_status s);
DZ_API const char* dz_last_error(const dz_ctx* ctx);

/* NCCL plumbing for Ulysses sequence parallelism (one process per GPU).
 * dz_nccl_unique_id fills 128 bytes on rank 0 (broadcast them with the host's
 * own process group); dz_nccl_comm_init creates a communicator on the current
 * device; dz_nccl_comm_destroy frees it. */
DZ_API dz_status dz_nccl_unique_id(void* id128);
DZ_API dz_status dz_nccl_comm_init(int32_t world_size, const void* id128, int32_t rank, void** comm);
DZ_API dz_status dz_nccl_comm_destroy(void* comm);

/* Hang diagnosis: every mbarrier wait in the kernels is bounded (5 s).  A wait
 * that times out records {1, block, warp, barrier smem address, parity, SM id,
 * barrier-block base, 0} and traps, so the launch fails with a CUDA error (seen at
 * the next sync; the context's next call returns DZ_ECUDA and poisons it) instead
 * of hanging the GPU or returning garbage.  In the diagnostics build
 * (libdz_trace.so) the kernel drains instead and this call reads the record.
 * Copies that record (zeros if no timeout) to host8[8]; reset != 0 clears it.
 * Synchronous. */
DZ_API dz_status dz_debug_watchdog(uint32_t* host8, int32_t reset);

/* Effective SM clock under the attention kernel: every attention launch adds, per
 * CTA, its SM's clock64() cycles and %globaltimer nanoseconds between the end of its
 * wait on the predecessor and its exit.  Copies {cycles, ns} (summed over CTAs and
 * launches since the last reset) to host2[2] when host2 != NULL; reset != 0 then
 * zeroes them.  cycles / ns is the mean SM clock in GHz.  Synchronous (device-wide). */
DZ_API dz_status dz_debug_k2_clock(uint64_t* host2, int32_t reset);

/* Pipeline diagnostics: enable != 0 makes later attention launches record a
 * clock() trace of CTA 0's first work unit (MMA waits/issues, softmax S-ready /
 * P-done per KV step, up to 256 steps; layout documented in attention.cu),
 * followed (words 8192 ..) by a per-CTA timeline of up to 160 CTAs x 64 words
 * (globaltimer ns of each work segment's start / end).  host != NULL copies up
 * to n words of the last trace.  Synchronous. */
DZ_API dz_status dz_debug_trace(int32_t enable, uint32_t* host, size_t n);

/* One transfer of the Ulysses all-to-all: this rank sends
 * `bytes` at storage + send_off to rank `peer` and receives `bytes` from it at
 * storage + recv_off (offsets into the caller's cache_storage).  tensor: 0 Q',
 * 1 K', 2 V, 3 O. */
typedef struct {
  int32_t peer;
  int32_t tensor;
  int64_t send_off;
  int64_t recv_off;
  int64_t bytes;
} dz_xfer;

/* The exchange plan the library issues (as one grouped ncclSend/ncclRecv per
 * entry) for an n_tokens chunk in the context's current cache state: phase 0
 * = attend pre-exchange (sequence shard -> head shard of Q', K', V: K'/V land
 * in the cache staging slots), 1 = append pre-exchange (K', V), 2 = attend
 * post-exchange (O head shard -> the receive buffer unpacked by K5).  Copies
 * up to cap entries to out (may be NULL) and returns the entry count, or a
 * negative dz_status.  Host only, no device access: lets host-side tests check
 * the plan with any process-group backend. */
DZ_API int32_t dz_sp_plan(const dz_ctx* ctx, int32_t phase, int32_t n_tokens, dz_xfer* out, int32_t cap);

/* Caller-driven exchange (DZ_FLAG_EXTERNAL_EXCHANGE).  Under SP, dz_attend_chunk,
 * dz_attend_spans and dz_append_kv enqueue their work up to the first all-to-all
 * and return DZ_OK with the exchange pending; every other call except these two
 * returns DZ_ESTATE until the operation completes.  dz_sp_pending copies up to cap
 * transfers of the pending exchange (the dz_sp_plan entries of *phase, offsets
 * into cache_storage) to out and returns their count (0 and *phase = -1 if none).
 * The caller delivers them -- this rank's send block of entry (peer p, tensor t,
 * k-th such entry) is the receive block of p's entry (peer = this rank, t, k-th) --
 * ordered before the next work on `stream`, then calls dz_sp_resume, which
 * enqueues the next stage on stream (attend: the attention, then after exchange 2
 * the unpack; append: the commit).  Lets a caller use its own transport (and the
 * tests run N ranks on one GPU with one device copy per transfer). */
DZ_API int32_t dz_sp_pending(const dz_ctx* ctx, int32_t* phase, dz_xfer* out, int32_t cap);

/* DZ_FLAG_PEER_STORE: storages[p] = rank p's cache_storage as addressable from this process (the
 * peer-mapped pointer on a node; storages[rank] must be this context's own).  Every rank's context
 * must have the same configuration and see the same sequence of calls.  Required before the first
 * compute call (else DZ_ESTATE).  Host only. */
DZ_API dz_status dz_sp_set_peers(dz_ctx* ctx, void* const* storages, int32_t n);
DZ_API dz_status dz_sp_resume(dz_ctx* ctx, void* stream);

/* K5 (the post-exchange unpack) on its own, for tests: recv bf16
 * [world_size][batch][n_local][heads_local][head_dim] -> out bf16
 * [batch][n_local][world_size * heads_local][head_dim], enqueued on stream. */
DZ_API dz_status dz_debug_sp_unpack(const void* recv, void* out, int32_t world_size, int32_t batch, int32_t n_local,
                                    int32_t heads_local, int32_t head_dim, void* stream);

/* Kernels this library has enqueued in this process so far (prologue, RoPE table,
 * attention, unpack), counted on the host at launch: the difference over a region
 * is the number of the library's kernels in it (benchmark evidence). */
DZ_API int64_t dz_kernel_launches(void);

/* Benchmark helper, not part of the path: invalidates the L2 lines of the
 * device buffer buf[0, bytes) without writing them back (PTX discard.global.L2;
 * the buffer's contents become undefined).  bench.py runs it after the 512 MB
 * L2-flush write so that the flush's dirty lines are not written back during the
 * timed step.  bytes must be a multiple of 128 (DZ_EINVAL otherwise); enqueued
 * on `stream`, not counted by dz_kernel_launches. */
DZ_API dz_status dz_debug_l2_discard(void* buf, size_t bytes, void* stream);

/* Number of attention work units (batch x heads/world_size x query-tile pairs)
 * for an n-token chunk; the persistent grid is min(units, SM count). */
DZ_API int32_t dz_attention_units(const dz_ctx* ctx, int32_t n_tokens);

#ifdef __cplusplus
}
#endif
#endif /* DZ_H_ */
