/*
 * libparse — B200-native (sm_100a) hot path of PARSE's parallel prefix
 * verification pass (arxiv 2605.04263).
 *
 * Citations: P:<line> = PAPER.md line (section in parentheses).
 *
 * The pass (§3.2 "Parallel Prefix Verification"): one prefill over a
 * packed sequence = the shared region (prompt + draft y_{1:T}, length N)
 * followed by K appended copies of the chat-template suffix (length S each).
 * Under the prefix-boundary mask, shared-region rows attend causally among
 * themselves; suffix copy k attends to shared keys [0, b_k) and causally to
 * itself, never to another copy.  The verdict logits (l_C, l_I) read at the
 * last row of each copy give the two-way confidence p_k (Eq. p2way,
 * P:530-536), the thresholded verdict and the maximal
 * valid prefix.
 *
 * C ABI: plain pointers and sizes, no C++ types, no exceptions across the
 * boundary.  All device buffers are allocated and owned by the caller; the
 * library never allocates device memory on the hot path.  Work is enqueued
 * on `stream` and the calls return immediately (argument validation is
 * synchronous).  There is NO CPU fallback: a non-sm_100 device returns
 * PARSE_ERR_UNSUPPORTED.
 */
#ifndef PARSE_H_
#define PARSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARSE_VERSION 100 /* 1.0.0 */

#if defined(__GNUC__)
#define PARSE_API __attribute__((visibility("default")))
#else
#define PARSE_API
#endif

typedef enum {
  PARSE_OK = 0,
  PARSE_ERR_INVALID = 1,     /* bad argument; see parse_last_error() */
  PARSE_ERR_UNSUPPORTED = 2, /* valid but not supported here (device, head_dim, ...) */
  PARSE_ERR_CUDA = 3,        /* a CUDA runtime/driver call failed */
  PARSE_ERR_WORKSPACE = 4    /* workspace NULL or smaller than required */
} parse_status_t;

typedef enum {
  PARSE_PREC_BF16 = 0,      /* tcgen05 path: bf16 QK^T and PV, fp32 accumulate, P rounded
                               to bf16, O written as bf16 */
  PARSE_PREC_FP32_DEBUG = 1, /* SIMT path: fp32 scores, fp32 P, O written as fp32 (parity mode) */
  PARSE_PREC_FP8_E4M3 = 2    /* tcgen05 kind::f8f6f4 path: e4m3 Q, K, V with fp32 descales, P
                                rounded to e4m3, fp32 accumulate, O written as bf16; only through
                                parse_verify_attn_fp8 (a variant: the paper's target
                                checkpoints are FP8, but its attention precision is unstated) */
} parse_precision_t;

typedef enum {
  PARSE_RULE_LEADING_RUN = 0, /* k* = largest k with v_k Correct and no Incorrect earlier
                                 (App. A.3) — default */
  PARSE_RULE_MAX_CORRECT = 1  /* k* = max{k : v_k Correct}  (§3.2) */
} parse_rule_t;

/* ------------------------------------------------------------------------ */
/* parse_verify_attn — one attention layer of the packed verification prefill */
/* ------------------------------------------------------------------------ */
/*
 * Shapes (BSHD, head_dim contiguous; strides in ELEMENTS):
 *   Q   [batch][L][num_q_heads][head_dim]   bf16   (already RoPE-rotated)
 *   K,V [batch][L][num_kv_heads][head_dim]  bf16
 *   O   [batch][L][num_q_heads][head_dim]   bf16 (PARSE_PREC_BF16) or fp32 (FP32_DEBUG)
 *   LSE [batch][num_q_heads][L]             fp32, natural log, contiguous (optional)
 * with L = draft_len + num_suffixes * suffix_len.  Packed row t < N is a
 * shared-region token; row N + k*S + s is token s of suffix copy k
 * (appended layout of P:208).  q head h reads kv head h / (Hq/Hkv) (GQA).
 *
 * Visibility (boundaries half-open, 0-indexed):
 *   row t < N            : keys {0..t}
 *   row N + k*S + s      : keys [0, b_k)  U  {N + k*S + s' : s' <= s}
 *                          (tree variant: s' ancestor-or-self of s)
 *
 * Output for row t, head h: O = sum_{j visible} softmax_j(scale * q.k_j) v_j,
 * LSE = log sum_{j visible} exp(scale * q.k_j).  All L rows are computed
 * (shared rows feed later layers of the prefill).
 *
 * Position ids are the caller's job: for model-level equivalence with K
 * standalone passes, suffix k must be rotated at positions b_k .. b_k+S-1
 * (see parse_suffix_positions).
 */
typedef struct {
  int32_t batch;          /* B >= 1 */
  int32_t num_q_heads;    /* Hq >= 1, Hq % Hkv == 0 */
  int32_t num_kv_heads;   /* Hkv >= 1 */
  int32_t head_dim;       /* 64 or 128 */
  int32_t draft_len;      /* N >= 1: shared region (prompt + draft) */
  int32_t num_suffixes;   /* K >= 1 */
  int32_t suffix_len;     /* S >= 1 */
  const int32_t* boundaries; /* HOST, [batch][K] (row stride boundary_batch_stride, 0 => one
                                shared [K] row); 0 <= b_k <= N; any order accepted here.
                                Read during the call, not retained. */
  int64_t boundary_batch_stride;
  const int16_t* tree_parent; /* HOST, [S] or NULL (NULL => causal suffix). parent[s] < s or -1;
                                 requires S <= 64. Shared by all copies. */
  float softmax_scale;    /* <= 0 => 1/sqrt(head_dim) */
  int32_t precision;      /* parse_precision_t */
  int64_t q_strides[3];   /* batch, token, head strides of Q (elements); multiples of 8 */
  int64_t k_strides[3];
  int64_t v_strides[3];
  int64_t o_strides[3];
} parse_attn_desc_t;

/* Bytes of device workspace parse_verify_attn needs for this descriptor
 * (schedule + boundary/tree tables).  Returns PARSE_ERR_INVALID for a bad
 * descriptor. */
PARSE_API parse_status_t parse_verify_attn_workspace_size(const parse_attn_desc_t* desc, size_t* bytes);

/* Enqueue the masked attention on `stream`.  q/k/v/o/lse/workspace are
 * DEVICE pointers (16-byte aligned); lse may be NULL.  The workspace is
 * written by the call (schedule upload) and must not be shared by calls in
 * flight on different streams.  The schedule (tile classification, SURVEY
 * §8 a2) is built on the host once per distinct problem (geometry +
 * boundaries + tree, per device) and cached by libparse (LRU, at most 16
 * problems / 256 MB): a pinned host copy and a device copy that libparse
 * allocates (cudaMalloc) and fills once on `stream`; every call copies the
 * device copy into the workspace with a small kernel on `stream`, so a
 * repeated problem costs no host rebuild and no copy-engine transfer.  Not
 * capturable into a CUDA graph (a cached image can be evicted): use a plan.
 * Errors: PARSE_ERR_INVALID (descriptor/pointers), PARSE_ERR_WORKSPACE,
 * PARSE_ERR_UNSUPPORTED (not sm_100, head_dim), PARSE_ERR_CUDA (launch). */
PARSE_API parse_status_t parse_verify_attn(const parse_attn_desc_t* desc, const void* q, const void* k,
                                 const void* v, void* o, float* lse, void* workspace,
                                 size_t workspace_bytes, void* stream /* cudaStream_t */);

/* FP8 variant of parse_verify_attn (desc->precision = PARSE_PREC_FP8_E4M3):
 * q, k, v are e4m3 (1 byte per element, same BSHD layout; strides in elements
 * = bytes, multiples of 16) holding Q/descale_q, K/descale_k, V/descale_v
 * (per-tensor descale factors, positive and finite).  It computes the same
 * masked attention of the dequantized tensors: scores = (q.k) * descale_q *
 * descale_k * softmax_scale, P rounded to e4m3 before PV (scaled by 2^4
 * internally, cancelled by the normaliser), O = descale_v * (P V) / l written
 * as bf16, LSE (optional) as parse_verify_attn.  head_dim must be 128 (else
 * PARSE_ERR_UNSUPPORTED); ragged / paged batches: parse_verify_attn_varlen_fp8.  Workspace as parse_verify_attn_workspace_size for
 * this desc.  Accuracy: per output element |dO| <= 2^-4 * max_j |V_j| (the
 * e4m3 rounding of P, relative 2^-4) + bf16 rounding of O. */
PARSE_API parse_status_t parse_verify_attn_fp8(const parse_attn_desc_t* desc, const void* q, const void* k,
                                               const void* v, float descale_q, float descale_k, float descale_v,
                                               void* o, float* lse, void* workspace, size_t workspace_bytes,
                                               void* stream /* cudaStream_t */);

/* Plans (serving / CUDA graphs): the schedule of a descriptor is built and
 * copied into `workspace` once (plan_create, enqueued on `stream`); each
 * plan_run then only encodes the tensor maps on the host, zeroes the work
 * counter (cudaMemsetAsync) and launches, so it can be captured into a CUDA
 * graph and replayed, and one plan serves every layer of a verification
 * prefill with the same geometry.  The workspace (size from
 * parse_verify_attn_workspace_size) belongs to the plan until destroy and
 * must stay alive; runs of one plan must not overlap (one work counter).
 * q/k/v/o/lse of a run must have the strides given in the descriptor.
 * precision: PARSE_PREC_BF16 or PARSE_PREC_FP32_DEBUG (else UNSUPPORTED).
 * Errors as parse_verify_attn. */
typedef struct parse_attn_plan_s* parse_attn_plan_t;
PARSE_API parse_status_t parse_verify_attn_plan_create(const parse_attn_desc_t* desc, void* workspace,
                                                       size_t workspace_bytes, void* stream, parse_attn_plan_t* plan);
PARSE_API parse_status_t parse_verify_attn_plan_run(parse_attn_plan_t plan, const void* q, const void* k,
                                                    const void* v, void* o, float* lse, void* stream);
PARSE_API parse_status_t parse_verify_attn_plan_destroy(parse_attn_plan_t plan);

/* Introspection (host only; no GPU needed): the tile schedule the bf16 path
 * launches for this descriptor.  Work item = up to two
 * 128-row Q tiles of one request and KV-head group with identical row
 * visibility; row r of tile i is packed token t0 + r / hpt, q head
 * h0 + i*hpt + r % hpt, stored iff token < t_end.  It reads the KV tiles at
 * keys [128j, 128j+128), j < n_draft, and [self_lo + 128j, ...), j < n_self.
 * flags: bits 0-7 = hpt (q heads packed per tile), bit 8 = two Q tiles.
 * Items are in launch (dynamic hand-out) order.  With items == NULL only
 * *n_items is written; otherwise up to `capacity` items are copied. */
typedef struct {
  int32_t b, h0, t0, t_end, self_lo, n_draft, n_self, flags;
} parse_work_item_t;
PARSE_API parse_status_t parse_verify_attn_schedule(const parse_attn_desc_t* desc, parse_work_item_t* items,
                                                    size_t capacity, size_t* n_items);

/* Introspection (host only): the work units of the 2-CTA cluster launch
 * (dense K/V, DESIGN §6.1 "K/V multicast"), as pairs (x, y) of indices into
 * the parse_verify_attn_schedule list: CTA 0 runs item x, CTA 1 runs
 *   y >= 0   item y, which reads the same K/V tiles as x: each tile is read
 *            from L2 once for the pair and multicast into both CTAs;
 *   y <= -2  item -y-2, with the same step and Q-tile counts (own K/V);
 *   y == -1  item x again, not stored (no partner).
 * Units are in launch order.  units: int32 [capacity][2] or NULL (only
 * *n_units is written).  Errors: PARSE_ERR_INVALID. */
PARSE_API parse_status_t parse_verify_attn_units(const parse_attn_desc_t* desc, int32_t* units, size_t capacity,
                                                 size_t* n_units);

/* ------------------------------------------------------------------------ */
/* parse_verify_attn_varlen — ragged and paged batches         */
/* ------------------------------------------------------------------------ */
/*
 * The operation of parse_verify_attn, with a shared length N_b and a suffix
 * count K_b per request b: a serving batch of heterogeneous drafts (P:180,
 * P:609-617).  The suffix length S is one per call: it is the judge's
 * chat-template suffix, the same for every request.  The packed
 * sequence of request b has L_b = N_b + K_b*S rows, laid out as in
 * parse_verify_attn.  K_b = 1 with b_0 = N_b is the full-verify pass pi_F
 * (Alg. 2 Stage 2); K_b = 0 is a plain causal prefill.
 *
 * Q and O are packed-row ("THD") tensors: packed row t of request b is row
 * row_offsets[b] + t of Q [total_rows][num_q_heads][head_dim] (q_strides =
 * {row, head} in elements), and likewise of O.  LSE (optional, fp32) is
 * [num_q_heads][total_rows]: column row_offsets[b] + t.  Row ranges of
 * different requests must not overlap.
 *
 * K and V are either
 *   contiguous (page_size == 0): packed key t of request b is row
 *     kv_row_offsets[b] + t of K [kv_total_rows][num_kv_heads][head_dim]
 *     (k_strides = {row, head, unused}); kv_row_offsets NULL => row_offsets
 *     and kv_total_rows = total_rows; or
 *   paged (page_size a power of two, 16 <= page_size): a pool
 *     [num_pages][page_size][num_kv_heads][head_dim] (k_strides = {page, row,
 *     head}) as a serving engine's KV cache holds it; packed key t of request
 *     b is row t % page_size of page block_table[b*block_table_stride +
 *     t / page_size] (block_table: DEVICE int32, ceil(L_b / page_size) entries
 *     used per request).  An entry outside [0, num_pages) reads as zeros.
 *     Pool rows past L_b in a request's last page must hold finite values
 *     (they are read, masked out, and multiplied by a zero weight).
 *
 * Boundaries are HOST, flat: request b's K_b values start at index
 * sum_{c<b} K_c, each in [0, N_b].  Other fields as parse_attn_desc_t.
 * Errors as parse_verify_attn; also PARSE_ERR_INVALID for inconsistent
 * offsets / page parameters.
 */
typedef struct {
  int32_t batch;              /* B >= 1 */
  int32_t num_q_heads;        /* Hq, Hq % Hkv == 0 */
  int32_t num_kv_heads;       /* Hkv */
  int32_t head_dim;           /* 64 or 128 */
  int32_t suffix_len;         /* S >= 1 */
  const int32_t* draft_lens;  /* HOST [B]: N_b >= 1 */
  const int32_t* num_suffixes; /* HOST [B]: K_b >= 0 */
  const int32_t* boundaries;  /* HOST, flat, sum_b K_b entries */
  const int16_t* tree_parent; /* HOST [S] or NULL, as parse_attn_desc_t */
  float softmax_scale;        /* <= 0 => 1/sqrt(head_dim) */
  int32_t precision;          /* parse_precision_t */
  const int64_t* row_offsets; /* HOST [B]: first Q/O row of each request */
  int64_t total_rows;         /* rows of Q, O and LSE; row_offsets[b] + L_b <= total_rows < 2^31 */
  const int64_t* kv_row_offsets; /* HOST [B] (contiguous K/V) or NULL */
  int64_t kv_total_rows;      /* contiguous K/V rows (ignored when kv_row_offsets is NULL) */
  int32_t page_size;          /* 0 = contiguous K/V; else paged */
  int32_t num_pages;          /* paged: pool size */
  const int32_t* block_table; /* paged: DEVICE [B][block_table_stride] */
  int32_t block_table_stride;
  int64_t q_strides[2];       /* row, head (elements; multiples of 8) */
  int64_t k_strides[3];       /* contiguous: row, head, -; paged: page, row, head */
  int64_t v_strides[3];
  int64_t o_strides[2];
} parse_varlen_desc_t;

PARSE_API parse_status_t parse_verify_attn_varlen_workspace_size(const parse_varlen_desc_t* desc, size_t* bytes);
PARSE_API parse_status_t parse_verify_attn_varlen(const parse_varlen_desc_t* desc, const void* q, const void* k,
                                                  const void* v, void* o, float* lse, void* workspace,
                                                  size_t workspace_bytes, void* stream /* cudaStream_t */);
/* FP8 variant of parse_verify_attn_varlen (desc->precision = PARSE_PREC_FP8_E4M3):
 * e4m3 Q/K/V (packed rows or an e4m3 page pool), per-tensor descales, head_dim
 * 128, strides multiples of 16 elements; otherwise as parse_verify_attn_fp8. */
PARSE_API parse_status_t parse_verify_attn_varlen_fp8(const parse_varlen_desc_t* desc, const void* q, const void* k,
                                                      const void* v, float descale_q, float descale_k,
                                                      float descale_v, void* o, float* lse, void* workspace,
                                                      size_t workspace_bytes, void* stream /* cudaStream_t */);
/* Host-only introspection of the varlen schedule (as parse_verify_attn_schedule;
 * t0 / t_end / self_lo are request-local packed rows). */
PARSE_API parse_status_t parse_verify_attn_varlen_schedule(const parse_varlen_desc_t* desc, parse_work_item_t* items,
                                                           size_t capacity, size_t* n_items);

/* ------------------------------------------------------------------------ */
/* parse_select_prefix — verdict readout + maximal valid prefix                 */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t n_incorrect;            /* #{k : v_k Incorrect}        (rho rule)  */
  int32_t trailing_incorrect_run; /* Incorrect run at the tail   (kappa rule) */
  int32_t n_below_aux;            /* #{k : p_k < aux_threshold}     */
  float min_score;                /* min_k p_k (NaNs ignored)    (P:705 p_min)      */
} parse_prefix_stats_t;

typedef struct {
  int32_t batch;               /* B >= 1 */
  int32_t num_prefixes;        /* K, 1 <= K <= 65536 */
  const void* verdict_logits;  /* DEVICE. Element (b, k): l_C at
                                  base + b*logits_batch_stride + k*logits_prefix_stride,
                                  l_I at that + logits_pair_stride (elements).  fp32, or
                                  bf16 when logits_bf16 = 1.  A strided view into full-vocab
                                  logits rows (pair stride = id_I - id_C) is allowed. */
  int32_t logits_bf16;
  int64_t logits_batch_stride;
  int64_t logits_prefix_stride;
  int64_t logits_pair_stride;
  const int32_t* boundaries;   /* DEVICE, [B][K] (stride boundary_batch_stride, 0 => shared),
                                  t_k in draft coordinates, used for accepted_len */
  int64_t boundary_batch_stride;
  double threshold;            /* tau in [0,1]: v_k Correct iff raw Correct and p_k >= tau,
                                  decided as l_C - l_I >= log(tau) - log1p(-tau) in fp64 */
  double aux_threshold;        /* tau for n_below_aux (e.g. tau_C^rx); < 0 => not counted */
  double eta;                  /* rollback in chunks, >= 0 (Eq. adopted) */
  int32_t rule;                /* parse_rule_t */
  int32_t tie_is_correct;      /* 1: l_C == l_I is a raw Correct (Alg. 2); 0: Incorrect */
} parse_select_desc_t;

/* Per request b (all outputs DEVICE, caller-owned):
 *   scores[b][k]     = p_k = exp(l_C)/(exp(l_C)+exp(l_I)) (Eq. p2way), fp64 rounded to fp32
 *   k_star[b]        = selected chunk index per `rule`, -1 if none
 *   accepted_len[b]  = L* = t_m with m = floor(max(0, k*+1-eta)), 0 if m = 0
 *                      (equals Eq. adopted min(T, Delta*m) for uniform boundaries)
 *   stats[b]         (nullable) counts above
 *   device_status    (nullable, one int32, OR-ed): bit0 = a non-finite logit was seen
 *                    (such a pair is treated as Incorrect).
 * Graph-capturable (no host work beyond validation). */
PARSE_API parse_status_t parse_select_prefix(const parse_select_desc_t* desc, int32_t* accepted_len,
                                   int32_t* k_star, float* scores, parse_prefix_stats_t* stats,
                                   int32_t* device_status, void* stream /* cudaStream_t */);

/* ------------------------------------------------------------------------ */
/* parse_select_prefix fused with the verdict all-gather (SURVEY §8 e)        */
/* ------------------------------------------------------------------------ */
/*
 * Multi-GPU runs shard requests across ranks (requests and suffix copies
 * are independent); the only exchange is every rank's selection.  This call
 * computes parse_select_prefix for the rank's `batch` requests and stores the
 * results straight into slot `rank` of every rank's gather buffer over peer
 * memory (NVLink P2P / CUDA IPC mappings), then raises this rank's flag in
 * every buffer and returns (on the device) once all `world` ranks' slots have
 * landed in its own buffer: one kernel, no separate collective.
 *
 * Gather buffer (one per rank, parse_peer_buffer_bytes bytes, ZEROED before
 * first use, identical batch / K on every rank):
 *   [header 256 B: flags uint32[world] at 0, counters at 128]
 *   [3 sets x world slots of batch*(2+K) int32]; set = epoch % 3; slot r =
 *   accepted_len[batch] | k_star[batch] | scores[batch][K] (fp32 bits), the
 *   values parse_select_prefix returns (equal rule / threshold semantics).
 * peer_buffers: DEVICE array [world] of every rank's buffer as mapped in this
 *   process (own buffer at [rank]; others from parse_peer_import).
 * epoch: 1, 2, 3, ... one per call, the same on every rank.  The results of
 *   call `epoch` stay valid in set epoch % 3 until THIS rank's call epoch + 2
 *   executes: a peer finishes call e only after every rank's call e has raised
 *   its flag, so it can be at most one call ahead of this rank (it may already
 *   be writing set (epoch + 1) % 3 while this rank reads set epoch % 3).
 *   Consume them on `stream` (or a stream ordered before call epoch + 2).
 * stats / device_status as parse_select_prefix (local, nullable).
 * A rank that never makes the matching call leaves the others waiting: the
 *   kernel traps after ~2^34 cycles (PARSE_ERR_CUDA on the next sync).
 */
typedef struct {
  unsigned char reserved[64];   /* cudaIpcMemHandle_t bytes */
} parse_ipc_handle_t;

PARSE_API parse_status_t parse_peer_buffer_bytes(int32_t batch, int32_t num_prefixes, int32_t world,
                                                 size_t* bytes);
/* IPC handle + byte offset of a device pointer inside its cudaMalloc allocation. */
PARSE_API parse_status_t parse_peer_export(const void* dev_ptr, parse_ipc_handle_t* handle, uint64_t* offset);
/* Map another process's buffer (handle, offset from parse_peer_export). */
PARSE_API parse_status_t parse_peer_import(const parse_ipc_handle_t* handle, uint64_t offset, void** dev_ptr);
/* Unmap a pointer returned by parse_peer_import. */
PARSE_API parse_status_t parse_peer_close(void* dev_ptr);
PARSE_API parse_status_t parse_select_prefix_allgather(const parse_select_desc_t* desc, void* const* peer_buffers,
                                                       int32_t rank, int32_t world, uint32_t epoch,
                                                       parse_prefix_stats_t* stats, int32_t* device_status,
                                                       void* stream /* cudaStream_t */);

/* ------------------------------------------------------------------------ */
/* Verdict logits from the judge ("read the verifier   */
/* logits l_C, l_I at the judgment position")                       */
/* ------------------------------------------------------------------------ */
/* Reading R17: the verdict logits are the target model's LM-head logits of the
 * Correct / Incorrect tokens at the judgment row of each copy:
 *   y = RMSNorm(h) = h / sqrt(mean(h^2) + eps) * gamma,   l_C = y . W_U[C],  l_I = y . W_U[I]
 * (the standard final norm + LM head of the Qwen3 / GLM judges), in fp32 from
 * bf16 inputs, fused into one pass over h. */
typedef struct {
  int32_t batch;              /* B >= 1 */
  int32_t num_prefixes;       /* K >= 1 */
  int32_t hidden;             /* hidden size, a multiple of 8 (Qwen3-235B: 4096) */
  const void* hidden_states;  /* DEVICE bf16; row (b, k) starts at b*hs_batch_stride + k*hs_prefix_stride
                                 (elements; the row itself contiguous).  Pointing at the first
                                 judgment row of a [B][L][hidden] tensor with prefix stride S*hidden
                                 reads the judgment rows in place. 16-byte aligned rows. */
  int64_t hs_batch_stride;
  int64_t hs_prefix_stride;
  const void* norm_weight;    /* DEVICE bf16 [hidden]: RMSNorm gamma */
  const void* verdict_rows;   /* DEVICE bf16 [2][hidden]: W_U rows of the Correct, Incorrect tokens */
  float eps;                  /* RMSNorm epsilon (> 0) */
} parse_verdict_head_desc_t;

/* logits: DEVICE fp32 [B][K][2] = (l_C, l_I), ready for parse_select_prefix. */
PARSE_API parse_status_t parse_verdict_logits(const parse_verdict_head_desc_t* desc, float* logits,
                                              void* stream /* cudaStream_t */);

/* parse_verdict_select — parse_verdict_logits followed by parse_select_prefix
 * in ONE launch (hidden states -> verdict logits -> maximal valid prefix; the
 * two passes of Eq. p2way / Eq. adopted, with reading
 * R17 for the logits).  Each CTA computes one judgment row's (l_C, l_I) and
 * writes it to `logits`; the CTA finishing the last row of request b then runs
 * b's selection (one warp, the parse_select_prefix scan).  Results equal the
 * two calls' bit for bit.
 *   head: as parse_verdict_logits.  sel: as parse_select_prefix, except that
 *     verdict_logits, logits_bf16 and the three logits strides are ignored
 *     (the selection reads `logits`); batch / num_prefixes must equal head's.
 *   logits: DEVICE fp32 [B][K][2] (written; also an output).
 *   counters: DEVICE uint32 [B] workspace, ZERO before the first call; every
 *     call leaves it zero.  Not shared by concurrent calls.
 *   accepted_len, k_star, scores, stats, device_status: as parse_select_prefix.
 */
PARSE_API parse_status_t parse_verdict_select(const parse_verdict_head_desc_t* head, const parse_select_desc_t* sel,
                                              float* logits, uint32_t* counters, int32_t* accepted_len,
                                              int32_t* k_star, float* scores, parse_prefix_stats_t* stats,
                                              int32_t* device_status, void* stream /* cudaStream_t */);

/* Full-vocabulary readout of the judgment rows: per row, lse = log sum_v exp(z_v)
 * (the softmax normaliser), the pair (z_C, z_I), and the verdict mass
 * P(C) + P(I) = exp(z_C - lse) + exp(z_I - lse) — how much of the judge's
 * next-token distribution sits on the two verdict tokens (the "format
 * mismatch" of P:202-206 shows up as a small mass). */
typedef struct {
  int32_t batch, num_prefixes;
  int32_t vocab;              /* V >= 1, a multiple of 8 (bf16) / 4 (fp32) */
  const void* vocab_logits;   /* DEVICE [B][K][V] rows (row contiguous, 16-byte aligned), strides in elements */
  int32_t logits_bf16;        /* 1 = bf16, 0 = fp32 */
  int64_t batch_stride, prefix_stride;
  int32_t id_correct, id_incorrect;  /* token ids in [0, V) */
} parse_vocab_readout_desc_t;

/* Outputs (DEVICE fp32): pair_logits [B][K][2], lse [B][K] (nullable), verdict_mass [B][K] (nullable). */
PARSE_API parse_status_t parse_vocab_readout(const parse_vocab_readout_desc_t* desc, float* pair_logits, float* lse,
                                             float* verdict_mass, void* stream /* cudaStream_t */);

/* Host helper: positions[k][s] = boundaries[k] + s (suffix position ids, see above). */
PARSE_API parse_status_t parse_suffix_positions(const int32_t* boundaries, int32_t num_suffixes,
                                      int32_t suffix_len, int32_t* positions);

/* Thread-local message describing the last non-OK status ("" if none). */
PARSE_API const char* parse_last_error(void);

/* PARSE_VERSION of the loaded library. */
PARSE_API int parse_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARSE_H_ */
