// Internal interfaces between the C-ABI layer (api.cu), the host schedule
// builder (schedule.cpp) and the kernels (attn_sm100.cu, attn_fp32.cu,
// select.cu).  Not part of the public ABI.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/parse.h"

namespace parse {

constexpr int kTile = 128;       // Q rows per tile = KV keys per tile
constexpr int kMaxTreeS = 64;    // tree masks are uint64 ancestor rows

// One unit of persistent-kernel work: nq (1 or 2) Q tiles of 128 rows that
// share one KV-head group, one request and one visibility pattern, plus the
// KV tiles they need.  Row r of Q tile i maps to packed token
// t0 + r / hpt and q head h0 + i*hpt + r % hpt.
//   draft segment: KV tiles at keys 128*j, j < n_draft
//   self  segment: KV tiles at keys self_lo + 128*j, j < n_self
// Rows with token >= t_end (token-major tiles) are computed but not stored.
// flags bit 9 ("copy pair"): tile 1 is the NEXT suffix copy (tokens + S) with
// the same heads, instead of the next head-pack of the same copy.
struct alignas(16) WorkItem {
  int32_t b;        // request
  int32_t h0;       // first q head of tile 0
  int32_t t0;       // first packed token
  int32_t t_end;    // one past the last stored token (token-major); t0 + S for head-packed
  int32_t self_lo;  // first key of the self segment
  int32_t n_draft;  // # draft-segment KV tiles
  int32_t n_self;   // # self-segment KV tiles
  int32_t flags;    // bits 0-7: hpt; bit 8: nq == 2; bit 9: tile 1 = next suffix copy
};
static_assert(sizeof(WorkItem) == 32, "WorkItem is 32 bytes");

// Per-request geometry (device copy: ReqDesc).  Dense batches
// (parse_verify_attn) have N_b = N, K_b = K for every b, row offsets 0 and
// TMA batch coordinate b; ragged batches (parse_verify_attn_varlen) address
// one packed-row tensor (batch coordinate 0) at per-request row offsets.
struct Problem {
  int B, Hq, Hkv, D, S;
  int N, K, L;                    // maxima over the requests (dense: the values)
  std::vector<int32_t> Nb, Kb;    // [B]
  std::vector<int32_t> bnd_off;   // [B] first index of request b in bnd
  std::vector<int32_t> bnd;       // flat boundaries
  std::vector<int32_t> q_row0, kv_row0;  // [B] (dense: 0)
  bool varlen = false;
  int self_align = 1;             // paged K/V: self tiles start on 128-key (page-aligned) boundaries
  bool tree;
  std::vector<uint64_t> anc;   // [S] ancestor-or-self bitmasks (tree only)
  float scale;
  int Lb(int b) const { return Nb[b] + Kb[b] * S; }
  int32_t bndv(int b, int k) const { return bnd[size_t(bnd_off[b]) + k]; }
};

struct alignas(16) ReqDesc {
  int32_t N, L, K, bnd_off;   // shared length, packed length, # copies, boundaries at bnd[bnd_off..]
  int32_t q_row0, kv_row0;    // first Q/O row and first K/V row (contiguous K/V)
  int32_t bcoord;             // TMA batch coordinate / batch index of the dense layout
  int32_t pad;
};
static_assert(sizeof(ReqDesc) == 32, "ReqDesc is 32 bytes");

// Validate a descriptor and produce a Problem.  Returns PARSE_OK or
// PARSE_ERR_INVALID / PARSE_ERR_UNSUPPORTED with *err set.
parse_status_t make_problem(const parse_attn_desc_t* d, Problem* p, std::string* err);
parse_status_t make_problem_varlen(const parse_varlen_desc_t* d, Problem* p, std::string* err);

// Head-packing factor for suffix tiles: hpt = 128/S q heads of
// one group per tile when S | 128 and hpt | (Hq/Hkv); 0 = token-major.
int suffix_heads_per_tile(const Problem& p);

// Build the LPT-ordered work list (largest KV-tile count first).
void build_schedule(const Problem& p, std::vector<WorkItem>* items);
size_t count_schedule(const Problem& p);

// Workspace layout (all offsets 256-byte aligned).
struct WorkspaceLayout {
  size_t counter_off, req_off, bnd_off, anc_off, items_off, pairs_off, total;
  size_t n_items;
};
// 2-SM kernel work list: pairs of schedule items with the same request, KV
// group, K/V sequence and tile count (one per CTA of a cluster); y = -1: the
// item runs alone (the peer CTA recomputes it without storing).
void build_pairs(const std::vector<WorkItem>& items, int Hkv, int Hq, std::vector<int2>* pairs);
// 2-CTA cluster kernel work list (schedule.cpp): pairs of items walking the
// same K/V tiles (multicast), or the same number of steps (lockstep), or one
// item recomputed unstored by the second CTA (y = -1); see build_units.
void build_units(const std::vector<WorkItem>& items, int Hkv, int Hq, std::vector<int2>* units);
WorkspaceLayout workspace_layout(const Problem& p, bool need_items);

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device property of a
// kernel: opt in once per (kernel, device).  Concurrent first launches may
// both set it (idempotent); no lock is needed.
template <auto kKernel>
cudaError_t opt_in_smem(int bytes) {
  static std::atomic<int> done[64];   // zero-initialised: bytes opted in per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (done[dev].load(std::memory_order_acquire) >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[dev].store(bytes, std::memory_order_release);
  return e;
}

// ------------------------------ kernels -----------------------------------
struct AttnParams {
  const ReqDesc* req;      // device [B]
  const int32_t* bnd;      // device, flat (ReqDesc::bnd_off)
  const uint64_t* anc;     // device [S] or nullptr (causal suffix)
  const WorkItem* items;   // device
  int32_t n_items;
  const int2* work;        // 2-CTA cluster kernel: units (build_units); 2-SM variant: pairs (build_pairs)
  int32_t n_work;
  int32_t* counter;        // device, zero at launch: next item to hand out
  int32_t B, Hq, Hkv, S;
  int32_t dense_N, dense_K, dense_L;   // dense batch: every ReqDesc is implied by these (no req load); 0 = varlen
  float scale_log2;        // softmax_scale * log2(e) (FP8: times the Q and K descales)
  float o_scale;           // multiplies O at the epilogue (FP8: the V descale; else 1)
  // paged K/V (page_log2 > 0): key t of request b at row t & (2^page_log2 - 1)
  // of page block_table[b * bt_stride + (t >> page_log2)]
  int32_t page_log2, num_pages, bt_stride;
  const int32_t* block_table;
  void* o;                 // bf16
  float* lse;              // nullable; [bcoord * lse_sb + h * lse_sh + q_row0 + t]
  int64_t lse_sb, lse_sh;
  long long* trace;        // debug timeline (PARSE_TRACE builds only), else nullptr
  int64_t o_s0, o_s1, o_s2;
  int32_t o_v8;            // O base and strides 32-byte aligned: 256-bit epilogue stores
};

cudaError_t launch_attn_sm100(const AttnParams& prm, int D, bool fp8, bool cluster, const CUtensorMap& tm_q_tok,
                              const CUtensorMap& tm_q_pack, const CUtensorMap& tm_k,
                              const CUtensorMap& tm_v,
                              int num_sms, cudaStream_t stream);

// CTA-pair (cta_group::2) bf16 kernel, head_dim 128, dense or packed-row K/V
// (tm_k64: K map with 64-key boxes): one M = 256 item per cluster, S and P
// double-buffered in TMEM.
cudaError_t launch_attn_pair(const AttnParams& prm, const CUtensorMap& tm_q_tok, const CUtensorMap& tm_q_pack,
                             const CUtensorMap& tm_k64, const CUtensorMap& tm_v, int num_sms, cudaStream_t stream);

// 2-SM (cta_group::2) bf16 kernel, head_dim 128, dense or packed-row K/V
// (tm_k64: K map with 64-key boxes).
cudaError_t launch_attn_sm100_2sm(const AttnParams& prm, const CUtensorMap& tm_q_tok, const CUtensorMap& tm_q_pack,
                                  const CUtensorMap& tm_k64, const CUtensorMap& tm_v, int num_sms, cudaStream_t stream);

struct AttnFp32Params {
  const uint16_t* q; const uint16_t* k; const uint16_t* v;
  float* o; float* lse;
  const ReqDesc* req; const int32_t* bnd; const uint64_t* anc;
  int32_t B, Hq, Hkv, D, S, Lmax;
  float scale;
  int32_t page_log2, num_pages, bt_stride;   // paged K/V as AttnParams
  const int32_t* block_table;
  int64_t lse_sb, lse_sh;
  // element strides; K/V: contiguous {batch, row, head}, paged {page, row, head}
  int64_t q_s0, q_s1, q_s2, k_s0, k_s1, k_s2, v_s0, v_s1, v_s2, o_s0, o_s1, o_s2;
};
cudaError_t launch_attn_fp32(const AttnFp32Params& prm, cudaStream_t stream);

struct SelectParams {
  const void* logits; int32_t bf16;
  int64_t ls_b, ls_k, ls_pair;
  const int32_t* bnd; int64_t bnd_s;
  int32_t B, K;
  double theta, theta_aux; int32_t use_aux;
  double eta; int32_t rule, tie;
  int32_t* accepted; int32_t* kstar; float* scores; parse_prefix_stats_t* stats;
  int32_t* status;
  // fused all-gather over peer memory (parse_select_prefix_allgather); peers == nullptr: plain select.
  // peers[q] = rank q's gather buffer as mapped in this process: [header kPeerHeader B | 3 sets x world
  // slots of slot_words int32], slot = [accepted_len (B) | k_star (B) | scores (B x K, fp32 bits)].
  uint8_t* const* peers;
  int32_t rank, world, set;
  uint32_t epoch;
  int64_t slot_words;
};
constexpr int kPeerHeader = 256;   // flags[32] (uint32) at 0, arrival counters[2] at 128
constexpr int kPeerMaxWorld = 32;
// Result sets rotate by epoch % 3: a peer can run at most one call ahead of
// this rank's latest executed call, so call e's set is rewritten no earlier
// than this rank's call e + 2 executes (include/parse.h).
constexpr int kPeerSets = 3;
cudaError_t launch_select(const SelectParams& prm, cudaStream_t stream);

struct VerdictHeadParams {
  const uint16_t* h; const uint16_t* g; const uint16_t* w;   // bf16 bits
  int64_t hs_b, hs_k;
  int32_t B, K, H;
  float eps;
  float* out;                                                // [B][K][2]
};
cudaError_t launch_verdict_head(const VerdictHeadParams& p, cudaStream_t stream);
// fused verdict head + selection (sp.logits = hp.out, fp32 [B][K][2]);
// counters: [B] uint32, zero on entry, left zero
cudaError_t launch_verdict_select(const VerdictHeadParams& hp, const SelectParams& sp, uint32_t* counters,
                                  cudaStream_t stream);

struct VocabReadoutParams {
  const void* z; int32_t bf16;
  int64_t s_b, s_k;
  int32_t B, K, V, id_c, id_i;
  float* pair; float* lse; float* mass;
};
cudaError_t launch_vocab_readout(const VocabReadoutParams& p, cudaStream_t stream);

}  // namespace parse
