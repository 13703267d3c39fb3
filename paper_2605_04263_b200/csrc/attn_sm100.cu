// parse_verify_attn, tensor-core path (bf16, and the e4m3 variant of
// parse_verify_attn_fp8): persistent warp-specialised tcgen05 kernel for
// sm_100a (SURVEY §8 a2-a6, f2 paged K/V, f4 FP8).
//
// What it computes (§3.2): masked attention over the packed sequence
// [shared region (N rows) | K appended suffix copies (S rows each)] where
// shared rows are causal, suffix copy k sees shared keys [0, b_k) plus itself
// causally (or its tree ancestors), and copies never see each other.
//
// Structure (one CTA per SM, 384 threads; CTAs paired into 2-CTA clusters
// that multicast K/V tiles, kCl = 2):
//   warp 0      TMA producer: Q tiles, then K_j / V_j tiles into an smem ring
//   warps 1, 3  MMA issuers for Q tiles 0 / 1 (one elected thread each):
//               S_i = Q_i K_j^T (SS, fp32 in TMEM); O_i += P_i V_j (TS: P from
//               TMEM, V from smem)
//   warp 2      TMEM allocator (512 columns: S | P0 | P1 | O0 | O1)
//   warps 4-7   softmax warpgroup for Q tile 0 (thread = row = TMEM lane)
//   warps 8-11  softmax warpgroup for Q tile 1
// One S buffer serves both Q tiles in turn (QK_0(j), QK_1(j), QK_0(j+1), ...):
// a tile's QK^T is issued as soon as the other tile's softmax has copied its
// S into registers (s_free), and P lives in its own TMEM columns, so QK^T(j+1)
// no longer waits for PV(j) to have read P(j) ("one S buffer").
// A work item holds up to two Q tiles with the same rows' visibility (two
// q heads, or two head-packs, of one KV group), so every K/V tile brought
// into shared memory is used by both.  The north_star's "each draft K/V tile
// is loaded once and shared by every suffix whose boundary covers it" is met
// as DESIGN.md reading R20 states it: once from HBM (group-major item order,
// K/V evict-last: DRAM bytes = algorithmic bytes), once from L2 per 2-CTA
// cluster (kCl = 2: two items with the same K/V walk, each CTA loading half
// of every tile's rows multicast into both), shared in shared memory by each
// item's two Q tiles, and through L2 by the other items of the group.
// The softmax is online with a lazy rescale: O is rescaled in TMEM only when
// a row max grows by more than 2^8 (log2 units) over the max in use.  The
// epilogue writes O with 256-bit stores (whole L2 sectors).
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace parse {
using namespace parse_sm100;

namespace {

constexpr int kThreads = 384;
// Optional softmax ping-pong between the two Q tiles (named-barrier turn
// taking).  Measured on B200 it is slower than letting the two warpgroups
// overlap (DESIGN §6.1 exploration table), so it is off unless built with
// PARSE_PINGPONG=1.
#ifndef PARSE_PINGPONG
#define PP(...)
#else
#define PP(...) __VA_ARGS__
#endif

#ifdef PARSE_TRACE
#define TR(cond, base, step, e) \
  if ((cond) && blockIdx.x == 0 && prm.trace && (step) < 1024) prm.trace[(base) + (step) * 8 + (e)] = clock64();
// MMA-group completion probes (CTA 0): the MMA warps commit probe[i] after
// every QK^T / PV group, the idle allocator warp timestamps each completion
// into trace[57344 + 4096 i + k] (tools/trace_attn.py).
#define TRP(...) __VA_ARGS__
#else
#define TR(cond, base, step, e)
#define TRP(...)
#endif
#ifdef PARSE_CTASTAT
// per-CTA accounting: [start ns, end ns, start clk, end clk, steps tile0, steps tile1, items, -]
#define CS(...) __VA_ARGS__
#else
#define CS(...)
#endif
constexpr float kRescaleThresh = 8.0f;  // log2 units
#ifndef PARSE_SMX_REGS
#define PARSE_SMX_REGS 216
#endif
#ifndef PARSE_WG0_REGS
#define PARSE_WG0_REGS 72
#endif
#ifdef PARSE_PF_EARLY
constexpr bool kPfEarly = true;    // claim the next item right after the current one starts
#else
constexpr bool kPfEarly = false;
#endif
#ifdef PARSE_PF_SYNC
constexpr bool kPfSync = true;     // no prefetch: claim + load when the item starts
#else
constexpr bool kPfSync = false;
#endif

template <int D, bool kFp8>
struct Cfg {
  static constexpr int kElem = kFp8 ? 1 : 2;      // bytes per Q / K / V element
  static constexpr int kChunkElems = 128 / kElem; // elements of d per 128-byte swizzle atom
  static constexpr int kChunks = D / kChunkElems; // 128-byte swizzle atoms along d
  static constexpr int kChunkBytes = 128 * 128;   // 128 rows x 128 B
  static constexpr int kTileBytes = 128 * D * kElem;  // one Q / K / V tile
  static constexpr int kKStep = kFp8 ? 32 : 16;   // MMA K per instruction (32 bytes of a row)
#ifndef PARSE_KV_STAGES
  static constexpr int kStages = (D == 128 && !kFp8) ? 5 : 8;
#else
  static constexpr int kStages = PARSE_KV_STAGES;
#endif
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kTileBytes;
  static constexpr int kBarOff = kKVOff + kStages * kTileBytes;
  // barriers: q_full[2] q_empty[2] s_full[2] p_full[2] o_full[2] kv_full[S] kv_empty[S]
  //           item_full[R] item_empty[R]; then the item ring (R x 64 B) and the TMEM slot
  static constexpr int kItemRing = 4;
  static constexpr int kMbox = 4;   // 2-CTA cluster: unit-index mailbox depth
  // + s_free[2] p_free[2] probe[2] mma_done mbox_full[kMbox] mbox_empty[kMbox]
  static constexpr int kNumBars = 17 + 2 * kStages + 2 * kItemRing + 2 * kMbox;
  static constexpr int kItemOff = (kBarOff + kNumBars * 8 + 15) / 16 * 16;
  static constexpr int kMboxOff = kItemOff + 64 * kItemRing + 16;   // after the ring and the TMEM slot
  static constexpr int kSmem = kMboxOff + 4 * kMbox + 1024;         // + align slack
  static constexpr int kTmemCols = 512;
  static constexpr int kSCol = 0;    // S: one 128-column buffer, used by the two Q tiles in turn
  static constexpr int kPCol = 128;  // P_i at 128 + i*64 (bf16 pairs, or e4m3 quads in 32 columns)
  static constexpr int kOCol = 256;  // O_i at 256 + i*D
};

struct Bars {
  uint32_t base;
  __device__ uint32_t q_full(int i) const { return base + 8 * (0 + i); }
  __device__ uint32_t q_empty(int i) const { return base + 8 * (2 + i); }
  __device__ uint32_t s_full(int i) const { return base + 8 * (4 + i); }
  __device__ uint32_t p_full(int i) const { return base + 8 * (6 + i); }
  __device__ uint32_t o_full(int i) const { return base + 8 * (8 + i); }
  __device__ uint32_t kv_full(int s) const { return base + 8 * (10 + s); }
  __device__ uint32_t kv_empty(int s, int nst) const { return base + 8 * (10 + nst + s); }
  __device__ uint32_t item_full(int r, int nst) const { return base + 8 * (10 + 2 * nst + r); }
  __device__ uint32_t item_empty(int r, int nst, int nring) const { return base + 8 * (10 + 2 * nst + nring + r); }
  // tile i's softmax has copied S into registers: the other tile's QK^T may overwrite it
  __device__ uint32_t s_free(int i, int nst, int nring) const { return base + 8 * (10 + 2 * nst + 2 * nring + i); }
  // PV_i(j) has completed (not committed for an item's last step: o_full covers it):
  // P_i may be overwritten and O_i rescaled
  __device__ uint32_t p_free(int i, int nst, int nring) const { return base + 8 * (12 + 2 * nst + 2 * nring + i); }
  // trace builds: MMA-group completion probes, and both MMA warps done
  __device__ uint32_t probe(int i, int nst, int nring) const { return base + 8 * (14 + 2 * nst + 2 * nring + i); }
  __device__ uint32_t mma_done(int nst, int nring) const { return base + 8 * (16 + 2 * nst + 2 * nring); }
  // 2-CTA cluster: CTA 1's mailbox slot m holds a unit index (written by CTA 0)
  __device__ uint32_t mbox_full(int m, int nst, int nring) const { return base + 8 * (17 + 2 * nst + 2 * nring + m); }
  // CTA 0: CTA 1 has read slot m
  __device__ uint32_t mbox_empty(int m, int nst, int nring, int nmb) const {
    return base + 8 * (17 + 2 * nst + 2 * nring + nmb + m);
  }
};
// flags bit 10 (set on the device only): the cluster's second CTA recomputes
// its partner's item without storing it (a unit with no partner item)
constexpr int kGhostFlag = 1 << 10;

__device__ __forceinline__ int item_hpt(const WorkItem& w) { return w.flags & 0xff; }
__device__ __forceinline__ int item_nq(const WorkItem& w) { return (w.flags >> 8) & 1 ? 2 : 1; }
// first token / first q head of Q tile i of an item
__device__ __forceinline__ int tile_t0(const WorkItem& w, int i, int S) { return w.t0 + ((w.flags >> 9) & 1 ? i * S : 0); }
__device__ __forceinline__ int tile_h0(const WorkItem& w, int i) {
  return w.h0 + ((w.flags >> 9) & 1 ? 0 : i * item_hpt(w));
}
__device__ __forceinline__ int kv_key0(const WorkItem& w, int j) {
  return j < w.n_draft ? j * kTile : w.self_lo + (j - w.n_draft) * kTile;
}

// exp2 on the FMA pipe for a pair: 2^x = 2^n * p(x - n), n = round(x), p the
// degree-3 minimax fit of 2^f on [-0.5, 0.5] (max rel err 7.5e-5, well below
// the 2^-9 rounding P gets as bf16).  Adding 1.5*2^23 + 127 leaves n + 127 in
// the low mantissa bits of t; shifting them into the exponent field builds
// 2^n exactly.  x is clamped at -125 so n + 127 >= 2 (2^-125 ~ 0); with
// kZeroMasked the clamp is -127: n + 127 = 0 builds a zero scale, so -inf (a
// masked key) maps to an exact 0 like MUFU.EX2 (and x < -126.5 to 0, as .ftz).
template <bool kZeroMasked = false>
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  constexpr float kMagic = 12582912.f + 127.f;
  constexpr float kLo = kZeroMasked ? -127.f : -125.f;
  x.x = fmaxf(x.x, kLo);
  x.y = fmaxf(x.y, kLo);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 r = fadd2(t, make_float2(-kMagic, -kMagic));   // n
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);      // x - n
  float2 p = ffma2(f, make_float2(0.05517172813f, 0.05517172813f), make_float2(0.24261118472f, 0.24261118472f));
  p = ffma2(p, f, make_float2(0.69326096773f, 0.69326096773f));
  p = ffma2(p, f, make_float2(0.99992805719f, 0.99992805719f));
#ifdef PARSE_EXP_SHF
  // t << 23 as a funnel shift (SHF, integer pipe) instead of IMAD.SHL (FMA pipe)
  uint32_t sx, sy;
  asm("shf.r.clamp.b32 %0, %1, %2, 9;" : "=r"(sx) : "r"(0u), "r"(__float_as_uint(t.x)));
  asm("shf.r.clamp.b32 %0, %1, %2, 9;" : "=r"(sy) : "r"(0u), "r"(__float_as_uint(t.y)));
  const float2 scale = make_float2(__uint_as_float(sx), __uint_as_float(sy));
#else
  const float2 scale = make_float2(__uint_as_float(__float_as_uint(t.x) << 23), __uint_as_float(__float_as_uint(t.y) << 23));
#endif
  return fmul2(p, scale);
}

// kPolyPer16 of every 16 exp pairs use exp2_poly2 (FMA pipe) and the rest
// MUFU.EX2, balancing the two pipes (both tiles' exps otherwise saturate the
// 16/clk/SM MUFU at exactly the tensor-core rate).
#ifndef PARSE_POLY16
constexpr int kPolyPer16 = 4;
#else
constexpr int kPolyPer16 = PARSE_POLY16;
#endif
template <bool kPoly>
__device__ __forceinline__ bool poly_pair(int e) { return kPoly && (e & 15) >= 16 - kPolyPer16; }
// Softmax stages on one thread's 128-column row, in place in registers:
// x = S*scale_log2 - m (FFMA2), p = 2^x for a range of pairs (MUFU for most,
// FMA-pipe polynomial for kPolyPer16 of 16), then row sum + bf16 packing into
// TMEM (P pair e -> column e of S_i, even key in the low half).
__device__ __forceinline__ void x_row_inplace(uint32_t* sr, float2 sl2x2, float2 negm) {
#pragma unroll
  for (int e = 0; e < kTile / 2; ++e) {
    const float2 x = ffma2(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sl2x2, negm);
    sr[2 * e] = __float_as_uint(x.x);
    sr[2 * e + 1] = __float_as_uint(x.y);
  }
}
// kMasked: the tile has masked (-inf) scores, which must become exact zeros
template <bool kPoly, int E0, int E1, bool kMasked = false>
__device__ __forceinline__ void exp_pairs(uint32_t* sr) {
#pragma unroll
  for (int e = E0; e < E1; ++e) {
    const float2 x = make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1]));
    const float2 pp = poly_pair<kPoly>(e) ? exp2_poly2<kMasked>(x) : make_float2(ex2(x.x), ex2(x.y));
    sr[2 * e] = __float_as_uint(pp.x);
    sr[2 * e + 1] = __float_as_uint(pp.y);
  }
}
// FP8 variant: P quad (keys 4c .. 4c+3) -> column c as four e4m3 (key 4c in the
// low byte), so the pairs [E0, E1) fill columns [E0/2, E1/2), 8 per store.
template <int E0, int E1>
__device__ __forceinline__ void store_p_e4m3(const uint32_t* sr, uint32_t tS, float2 (&acc)[4]) {
  static_assert(E0 % 16 == 0 && (E1 - E0) % 16 == 0, "8-column TMEM stores");
#pragma unroll
  for (int e0 = E0; e0 < E1; e0 += 16) {
    uint32_t pk[8];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 pp = make_float2(__uint_as_float(sr[2 * (e0 + e)]), __uint_as_float(sr[2 * (e0 + e) + 1]));
      if (e0 == 0 && e < 4) acc[e] = pp;
      else acc[e & 3] = fadd2(acc[e & 3], pp);
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      pk[c] = pack_e4m3x4(__uint_as_float(sr[2 * e0 + 4 * c]), __uint_as_float(sr[2 * e0 + 4 * c + 1]),
                          __uint_as_float(sr[2 * e0 + 4 * c + 2]), __uint_as_float(sr[2 * e0 + 4 * c + 3]));
    tmem_st8(tS + e0 / 2, pk);
  }
}
template <int E0, int E1>
__device__ __forceinline__ void store_p_pairs(const uint32_t* sr, uint32_t tS, float2 (&acc)[4]) {
  static_assert(E0 % 16 == 0 && (E1 - E0) % 16 == 0, "16-column TMEM stores");
#pragma unroll
  for (int e0 = E0; e0 < E1; e0 += 16) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const float2 pp = make_float2(__uint_as_float(sr[2 * (e0 + e)]), __uint_as_float(sr[2 * (e0 + e) + 1]));
      if (e0 == 0 && e < 4) acc[e] = pp;
      else acc[e & 3] = fadd2(acc[e & 3], pp);
      pk[e] = pack_bf16x2(pp.x, pp.y);
    }
    tmem_st16(tS + e0, pk);
  }
}

// Item ring entry (smem): the work item and its request's geometry, written
// by the producer (which fetched both one item ahead), so the MMA and softmax
// warps never wait on a global load for item metadata.  n_draft < 0 = end.
struct alignas(16) RingEntry {
  WorkItem w;
  ReqDesc r;
};
static_assert(sizeof(RingEntry) == 64, "ring entry is 64 bytes");

// Request geometry of item b: implied by the launch for dense batches, else
// the uploaded per-request table.
__device__ __forceinline__ ReqDesc load_req(const AttnParams& prm, int b) {
  if (prm.dense_L) return ReqDesc{prm.dense_N, prm.dense_L, prm.dense_K, b * prm.dense_K, 0, 0, b, 0};
  return prm.req[b];
}

template <int kStages, int kRing>
__device__ __forceinline__ bool next_item(const Bars& bars, const RingEntry* ring, int& slot, uint32_t& phase,
                                          WorkItem& w, ReqDesc& r) {
  mbar_wait(bars.item_full(slot, kStages), phase);
  w = ring[slot].w;
  r = ring[slot].r;
  mbar_arrive(bars.item_empty(slot, kStages, kRing));
  if (++slot == kRing) { slot = 0; phase ^= 1; }
  return w.n_draft >= 0;
}

// kCl = 2: the grid runs as 2-CTA clusters over work units (build_units):
// both CTAs walk the same K/V steps and, for a multicast unit, each loads
// half of every K/V tile's rows into both CTAs' shared memory, so the pair
// reads each tile from L2 once ("K/V multicast").
template <int D, bool kPaged, bool kFp8, int kCl>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_kernel(const __grid_constant__ AttnParams prm,
                      const __grid_constant__ CUtensorMap tm_q_tok,
                      const __grid_constant__ CUtensorMap tm_q_pack,
                      const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v) {
  using C = Cfg<D, kFp8>;
  // Lazy-rescale threshold and P bias (log2 units).  FP8: P is stored as
  // e4m3 (max 448), so P <= 2^(kThresh + kPBias) = 2^8 and the bias keeps
  // small probabilities out of e4m3's subnormal range; O / l is unaffected
  // (l sums the same biased values) and the LSE subtracts the bias.
  constexpr float kThresh = kFp8 ? 4.0f : kRescaleThresh;
  constexpr float kPBias = kFp8 ? 4.0f : 0.0f;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  Bars bars{sbase + C::kBarOff};
  RingEntry* ring = reinterpret_cast<RingEntry*>(smem + C::kItemOff);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kItemOff + 64 * C::kItemRing);
  // Consumers take work items from the producer's smem ring (dynamic,
  // group-major schedule: co-running CTAs share one request/KV-group in L2).
  int ring_slot = 0;
  uint32_t ring_phase = 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bars.q_full(i), 1);
      mbar_init(bars.q_empty(i), 1);
      mbar_init(bars.s_full(i), 1);
      mbar_init(bars.p_full(i), 128);
      mbar_init(bars.s_free(i, C::kStages, C::kItemRing), 128);
      mbar_init(bars.p_free(i, C::kStages, C::kItemRing), 1);
      mbar_init(bars.probe(i, C::kStages, C::kItemRing), 1);
      mbar_init(bars.o_full(i), 1);
    }
    mbar_init(bars.mma_done(C::kStages, C::kItemRing), 2);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(bars.kv_full(s), 1);
#ifndef PARSE_CL_LOCAL
      mbar_init(bars.kv_empty(s, C::kStages), 2 * kCl);   // both MMA warps (of both CTAs)
#else
      mbar_init(bars.kv_empty(s, C::kStages), 2);         // diagnostic: stages released per CTA
#endif
    }
    if constexpr (kCl == 2) {
      for (int m = 0; m < C::kMbox; ++m) {
        mbar_init(bars.mbox_full(m, C::kStages, C::kItemRing), 1);
        mbar_init(bars.mbox_empty(m, C::kStages, C::kItemRing, C::kMbox), 1);
      }
    }
    for (int r = 0; r < C::kItemRing; ++r) {
      mbar_init(bars.item_full(r, C::kStages), 1);
      mbar_init(bars.item_empty(r, C::kStages, C::kItemRing), 64 + 256);  // MMA warps + softmax WGs
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q_tok);
    tma_prefetch_desc(&tm_q_pack);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) {
    tmem_alloc(smem_u32(tmem_slot), C::kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCl == 2) cl_sync();   // the peer's barriers exist before any remote arrive / multicast
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t crank = kCl == 2 ? cl_rank() : 0u;
  CS(if (threadIdx.x == 0 && prm.trace) {
    long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    prm.trace[blockIdx.x * 8 + 0] = ns;
    prm.trace[blockIdx.x * 8 + 2] = clock64();
  })
  const int r_heads = prm.Hq / prm.Hkv;
  // Warpgroup 0 (TMA / MMA / allocator) needs few registers; hand them to the
  // two softmax warpgroups.  The CTA's pool is what it launched with
  // (384 x 168), so 128*(168-72) released >= 256*(216-168) requested.
  static_assert(128 * (168 - PARSE_WG0_REGS) >= 256 * (PARSE_SMX_REGS - 168), "setmaxnreg budget");
  if (warp < 4) {
    setmaxnreg_dec<PARSE_WG0_REGS>();
  if (warp == 0) {
    // ============================ TMA producer ============================
    // The whole warp walks the schedule; one elected lane issues the TMA.
    int stage = 0;
    uint32_t kv_phase = 0;
    uint32_t q_phase[2] = {0, 0};
    const uint64_t pol_stream = make_policy_evict_first();   // Q: read once
    const uint64_t pol_keep = make_policy_evict_last();      // K/V: re-read by many tiles
    int pstep = 0;
    // The next item is fetched one ahead, in three hops spread over the last
    // KV steps of the current item (claim index -> load item -> load
    // request), so none of the dependent global round trips sits between the
    // release of the Q buffers and the next item's Q load.
    int it_raw = 0;
    int it_n = 0;
    WorkItem wn{};
    ReqDesc rn{};
    bool mc_n = false;          // cluster: the unit's two items walk the same K/V tiles
    // kCl = 1: items; kCl = 2: units, claimed by CTA 0 and passed to CTA 1
    // through its mailbox (st.shared::cluster + a release arrive)
    const int n_total = kCl == 1 ? prm.n_items : prm.n_work;
    [[maybe_unused]] int mslot = 0;
    [[maybe_unused]] uint32_t mphase = 0;
    const uint32_t mbox_addr = sbase + C::kMboxOff;
    auto hop_claim = [&]() {
      if (crank == 0 && lane == 0) it_raw = atomicAdd(prm.counter, 1);
    };
    auto hop_item = [&]() {
      if constexpr (kCl == 1) {
        it_n = __shfl_sync(0xffffffffu, it_raw, 0);
        if (it_n < n_total) wn = prm.items[it_n];
      } else {
        if (crank == 0) {
          it_n = __shfl_sync(0xffffffffu, it_raw, 0);
          if (lane == 0) {
            mbar_wait_acq_cl(bars.mbox_empty(mslot, C::kStages, C::kItemRing, C::kMbox), mphase ^ 1);
            cl_st_u32(cl_map(mbox_addr + 4 * mslot, 1), uint32_t(it_n));
            cl_arrive(cl_map(bars.mbox_full(mslot, C::kStages, C::kItemRing), 1));
          }
        } else {
          mbar_wait_acq_cl(bars.mbox_full(mslot, C::kStages, C::kItemRing), mphase);
          it_n = *reinterpret_cast<volatile int*>(smem + C::kMboxOff + 4 * mslot);
          __syncwarp();
          if (lane == 0) cl_arrive(cl_map(bars.mbox_empty(mslot, C::kStages, C::kItemRing, C::kMbox), 0));
        }
        __syncwarp();
        if (++mslot == C::kMbox) { mslot = 0; mphase ^= 1; }
        if (it_n < n_total) {
          const int2 u = prm.work[it_n];
          int idx = u.x;
          bool ghost = false;
          if (crank == 1) {
            if (u.y >= 0) idx = u.y;
            else if (u.y == -1) ghost = true;
            else idx = -u.y - 2;
          }
          wn = prm.items[idx];
          if (ghost) wn.flags |= kGhostFlag;
#if defined(PARSE_CL_NOMC) || defined(PARSE_CL_LOCAL)
          mc_n = false;       // diagnostic builds: no multicast
#else
          mc_n = u.y >= -1;   // a ghost walks its partner's K/V too
#endif
        }
      }
    };
    auto hop_req = [&]() {
      if (it_n < n_total) rn = load_req(prm, wn.b);
    };
    auto fetch_now = [&]() {
      hop_claim();
      hop_item();
      hop_req();
    };
    if (!kPfSync) fetch_now();
    for (;;) {
      if (kPfSync) fetch_now();
      const int it = it_n;
      const WorkItem w = wn;
      const ReqDesc rq = rn;
      [[maybe_unused]] const bool mc = mc_n;
      mbar_wait(bars.item_empty(ring_slot, C::kStages, C::kItemRing), ring_phase ^ 1);
      if (lane == 0) {
        WorkItem wp = w;
        if (it >= n_total) wp.n_draft = -1;   // end marker
        ring[ring_slot].w = wp;
        ring[ring_slot].r = rq;
        mbar_arrive(bars.item_full(ring_slot, C::kStages));
      }
      __syncwarp();
      if (++ring_slot == C::kItemRing) { ring_slot = 0; ring_phase ^= 1; }
      if (it >= n_total) break;
      int pf = kPfSync ? 3 : 0;         // prefetch hops done for the next item
      auto prefetch_hop = [&]() {
        if (pf == 0) hop_claim();
        else if (pf == 1) hop_item();
        else if (pf == 2) hop_req();
        ++pf;
      };
      const int hpt = item_hpt(w), nq = item_nq(w);
      const int g = w.h0 / r_heads;
      const CUtensorMap* qm = hpt == 1 ? &tm_q_tok : &tm_q_pack;
      for (int i = 0; i < nq; ++i) {
        mbar_wait(bars.q_empty(i), q_phase[i] ^ 1);
        q_phase[i] ^= 1;
        if (elect_one()) {
          mbar_arrive_expect_tx(bars.q_full(i), C::kTileBytes);
          const uint32_t dst = sbase + C::kQOff + i * C::kTileBytes;
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_4d(qm, bars.q_full(i), dst + c * C::kChunkBytes, c * C::kChunkElems, tile_h0(w, i),
                        rq.q_row0 + tile_t0(w, i, prm.S), rq.bcoord, pol_stream);
        }
        __syncwarp();
      }
      const int n = w.n_draft + w.n_self;
      for (int j = 0; j < n; ++j) {
        const int key0 = kv_key0(w, j);
        // paged K/V: lane s resolves the page of the tile's s-th sub-box
        // (box = min(page, 128) keys); pages past the request read as zeros
        // (out-of-bounds page coordinate -> TMA zero fill)
        int pg = 0, prow = 0;
        const int box = kPaged ? min(1 << prm.page_log2, kTile) : kTile;
        if (kPaged) {
          const int key = key0 + lane * box;
          pg = prm.num_pages;
          if (lane < kTile / box && key < rq.L) pg = __ldg(prm.block_table + int64_t(w.b) * prm.bt_stride + (key >> prm.page_log2));
          if (pg < 0) pg = prm.num_pages;
          prow = key & ((1 << prm.page_log2) - 1);
        }
#pragma unroll
        for (int kv = 0; kv < 2; ++kv) {
          TR(lane == 0, 32768, pstep, 2 * kv);
          mbar_wait(bars.kv_empty(stage, C::kStages), kv_phase ^ 1);
          TR(lane == 0, 32768, pstep, 2 * kv + 1);
          const CUtensorMap* km = kv == 0 ? &tm_k : &tm_v;
          const uint32_t dst = sbase + C::kKVOff + stage * C::kTileBytes;
          if (!kPaged) {
#ifdef PARSE_NO_KV_LOAD
            // timing experiment only: after the first steps the stages keep stale tiles
            if (pstep >= 4) {
              if (lane == 0) mbar_arrive(bars.kv_full(stage));
            } else
#endif
            if constexpr (kCl == 2) {
              // a multicast unit: one CTA loads the tile into both CTAs (same
              // offsets; each CTA's kv_full at the same address counts all 32
              // KB, announced by its own producer); K tiles come from CTA 0 and
              // V tiles from CTA 1, so each tile has one issuer (measured
              // against each CTA loading half of every tile's rows: 23.48 vs
              // 23.65 M cycles on config 3).  Otherwise each CTA loads its own.
              if (elect_one()) {
                mbar_arrive_expect_tx(bars.kv_full(stage), C::kTileBytes);
                if (!mc || uint32_t(kv) == crank) {
#pragma unroll
                  for (int c = 0; c < C::kChunks; ++c) {
                    if (mc)
                      tma_load_4d_mc(km, bars.kv_full(stage), dst + c * C::kChunkBytes, c * C::kChunkElems, g,
                                     rq.kv_row0 + key0, rq.bcoord, 0x3, pol_keep);
                    else
                      tma_load_4d(km, bars.kv_full(stage), dst + c * C::kChunkBytes, c * C::kChunkElems, g,
                                  rq.kv_row0 + key0, rq.bcoord, pol_keep);
                  }
                }
              }
            } else
            if (elect_one()) {
#ifndef PARSE_HALF_KV_LOAD
              mbar_arrive_expect_tx(bars.kv_full(stage), C::kTileBytes);
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c)
#else
              // timing experiment only (stale second chunk): half the L2 -> SMEM bytes
              mbar_arrive_expect_tx(bars.kv_full(stage), C::kChunkBytes);
              for (int c = 0; c < 1; ++c)
#endif
                tma_load_4d(km, bars.kv_full(stage), dst + c * C::kChunkBytes, c * C::kChunkElems, g, rq.kv_row0 + key0,
                            rq.bcoord, pol_keep);
            }
          } else {
            if (lane == 0) mbar_arrive_expect_tx(bars.kv_full(stage), C::kTileBytes);
            __syncwarp();
            // cluster, multicast unit: the tile's owner (K: CTA 0, V: CTA 1)
            // loads every page box into both CTAs
            if (lane < kTile / box && (kCl == 1 || !mc || uint32_t(kv) == crank)) {
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c) {
                if (kCl == 2 && mc)
                  tma_load_4d_mc(km, bars.kv_full(stage), dst + c * C::kChunkBytes + lane * box * 128,
                                 c * C::kChunkElems, g, prow, pg, 0x3, pol_keep);
                else
                  tma_load_4d(km, bars.kv_full(stage), dst + c * C::kChunkBytes + lane * box * 128, c * C::kChunkElems,
                              g, prow, pg, pol_keep);
              }
            }
          }
          __syncwarp();
          if (++stage == C::kStages) { stage = 0; kv_phase ^= 1; }
        }
        ++pstep;
        // hops at the last three KV steps: the next item is claimed as late as
        // possible (dynamic balance) but its metadata is ready by the time the
        // Q buffers are released
        if (pf < 3 && (kPfEarly || j >= n - 3)) prefetch_hop();
      }
      while (pf < 3) prefetch_hop();
    }
    if constexpr (kCl == 2) {
      // every stage's last fill released by both CTAs: no arrive of the
      // peer's MMA warps is still on its way to this CTA's barriers
      for (int k = 0; k < C::kStages; ++k) {
        mbar_wait(bars.kv_empty(stage, C::kStages), kv_phase ^ 1);
        if (++stage == C::kStages) { stage = 0; kv_phase ^= 1; }
      }
    }
  }
#ifdef PARSE_TRACE
  else if (warp == 2 && blockIdx.x == 0 && prm.trace) {
    // timestamp every MMA-group completion of both tiles (busy polling: trace builds only)
    auto test = [&](uint32_t bar, uint32_t par) {
      uint32_t ok;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(bar), "r"(par) : "memory");
      return ok != 0;
    };
    uint32_t ph[2] = {0, 0};
    int k[2] = {0, 0};
    bool fin = false;
    for (;;) {
      for (int i = 0; i < 2; ++i) {
        if (test(bars.probe(i, C::kStages, C::kItemRing), ph[i])) {
          if (lane == 0 && k[i] < 4096) prm.trace[57344 + 4096 * i + k[i]] = clock64();
          ph[i] ^= 1;
          ++k[i];
        }
      }
      if (!fin) fin = test(bars.mma_done(C::kStages, C::kItemRing), 0);
      if (fin) {
        const volatile int* np = reinterpret_cast<volatile int*>(tmem_slot);
        if (k[0] >= np[1] && k[1] >= np[2]) break;
      }
    }
  }
#endif
  else if (warp == 1 || warp == 3) {
    // ============================ MMA issuers =============================
    // One warp per Q tile (warp 1: tile 0, warp 3: tile 1), so each tile's
    // MMAs wait only on its own softmax and on the S buffer: the two tiles'
    // MMAs interleave in the tensor pipe without head-of-line blocking.  An
    // elected lane issues; descriptors are precomputed (advancing along K /
    // across stages only changes the 14-bit start-address field).  Both warps
    // walk every K/V stage; a stage is released when both have committed
    // (kv_empty count 2; kCl = 2: count 4, each commit multicast to both
    // CTAs' barriers, since the peer's producer writes into this CTA's copy
    // of the stage), an absent tile 1 releasing its stages by a plain arrive
    // (and a remote one) after the stage has landed.
    //
    // The S buffer is used in the fixed order QK_0(g), QK_1(g), QK_0(g+1), ...
    // over the global key-step index g (all items of this CTA, in ring
    // order): QK_1(g) waits for tile 0's softmax to have loaded S(g)
    // (s_free[0] completion g), QK_0(g+1) for tile 1's (s_free[1] completion
    // g).  An absent tile 1 keeps the order with a dummy use (plain arrive on
    // s_full[1], answered by its softmax warpgroup arriving on s_free[1]), so
    // every barrier advances one phase per step and no waiter can fall two
    // phases behind.  Per step the order is QK_i(j+1), then PV_i(j): tile
    // i's next S is computed while its softmax still works on step j.
    const int i = warp == 1 ? 0 : 1;
    constexpr uint32_t idesc_qk = kFp8 ? make_idesc_e4m3(128, 128, 0) : make_idesc_bf16(128, 128, 0);
    constexpr uint32_t idesc_pv = kFp8 ? make_idesc_e4m3(128, D, 1) : make_idesc_bf16(128, D, 1);
    const uint64_t qdesc = make_sdesc_sw128(sbase + C::kQOff + i * C::kTileBytes, 16, 1024);
    const uint64_t kdesc0 = make_sdesc_sw128(sbase + C::kKVOff, 16, 1024);
    const uint64_t vdesc0 = make_sdesc_sw128(sbase + C::kKVOff, C::kChunkBytes, 1024);
    const uint32_t s_tmem = tmem + C::kSCol;
    const uint32_t p_tmem = tmem + C::kPCol + i * 64;
    const uint32_t o_tmem = tmem + C::kOCol + i * D;
    const uint32_t sfree_other = bars.s_free(i ^ 1, C::kStages, C::kItemRing);
    // release a K/V stage: in a cluster, in both CTAs (the peer's producer
    // multicasts into this CTA's copy of the stage)
    auto release_kv_mma = [&](int st) {
#ifndef PARSE_CL_LOCAL
      if constexpr (kCl == 2) mma_commit_mc(bars.kv_empty(st, C::kStages), 0x3);
#else
      if constexpr (false) {}
#endif
      else mma_commit(bars.kv_empty(st, C::kStages));
    };
    auto release_kv_plain = [&](int st) {   // lane 0: a stage no MMA of this tile reads
      mbar_arrive(bars.kv_empty(st, C::kStages));
#ifndef PARSE_CL_LOCAL
      if constexpr (kCl == 2) cl_arrive(cl_map(bars.kv_empty(st, C::kStages), crank ^ 1u));
#endif
    };
    int stage = 0;
    uint32_t kv_phase = 0;
    uint32_t q_phase = 0, p_phase = 0;
    uint32_t g = 0;          // global key-step index of the S use about to be issued
    int mstep = 0;
    TRP(int n_probe = 0;)
    CS(long long cs_steps = 0, cs_items = 0;)
    auto issue_qk = [&](int kst, int tstep) {
      const uint64_t kd = kdesc0 + uint64_t((kst * C::kTileBytes) >> 4);
#pragma unroll
      for (int kk = 0; kk < D / C::kKStep; ++kk) {
        // K-step kk = bytes [32kk, 32kk + 32) of each row: atom kk / 4, 32-byte column kk % 4
        const uint64_t off = uint64_t(((kk >> 2) * C::kChunkBytes + (kk & 3) * 32) >> 4);
        if constexpr (kFp8) mma_ss_f8(s_tmem, qdesc + off, kd + off, idesc_qk, kk > 0);
        else mma_ss(s_tmem, qdesc + off, kd + off, idesc_qk, kk > 0);
        // trace: first and last MMA of tile 0's QK^T(j+1) accepted
        TR(kk == 0 && i == 0 && tstep >= 0, 40960, tstep, 7);
        TR(kk == D / C::kKStep - 1 && i == 0 && tstep >= 0, 49152, tstep, 7);
      }
    };
    auto issue_pv = [&](int vst, bool acc, int kk0, int kk1) {
      const uint64_t vd = vdesc0 + uint64_t((vst * C::kTileBytes) >> 4);
      // K-step kk = keys [kKStep*kk, +kKStep): P columns 8kk.. (2 bf16 or 4 e4m3 per
      // column), V rows of kKStep/8 8-row groups (1024 B each)
#pragma unroll
      for (int kk = kk0; kk < kk1; ++kk) {
        const uint64_t voff = uint64_t((kk * (C::kKStep / 8) * 1024) >> 4);
        if constexpr (kFp8) mma_ts_f8(o_tmem, p_tmem + kk * 8, vd + voff, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        else mma_ts(o_tmem, p_tmem + kk * 8, vd + voff, idesc_pv, (acc || kk > 0) ? 1u : 0u);
      }
    };
    auto next_stage = [&](int& st) {
      st = stage;
      mbar_wait(bars.kv_full(stage), kv_phase);
      if (++stage == C::kStages) { stage = 0; kv_phase ^= 1; }
    };
    // S use g of this tile: wait until the previous user's softmax has loaded
    // S (tile 0: tile 1's use g-1; tile 1: tile 0's use g), then issue QK^T
    // (or the dummy use of an absent tile 1) and release the K stage.
    auto use_s = [&](bool real, int kst, bool last_qk, int tstep) {
      TR(lane == 0 && tstep >= 0, 16384 + i * 8192, tstep, 3);
      // polled without the suspend hint: the S hand-off between the tiles is
      // the kernel's critical chain and the poll saves the wake-up latency
      // (config 3 23.13 -> 23.02 M cycles, config 2 -1.2%; polling the
      // p_full or the softmax's s_full waits as well measured slower).  No
      // watchdog in this loop (it costs 0.3%): a deadlock leaves the other
      // roles in mbar_wait, whose watchdog traps the grid.
      if (i == 1 || g > 0) {
        const uint32_t par = (i == 1 ? g : g - 1) & 1;
#ifndef PARSE_SFREE_SLEEP
        while (!mbar_test(sfree_other, par)) {}
#else
        mbar_wait(sfree_other, par);   // A/B build: suspend-hinted wait (less issue / power)
#endif
      }
      TR(lane == 0 && tstep >= 0, 16384 + i * 8192, tstep, 4);
      ++g;
      if (real) {
        tc_fence_after();
        if (elect_one()) {
          issue_qk(kst, tstep);
          TRP(if (blockIdx.x == 0 && prm.trace) { mma_commit(bars.probe(i, C::kStages, C::kItemRing)); ++n_probe; })
          mma_commit(bars.s_full(i));
          release_kv_mma(kst);
          if (last_qk) mma_commit(bars.q_empty(i));
        }
      } else if (lane == 0) {
        mbar_arrive(bars.s_full(i));
        release_kv_plain(kst);
      }
      __syncwarp();
    };
    for (;;) {
      WorkItem w;
      ReqDesc rq_unused;
      if (!next_item<C::kStages, C::kItemRing>(bars, ring, ring_slot, ring_phase, w, rq_unused)) break;
      const int nq = item_nq(w);
      const int n = w.n_draft + w.n_self;
      const bool real = i < nq;
      CS(if (real) { cs_steps += n; cs_items += 1; })
      if (real) {
        TR(lane == 0 && i == 0, 32768, mstep, 4);
        mbar_wait(bars.q_full(i), q_phase);
        TR(lane == 0 && i == 0, 32768, mstep, 5);
        q_phase ^= 1;
      }
      int kst, vst;
      next_stage(kst);
      TR(lane == 0 && i == 0, 32768, mstep, 6);
      use_s(real, kst, n == 1, -1);
      TR(lane == 0 && real, 16384 + i * 8192, mstep, 5);   // QK(0) of the item issued
      TR(lane == 0 && i == 0, 32768, mstep, 7);
      for (int j = 0; j < n; ++j, ++mstep) {
        const bool more = j + 1 < n;
        TR(lane == 0, 16384 + i * 8192, mstep, 6);
        next_stage(vst);
        if (more) {
          next_stage(kst);
          use_s(real, kst, j + 2 == n, mstep);
        }
        TR(lane == 0, 16384 + i * 8192, mstep, 7);
        if (!real) {
          if (lane == 0) release_kv_plain(vst);
          __syncwarp();
          continue;
        }
        TR(lane == 0, 16384 + i * 8192, mstep, 0);
        mbar_wait(bars.p_full(i), p_phase);
        TR(lane == 0, 16384 + i * 8192, mstep, 1);
        p_phase ^= 1;
        tc_fence_after();
        if (elect_one()) {
          issue_pv(vst, j > 0, 0, kTile / C::kKStep);
          TRP(if (blockIdx.x == 0 && prm.trace) { mma_commit(bars.probe(i, C::kStages, C::kItemRing)); ++n_probe; })
          // O complete: the epilogue needs it (one phase per item); within
          // the item the softmax's next P stores / O rescale wait on p_free
          mma_commit(more ? bars.p_free(i, C::kStages, C::kItemRing) : bars.o_full(i));
          release_kv_mma(vst);
        }
        __syncwarp();
        TR(lane == 0, 16384 + i * 8192, mstep, 2);
      }
    }
    TRP(if (blockIdx.x == 0 && prm.trace) {
      n_probe = __reduce_add_sync(0xffffffffu, n_probe);   // counted by whichever lane was elected
      if (lane == 0) {
        reinterpret_cast<volatile int*>(tmem_slot)[1 + i] = n_probe;
        mbar_arrive(bars.mma_done(C::kStages, C::kItemRing));
      }
    })
    CS(if (lane == 0 && prm.trace) {
      prm.trace[blockIdx.x * 8 + 4 + i] = cs_steps;
      if (i == 0) prm.trace[blockIdx.x * 8 + 6] = cs_items;
    })
  }
  } else {
    setmaxnreg_inc<PARSE_SMX_REGS>();
    // ========================== softmax warpgroups ==========================
    const int wg = (warp - 4) >> 2;             // Q tile index
    const int row = threadIdx.x & 127;          // = TMEM lane
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + C::kSCol;            // shared with the other tile
    const uint32_t tP = tmem + lane_base + C::kPCol + wg * 64;
    const uint32_t tO = tmem + lane_base + C::kOCol + wg * D;
    // Ping-pong: the two softmax warpgroups take turns on the SM sub-partition
    // pipes (MUFU / FMA / issue), so each tile's softmax runs at full rate
    // while the tensor core works on the other tile.  Named barriers:
    // WG i waits on turn[i] (its 128 threads sync, the other WG's 128 arrive).
    constexpr uint32_t kTurnBar0 = 1;
    [[maybe_unused]] const uint32_t my_turn = kTurnBar0 + wg, other_turn = kTurnBar0 + (wg ^ 1);
    PP(if (wg == 1) named_bar_arrive(kTurnBar0, 256);)  // tile 0 goes first
    uint32_t s_phase = 0;
    uint32_t pf_phase = 0;                      // p_free[wg]: steps 1.. of every item
    uint32_t o_phase = 0;                       // o_full[wg] completes once per item
    int sstep = 0;
    const float sl2 = prm.scale_log2;
    const uint64_t pol_out = make_policy_evict_first();      // O: written once
    // visibility of a row: keys [0, lim) of the shared region, plus
    // own-copy keys [sbase, t] (or the tree ancestors of suffix position sidx)
    struct RowVis { int t, lim, sbase_k, sidx; uint64_t anc; };
    auto row_setup = [&](const WorkItem& w_, const ReqDesc& rq_) {
      RowVis v;
      v.t = tile_t0(w_, wg, prm.S) + row / item_hpt(w_);
      v.sbase_k = 0x7fffffff;
      v.sidx = 0;
      if (v.t < rq_.N) {
        v.lim = v.t + 1;
      } else if (v.t < rq_.L) {
        const int k = (v.t - rq_.N) / prm.S;
        v.sidx = v.t - rq_.N - k * prm.S;
        v.lim = prm.bnd[rq_.bnd_off + k];
        v.sbase_k = rq_.N + k * prm.S;
      } else {
        v.lim = 0;
      }
      v.anc = prm.anc ? prm.anc[v.sidx] : 0ull;
      return v;
    };
    WorkItem w;
    ReqDesc rq;
    RowVis vis{};
    bool have = next_item<C::kStages, C::kItemRing>(bars, ring, ring_slot, ring_phase, w, rq);
    if (have && wg < item_nq(w)) vis = row_setup(w, rq);
    for (; have;) {
      TR(row == 0, 40960 + wg * 8192, sstep, 3);
      const int nq = item_nq(w);
      if (wg >= nq) {
        // tile 1 absent: answer the MMA warp's dummy S uses (the S buffer
        // order stays QK_0, QK_1, QK_0, ...) and keep the turn-taking in step
        for (int j = 0; j < w.n_draft + w.n_self; ++j) {
          mbar_wait(bars.s_full(wg), s_phase);
          s_phase ^= 1;
          mbar_arrive(bars.s_free(wg, C::kStages, C::kItemRing));
          PP(named_bar_sync(my_turn, 256);)
          PP(named_bar_arrive(other_turn, 256);)
        }
        have = next_item<C::kStages, C::kItemRing>(bars, ring, ring_slot, ring_phase, w, rq);
        if (have && wg < item_nq(w)) vis = row_setup(w, rq);
        continue;
      }
      const int hpt = item_hpt(w);
      const int n = w.n_draft + w.n_self;
      const int t = vis.t, lim = vis.lim, sbase_k = vis.sbase_k;
      const uint64_t anc_row = vis.anc;
      TR(row == 0, 40960 + wg * 8192, sstep, 4);
      float m_used = -INFINITY, l_sum = 0.f;
      for (int j = 0; j < n; ++j, ++sstep) {
        TR(row == 0, wg * 8192, sstep, 0);
        mbar_wait(bars.s_full(wg), s_phase);
        TR(row == 0, wg * 8192, sstep, 1);
        s_phase ^= 1;
        tc_fence_after();
        uint32_t sr[kTile];
        tmem_ld64(tS, sr);
        tmem_ld64(tS + 64, sr + 64);
        tmem_wait_ld();
        reg_fence<kTile>(sr);
        // S is in registers: the other tile's QK^T may overwrite the buffer
        tc_fence_before();
        mbar_arrive(bars.s_free(wg, C::kStages, C::kItemRing));
        PP(named_bar_sync(my_turn, 256);)
        TR(row == 0, wg * 8192, sstep, 2);
        const int key0 = kv_key0(w, j);
        bool masked = true;
        if (j < w.n_draft) {
          const int nvis = lim - key0;           // keys [key0, lim) visible
          masked = nvis < kTile;
          if (masked) {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c >= nvis) sr[c] = 0xff800000u;  // -inf
          }
        } else {
          const int lo = sbase_k - key0;         // own copy starts at column lo
          const int hi = t - key0;               // causal: columns <= hi
          if (prm.anc) {
#pragma unroll
            for (int c = 0; c < kTile; ++c) {
              const int rel = c - lo;
              const bool vis = rel >= 0 && rel < 64 && ((anc_row >> (rel & 63)) & 1ull);
              if (!vis) sr[c] = 0xff800000u;  // -inf
            }
          } else {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c < lo || c > hi) sr[c] = 0xff800000u;  // -inf
          }
        }
        // row max: 8 independent 3-input max chains, then a tree
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float m = fmax3(__uint_as_float(sr[16 * i]), __uint_as_float(sr[16 * i + 1]), __uint_as_float(sr[16 * i + 2]));
#pragma unroll
          for (int e = 3; e < 15; e += 2) m = fmax3(m, __uint_as_float(sr[16 * i + e]), __uint_as_float(sr[16 * i + e + 1]));
          mx[i] = fmaxf(m, __uint_as_float(sr[16 * i + 15]));
        }
        const float mt = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float m_tile = mt * sl2;
        TR(row == 0, wg * 8192, sstep, 3);
        float alpha = 1.f;
        bool rescale_o = false;
        if (m_tile > m_used + kThresh) {
          alpha = ex2(m_used - m_tile);
          rescale_o = (m_used != -INFINITY);
          m_used = m_tile;
        }
        const bool any_rescale = __any_sync(0xffffffffu, rescale_o);
        const float m_eff = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2x2 = make_float2(sl2, sl2);
        const float2 negm = make_float2(kPBias - m_eff, kPBias - m_eff);
        float2 acc[4];
        const bool all_full = __all_sync(0xffffffffu, !masked);
#ifndef PARSE_NO_SOFTMAX_MATH
        x_row_inplace(sr, sl2x2, negm);
        if (all_full) exp_pairs<true, 0, kTile / 2>(sr);
#ifndef PARSE_POLY_MASKED2
        else exp_pairs<false, 0, kTile / 2>(sr);
#else
        else exp_pairs<true, 0, kTile / 2, true>(sr);   // A/B build: polynomial pairs on masked tiles too
#endif
#endif
        TR(row == 0, 40960 + wg * 8192, sstep, 5);
        if (j > 0) {
          // PV(j-1) has read P(j-1) and updated O (it normally completed long ago)
          mbar_wait(bars.p_free(wg, C::kStages, C::kItemRing), pf_phase);
          pf_phase ^= 1;
          tc_fence_after();
        }
        TR(row == 0, 40960 + wg * 8192, sstep, 6);
        if constexpr (kFp8) store_p_e4m3<0, kTile / 2>(sr, tP, acc);
        else store_p_pairs<0, kTile / 2>(sr, tP, acc);
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        l_sum = fmaf(l_sum, alpha, a.x + a.y);
        PP(named_bar_arrive(other_turn, 256);)
        TR(row == 0, wg * 8192, sstep, 4);
        if (any_rescale) {
          // rare: O_i must hold PV(j-1) before it is rescaled in place (p_free,
          // waited above; at j = 0 nothing is rescaled), and the rescale must
          // land before PV(j) starts (the p_full hand-off below)
          const float2 al2 = make_float2(alpha, alpha);
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t ro[32];
            tmem_ld32(tO + c * 32, ro);
            tmem_wait_ld();
            reg_fence<32>(ro);
#pragma unroll
            for (int e = 0; e < 32; e += 2) {
              const float2 v = fmul2(make_float2(__uint_as_float(ro[e]), __uint_as_float(ro[e + 1])), al2);
              ro[e] = __float_as_uint(v.x);
              ro[e + 1] = __float_as_uint(v.y);
            }
            tmem_st32(tO + c * 32, ro);
          }
        }
        // P (and a rescaled O) in TMEM: PV(j) may start
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bars.p_full(wg));
        TR(row == 0, wg * 8192, sstep, 5);
      }
      // ------------------------------ epilogue ------------------------------
      // The next item's ring entry and row setup (a global boundary load)
      // first: their latency overlaps the wait for the last PV.
      const int h = tile_h0(w, wg) + row % hpt;
      const bool row_valid = t < w.t_end && !(w.flags & kGhostFlag);
      const int64_t o_off = rq.bcoord * prm.o_s0 + int64_t(rq.q_row0 + t) * prm.o_s1 + int64_t(h) * prm.o_s2;
      const int64_t lse_off = rq.bcoord * prm.lse_sb + h * prm.lse_sh + rq.q_row0 + t;
      TR(row == 0, 40960 + wg * 8192, sstep, 2);
      have = next_item<C::kStages, C::kItemRing>(bars, ring, ring_slot, ring_phase, w, rq);
      if (have && wg < item_nq(w)) vis = row_setup(w, rq);
      TR(row == 0, wg * 8192, sstep, 6);
      mbar_wait(bars.o_full(wg), o_phase);
      TR(row == 0, wg * 8192, sstep, 7);
      o_phase ^= 1;
      tc_fence_after();
      const float inv_l = l_sum > 0.f ? prm.o_scale / l_sum : 0.f;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.o) + o_off;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t raw[32];
        tmem_ld32(tO + c * 32, raw);
        tmem_wait_ld();
        reg_fence<32>(raw);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          pk[e] = pack_bf16x2(__uint_as_float(raw[2 * e]) * inv_l, __uint_as_float(raw[2 * e + 1]) * inv_l);
        }
        if (row_valid) {
          if (prm.o_v8) {
            // 32-byte stores: each is one whole L2 sector (the 16-byte form
            // writes every sector in two halves and made the epilogue LSU-bound)
#pragma unroll
            for (int e = 0; e < 2; ++e) st_global_v8_hint(orow + c * 32 + 16 * e, pk + 8 * e, pol_out);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              st_global_v4_hint(dst + e, make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]), pol_out);
          }
        }
      }
      TR(row == 0, 40960 + wg * 8192, sstep, 0);
      if (row_valid && prm.lse) prm.lse[lse_off] = (m_used + __log2f(l_sum) - kPBias) * 0.69314718055994531f;
    }
    PP(if (wg == 0) named_bar_sync(kTurnBar0, 256);)    // absorb tile 1's last hand-back
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (kCl == 2) cl_sync();   // the peer no longer multicasts into / arrives on this CTA
  CS(if (threadIdx.x == 0 && prm.trace) {
    long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    prm.trace[blockIdx.x * 8 + 1] = ns;
    prm.trace[blockIdx.x * 8 + 3] = clock64();
  })
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

template <int D, bool kPaged, bool kFp8, int kCl>
cudaError_t launch_impl(const AttnParams& prm, const CUtensorMap& a, const CUtensorMap& b,
                        const CUtensorMap& c, const CUtensorMap& d,
                        int num_sms, cudaStream_t stream) {
  using Cf = Cfg<D, kFp8>;
  auto kern = attn_sm100_kernel<D, kPaged, kFp8, kCl>;
  cudaError_t e = opt_in_smem<attn_sm100_kernel<D, kPaged, kFp8, kCl>>(Cf::kSmem);
  if (e != cudaSuccess) return e;
  if constexpr (kCl == 1) {
    const int grid = prm.n_items < num_sms ? prm.n_items : num_sms;  // persistent, items fetched dynamically
    if (grid <= 0) return cudaSuccess;
    kern<<<grid, kThreads, Cf::kSmem, stream>>>(prm, a, b, c, d);
    return cudaGetLastError();
  } else {
    // persistent 2-CTA clusters: as many as can be co-resident (queried once
    // per device), units fetched dynamically
    static std::atomic<int> max_clusters[64];
    int dev = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cf::kSmem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int mc = max_clusters[dev].load(std::memory_order_acquire);
    if (mc <= 0) {
      cfg.gridDim = dim3(2 * (num_sms / 2));
      if ((e = cudaOccupancyMaxActiveClusters(&mc, kern, &cfg)) != cudaSuccess) return e;
      if (mc <= 0) return cudaErrorLaunchOutOfResources;
      if (mc > num_sms / 2) mc = num_sms / 2;
      max_clusters[dev].store(mc, std::memory_order_release);
    }
    const int clusters = prm.n_work < mc ? prm.n_work : mc;
    if (clusters <= 0) return cudaSuccess;
    cfg.gridDim = dim3(2 * clusters);
    return cudaLaunchKernelEx(&cfg, kern, prm, a, b, c, d);
  }
}

}  // namespace

// Paged K/V is a separate instantiation so the dense kernel carries none of
// its producer code (the softmax loop is large; instruction-cache footprint
// measurably matters).  FP8 (e4m3 Q/K/V, P): head_dim 128.  cluster: 2-CTA
// clusters with K/V multicast (prm.work = build_units); else one CTA per SM
// (the PARSE_NO_CLUSTER / experimental-kernel builds).
cudaError_t launch_attn_sm100(const AttnParams& prm, int D, bool fp8, bool cluster, const CUtensorMap& tm_q_tok,
                              const CUtensorMap& tm_q_pack, const CUtensorMap& tm_k,
                              const CUtensorMap& tm_v,
                              int num_sms, cudaStream_t stream) {
  const bool paged = prm.page_log2 > 0;
#if defined(PARSE_NO_CLUSTER) || defined(PARSE_WITH_PAIR) || defined(PARSE_WITH_2SM)
  // A/B and experimental-kernel builds: the one-CTA kernel (kCl = 1)
  if (cluster) return cudaErrorInvalidValue;
#define PARSE_LAUNCH(D_, FP8_)                                                                                   \
  return paged ? launch_impl<D_, true, FP8_, 1>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream)           \
               : launch_impl<D_, false, FP8_, 1>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream);
#else
  // libparse.so: one kernel family, the 2-CTA cluster instantiations
  if (!cluster) return cudaErrorInvalidValue;
#define PARSE_LAUNCH(D_, FP8_)                                                                                   \
  return paged ? launch_impl<D_, true, FP8_, 2>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream)           \
               : launch_impl<D_, false, FP8_, 2>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream);
#endif
  if (fp8) {
    if (D != 128) return cudaErrorInvalidValue;
    PARSE_LAUNCH(128, true)
  }
  if (D == 128) {
    PARSE_LAUNCH(128, false)
  }
  PARSE_LAUNCH(64, false)
#undef PARSE_LAUNCH
}

}  // namespace parse
