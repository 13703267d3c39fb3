// parse_verify_attn, bf16, head_dim 128, dense or packed-row K/V: the CTA-pair
// kernel.  Same work items, same visibility (§3.2),
// same online softmax as attn_sm100_kernel; a different pipeline.
//
// Why: in the one-CTA kernel each Q tile's P aliases its S in
// TMEM (round 1's one-CTA layout: S0 | S1 | O0 | O1 fill all 512 columns), so QK^T(j+1) of a tile waits
// for PV(j) to have read P(j): S ready -> softmax -> PV -> QK^T -> S ready is a
// serial loop of ~2.75k cycles against 2048 tensor cycles per step.
//
// Here a cluster of two CTAs runs one work item at a time as ONE M = 256 tile
// (tcgen05 cta_group::2): CTA r holds the 128 rows of the item's Q tile r, half
// of every K tile (64 keys) and half of every V tile (64 head-dim columns), so
// each CTA has a single 128-row tile in TMEM and room to decouple:
//   TMEM (per CTA, 512 columns): S_a | S_b | P_a | P_b | O
//     S double-buffered (QK^T(j+1) runs while the softmax works on S(j)),
//     P (bf16 pairs) double-buffered in its own columns (PV(j) reads P(j)
//     while the softmax writes P(j+1)); nothing waits on a serial loop.
//   softmax: two warpgroups per CTA, each owning 64 of the 128 key columns of
//     every row (thread = row = TMEM lane, as before), so each SM sub-partition
//     runs two softmax warps on the tile; the row max is exchanged between
//     the pair of warps through shared memory every step, the row sums are
//     kept per half and added in the epilogue.
//   epilogue: a fourth warpgroup drains O (TMEM -> bf16 -> global) while the
//     softmax warpgroups and the tensor core already run the next item; the
//     next item's first PV waits only for the drain (o_free).
//
//   warp 0      producer (both CTAs): Q tile (double-buffered by item), K/V
//               halves into a 4-stage ring; TMA completes on the leader's
//               barriers.  The leader's also fetches items (dynamic,
//               group-major schedule) and writes them to both CTAs' rings.
//   warp 1      MMA issuer (leader CTA): QK^T(j) then PV(j-1), cta_group::2
//   warp 2      TMEM allocator (cta_group::2, both CTAs)
//   warps 4-7   softmax, key columns 0-63;  warps 8-11  key columns 64-127
//   warps 12-15 epilogue
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace parse {
using namespace parse_sm100;

namespace {

constexpr int kThreadsP = 512;
constexpr int kQBytesP = 128 * 128 * 2;        // one Q tile (2 SW128 atoms of 128 rows x 128 B)
constexpr int kKHalfP = 64 * 128 * 2;          // 64 keys x 128 d  (2 atoms of 64 rows x 128 B)
constexpr int kVHalfP = 128 * 64 * 2;          // 128 keys x 64 d  (1 atom of 128 rows x 128 B)
constexpr int kStageP = kKHalfP + kVHalfP;     // one K/V step of this CTA
#ifndef PARSE_PAIR_STAGES
constexpr int kStagesP = 4;
#else
constexpr int kStagesP = PARSE_PAIR_STAGES;
#endif
constexpr int kRingP = 4;
constexpr int kQOffP = 0;                      // Q buffers 0, 1
constexpr int kKVOffP = 2 * kQBytesP;
constexpr int kMxOffP = kKVOffP + kStagesP * kStageP;           // float mshare[2][128]
constexpr int kStatOffP = kMxOffP + 2 * 128 * 4;                // float lsum[2][2][128], mlast[2][2][128]
constexpr int kBarOffP = kStatOffP + 2 * 4 * 128 * 4;
// barriers: q_full[2] q_empty[2] s_full[2] s_free[2] p_full[2] p_empty[2] o_full o_free
//           stats_full[2] stats_empty[2] kv_full[S] kv_empty[S] item_full[R] item_empty[R] m_ready[2][4]
constexpr int kNumBarsP = 18 + 2 * kStagesP + 2 * kRingP + 8;
constexpr int kItemOffP = (kBarOffP + kNumBarsP * 8 + 15) / 16 * 16;
constexpr int kSmemP = kItemOffP + 64 * kRingP + 16 + 1024;
static_assert(kSmemP <= 232448, "shared memory budget");
constexpr int kSColP = 0;      // S_a at 0, S_b at 128
constexpr int kPColP = 256;    // P_a at 256, P_b at 320 (64 columns: bf16 pairs of 128 keys)
constexpr int kOColP = 384;    // O: 128 columns
constexpr float kThreshP = 8.0f;   // lazy rescale threshold (log2 units), as attn_sm100_kernel
constexpr uint16_t kBothP = 3;
#ifdef PARSE_TRACE
// clock64 timeline of cluster 0 (tools/trace_pair.py): trace[(role * 1024 + step) * 8 + event]
#define TRP(cond, role, step, e) \
  if ((cond) && blockIdx.x < 2 && prm.trace && (step) < 1024) prm.trace[((role) * 1024 + (step)) * 8 + (e)] = clock64();
#else
#define TRP(cond, role, step, e)
#endif

struct BarsP {
  uint32_t base;
  __device__ uint32_t q_full(int b) const { return base + 8 * (0 + b); }
  __device__ uint32_t q_empty(int b) const { return base + 8 * (2 + b); }
  __device__ uint32_t s_full(int b) const { return base + 8 * (4 + b); }
  __device__ uint32_t s_free(int b) const { return base + 8 * (6 + b); }
  __device__ uint32_t p_full(int b) const { return base + 8 * (8 + b); }
  __device__ uint32_t p_empty(int b) const { return base + 8 * (10 + b); }
  __device__ uint32_t o_full() const { return base + 8 * 12; }
  __device__ uint32_t o_free() const { return base + 8 * 13; }
  __device__ uint32_t stats_full(int b) const { return base + 8 * (14 + b); }
  __device__ uint32_t stats_empty(int b) const { return base + 8 * (16 + b); }
  __device__ uint32_t kv_full(int s) const { return base + 8 * (18 + s); }
  __device__ uint32_t kv_empty(int s) const { return base + 8 * (18 + kStagesP + s); }
  __device__ uint32_t item_full(int r) const { return base + 8 * (18 + 2 * kStagesP + r); }
  __device__ uint32_t item_empty(int r) const { return base + 8 * (18 + 2 * kStagesP + kRingP + r); }
  // max in use after a step of parity b, posted by warp quad of that step's warpgroup
  __device__ uint32_t m_ready(int b, int quad) const { return base + 8 * (18 + 2 * kStagesP + 2 * kRingP + 4 * b + quad); }
};

// ------------------------------ cluster PTX --------------------------------
__device__ __forceinline__ uint32_t cta_rank_p() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_p() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank_p(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// Wait on a barrier that receives arrivals from the other CTA (acquire at
// cluster scope); watchdog as mbar_wait.
__device__ __forceinline__ void mbar_wait_acq_cl(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  long long t0 = 0;
  uint32_t polls = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(kSuspendHint)
        : "memory");
    if (ok) return;
    if (polls == 0) t0 = clock64();
    if ((++polls & 255u) == 0 && clock64() - t0 > (1ll << 32)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Per-step hand-offs of TMEM data (S read, P written, O read) to the leader's
// MMA warp.  The data's ordering comes from the tcgen05 side: the thread has
// completed its tcgen05.ld / tcgen05.st (wait::ld / wait::st) and issued
// tcgen05.fence::before_thread_sync; the leader waits with acquire.cluster and
// issues tcgen05.fence::after_thread_sync before its MMA.  A release at cluster
// scope would also drain this thread's generic memory operations, which the
// MMA does not read (measured ~1k cycles per arrive).
__device__ __forceinline__ void mbar_arrive_remote_tc(uint32_t cluster_addr) {
#ifdef PARSE_PAIR_RELEASE
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
__device__ __forceinline__ void st_cluster_v4_p(uint32_t cluster_addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// TMA into this CTA's shared memory, transaction bytes on the leader's barrier
__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1,
                                                 int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar & 0xFEFFFFFFu), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma2_ss_p(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts_p(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2_p(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, %1;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar),
      "h"(kBothP)
      : "memory");
}

__device__ __forceinline__ int item_hpt_p(const WorkItem& w) { return w.flags & 0xff; }
__device__ __forceinline__ int item_nq_p(const WorkItem& w) { return (w.flags >> 8) & 1 ? 2 : 1; }
__device__ __forceinline__ int tile_t0_p(const WorkItem& w, int i, int S) { return w.t0 + ((w.flags >> 9) & 1 ? i * S : 0); }
__device__ __forceinline__ int tile_h0_p(const WorkItem& w, int i) {
  return w.h0 + ((w.flags >> 9) & 1 ? 0 : i * item_hpt_p(w));
}
__device__ __forceinline__ int kv_key0_p(const WorkItem& w, int j) {
  return j < w.n_draft ? j * kTile : w.self_lo + (j - w.n_draft) * kTile;
}
__device__ __forceinline__ ReqDesc load_req_p(const AttnParams& prm, int b) {
  if (prm.dense_L) return ReqDesc{prm.dense_N, prm.dense_L, prm.dense_K, b * prm.dense_K, 0, 0, b, 0};
  return prm.req[b];
}

// exp2 of a pair on the FMA pipe (degree-3 minimax, see attn_sm100.cu)
__device__ __forceinline__ float2 exp2_poly_p(float2 x) {
  constexpr float kMagic = 12582912.f + 127.f;
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = fadd2(x, make_float2(kMagic, kMagic));
  const float2 r = fadd2(t, make_float2(-kMagic, -kMagic));
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(f, make_float2(0.05517172813f, 0.05517172813f), make_float2(0.24261118472f, 0.24261118472f));
  p = ffma2(p, f, make_float2(0.69326096773f, 0.69326096773f));
  p = ffma2(p, f, make_float2(0.99992805719f, 0.99992805719f));
  const float2 scale = make_float2(__uint_as_float(__float_as_uint(t.x) << 23), __uint_as_float(__float_as_uint(t.y) << 23));
  return fmul2(p, scale);
}
#ifndef PARSE_PAIR_POLY
constexpr int kPolyPer16P = 6;   // of every 16 exp pairs on the FMA pipe (rest: MUFU.EX2)
#else
constexpr int kPolyPer16P = PARSE_PAIR_POLY;
#endif

struct alignas(16) RingEntryP {
  WorkItem w;
  ReqDesc r;
};
static_assert(sizeof(RingEntryP) == 64, "ring entry is 64 bytes");

// Take the next ring entry; one arrive per warp on the leader's item_empty.
__device__ __forceinline__ bool next_item_p(const BarsP& bars, const RingEntryP* ring, int& slot, uint32_t& phase,
                                            RingEntryP& e, bool leader, uint32_t leader_item_empty0) {
  mbar_wait_acq_cl(bars.item_full(slot), phase);
  e = ring[slot];
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    if (leader) mbar_arrive(bars.item_empty(slot));
    else mbar_arrive_remote(leader_item_empty0 + 8 * slot);
  }
  if (++slot == kRingP) { slot = 0; phase ^= 1; }
  return e.w.n_draft >= 0;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsP, 1)
    attn_pair_kernel(const __grid_constant__ AttnParams prm, const __grid_constant__ CUtensorMap tm_q_tok,
                     const __grid_constant__ CUtensorMap tm_q_pack, const __grid_constant__ CUtensorMap tm_k64,
                     const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank_p();
  const bool leader = rank == 0;
  BarsP bars{sbase + kBarOffP};
  RingEntryP* ring = reinterpret_cast<RingEntryP*>(smem + kItemOffP);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kItemOffP + 64 * kRingP);
  const uint32_t leader_item_empty0 = map_rank_p(bars.item_empty(0), 0);
  int ring_slot = 0;
  uint32_t ring_phase = 0;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(bars.q_full(b), 1);
      mbar_init(bars.q_empty(b), 1);
      mbar_init(bars.s_full(b), 1);
      mbar_init(bars.s_free(b), 8);       // one arrive per warp of softmax warpgroup b, both CTAs
      mbar_init(bars.p_full(b), 8);
      mbar_init(bars.p_empty(b), 1);
      mbar_init(bars.stats_full(b), 8);   // softmax warps of this CTA
      mbar_init(bars.stats_empty(b), 4);  // epilogue warps of this CTA
    }
    mbar_init(bars.o_full(), 1);
    mbar_init(bars.o_free(), 8);          // epilogue warps, both CTAs
    for (int s = 0; s < kStagesP; ++s) {
      mbar_init(bars.kv_full(s), 1);
      mbar_init(bars.kv_empty(s), 1);
    }
    for (int q = 0; q < 8; ++q) mbar_init(bars.m_ready(q >> 2, q & 3), 1);
    for (int r = 0; r < kRingP; ++r) {
      mbar_init(bars.item_full(r), 1);
      // MMA warp + peer producer + 8 + 8 softmax warps + 4 + 4 epilogue warps
      mbar_init(bars.item_empty(r), 1 + 1 + 16 + 8);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q_tok);
    tma_prefetch_desc(&tm_q_pack);
    tma_prefetch_desc(&tm_k64);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_p();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int r_heads = prm.Hq / prm.Hkv;

#ifndef PARSE_PAIR_SMX_REGS
#define PARSE_PAIR_SMX_REGS 208
#endif
#ifndef PARSE_PAIR_WG0_REGS
#define PARSE_PAIR_WG0_REGS 48
#endif
#ifndef PARSE_PAIR_EPI_REGS
#define PARSE_PAIR_EPI_REGS 48
#endif
  // register split of the launch pool (512 x 128)
  static_assert(128 * PARSE_PAIR_WG0_REGS + 256 * PARSE_PAIR_SMX_REGS + 128 * PARSE_PAIR_EPI_REGS <= 65536,
                "setmaxnreg budget");
  if (warp < 4) {
  setmaxnreg_dec<PARSE_PAIR_WG0_REGS>();
  if (warp == 0) {
    // ================================ producer ================================
    int stage = 0;
    uint32_t kv_phase = 0;
    uint32_t n_items = 0;
    const uint64_t pol_stream = make_policy_evict_first();   // Q: read once
    const uint64_t pol_keep = make_policy_evict_last();      // K/V: re-read by the group's items
    for (;; ++n_items) {
      RingEntryP e;
      if (leader) {
        int it = 0;
        if (lane == 0) it = atomicAdd(prm.counter, 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it < prm.n_items) {
          e.w = prm.items[it];
          e.r = load_req_p(prm, e.w.b);
        } else {
          e.w = WorkItem{};
          e.w.n_draft = -1;
          e.r = ReqDesc{};
        }
        mbar_wait_acq_cl(bars.item_empty(ring_slot), ring_phase ^ 1);
        if (lane == 0) {
          ring[ring_slot] = e;
          const uint32_t peer = map_rank_p(smem_u32(&ring[ring_slot]), 1);
          const uint4* src = reinterpret_cast<const uint4*>(&e);
#pragma unroll
          for (int q = 0; q < 4; ++q) st_cluster_v4_p(peer + 16 * q, src[q]);
          mbar_arrive(bars.item_full(ring_slot));
          mbar_arrive_remote(map_rank_p(bars.item_full(ring_slot), 1));
        }
        __syncwarp();
        if (++ring_slot == kRingP) { ring_slot = 0; ring_phase ^= 1; }
        if (e.w.n_draft < 0) break;
      } else {
        if (!next_item_p(bars, ring, ring_slot, ring_phase, e, false, leader_item_empty0)) break;
      }
      const WorkItem& w = e.w;
      const ReqDesc& rq = e.r;
      const int ti = item_nq_p(w) == 2 ? int(rank) : 0;      // tile of this CTA (a lone tile: both compute it)
      const int hpt = item_hpt_p(w);
      const int g = w.h0 / r_heads;
      const CUtensorMap* qm = hpt == 1 ? &tm_q_tok : &tm_q_pack;
      const int qb = n_items & 1;
      mbar_wait(bars.q_empty(qb), ((n_items >> 1) & 1) ^ 1);
      if (elect_one()) {
        if (leader) mbar_arrive_expect_tx(bars.q_full(qb), 2 * kQBytesP);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          tma_load_4d_pair(qm, bars.q_full(qb), sbase + kQOffP + qb * kQBytesP + c * 16384, c * 64, tile_h0_p(w, ti),
                           rq.q_row0 + tile_t0_p(w, ti, prm.S), rq.bcoord, pol_stream);
      }
      __syncwarp();
      const int n = w.n_draft + w.n_self;
      for (int j = 0; j < n; ++j) {
        const int key0 = kv_key0_p(w, j);
        mbar_wait(bars.kv_empty(stage), kv_phase ^ 1);
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(bars.kv_full(stage), 2 * kStageP);
          const uint32_t dst = sbase + kKVOffP + stage * kStageP;
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d_pair(&tm_k64, bars.kv_full(stage), dst + c * 8192, c * 64, g,
                             rq.kv_row0 + key0 + 64 * int(rank), rq.bcoord, pol_keep);
          tma_load_4d_pair(&tm_v, bars.kv_full(stage), dst + kKHalfP, 64 * int(rank), g, rq.kv_row0 + key0, rq.bcoord,
                           pol_keep);
        }
        __syncwarp();
        if (++stage == kStagesP) { stage = 0; kv_phase ^= 1; }
      }
    }
  } else if (warp == 1 && leader) {
    // ============================ MMA issuer (leader) ===========================
    constexpr uint32_t idesc_qk = make_idesc_bf16(256, 128, 0);
    constexpr uint32_t idesc_pv = make_idesc_bf16(256, 128, 1);
    const uint64_t qdesc0 = make_sdesc_sw128(sbase + kQOffP, 16, 1024);
    const uint64_t kdesc0 = make_sdesc_sw128(sbase + kKVOffP, 16, 1024);
    const uint64_t vdesc0 = make_sdesc_sw128(sbase + kKVOffP + kKHalfP, 8192, 1024);
    int stage = 0;
    uint32_t kv_phase = 0;
    uint32_t g = 0;          // global step counter (S / P buffer = g & 1, use = g >> 1)
    uint32_t n_items = 0;
    for (;; ++n_items) {
      RingEntryP e;
      if (!next_item_p(bars, ring, ring_slot, ring_phase, e, true, leader_item_empty0)) break;
      const WorkItem& w = e.w;
      const int n = w.n_draft + w.n_self;
      const int qb = n_items & 1;
      mbar_wait(bars.q_full(qb), (n_items >> 1) & 1);
      const uint64_t qdesc = qdesc0 + uint64_t((qb * kQBytesP) >> 4);
      const int stage0 = stage;
      const uint32_t phase0 = kv_phase;
      auto st_of = [&](int j) { return (stage0 + j) % kStagesP; };
      auto ph_of = [&](int j) { return phase0 ^ uint32_t(((stage0 + j) / kStagesP) & 1); };
      for (int j = 0; j <= n; ++j) {
        if (j < n) {
          // QK^T(j) -> S_(g+j)&1 once both CTAs' softmax have read its previous contents
          const uint32_t gs = g + j, sb = gs & 1;
          TRP(lane == 0, 0, gs, 0);
          mbar_wait_acq_cl(bars.s_free(sb), ((gs >> 1) & 1) ^ 1);
          TRP(lane == 0, 0, gs, 1);
          mbar_wait(bars.kv_full(st_of(j)), ph_of(j));
          TRP(lane == 0, 0, gs, 2);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t kd = kdesc0 + uint64_t((st_of(j) * kStageP) >> 4);
            const uint32_t s_tm = tmem + kSColP + sb * 128;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t qoff = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
              const uint64_t koff = uint64_t(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
              mma2_ss_p(s_tm, qdesc + qoff, kd + koff, idesc_qk, kk > 0);
            }
            commit2_p(bars.s_full(sb));
            if (j == n - 1) commit2_p(bars.q_empty(qb));
          }
          __syncwarp();
          TRP(lane == 0, 0, gs, 3);
        }
        if (j >= 1) {
          // PV(j-1): O += P_(g+j-1)&1 . V_half
          const uint32_t gp = g + j - 1, pb = gp & 1;
          TRP(lane == 0, 0, gp, 4);
          mbar_wait_acq_cl(bars.p_full(pb), (gp >> 1) & 1);
          TRP(lane == 0, 0, gp, 5);
          if (j == 1) mbar_wait_acq_cl(bars.o_free(), (n_items & 1) ^ 1);   // previous item's O drained
          TRP(lane == 0, 0, gp, 6);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t vd = vdesc0 + uint64_t((st_of(j - 1) * kStageP) >> 4);
            const uint32_t p_tm = tmem + kPColP + pb * 64;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma2_ts_p(tmem + kOColP, p_tm + kk * 8, vd + uint64_t((kk * 2048) >> 4), idesc_pv, (j > 1 || kk > 0) ? 1u : 0u);
            commit2_p(bars.p_empty(pb));
            commit2_p(bars.kv_empty(st_of(j - 1)));
            if (j == n) commit2_p(bars.o_full());
          }
          __syncwarp();
        }
      }
      g += n;
      const int adv = stage0 + n;
      kv_phase = phase0 ^ uint32_t((adv / kStagesP) & 1);
      stage = adv % kStagesP;
    }
  }
  } else if (warp < 12) {
    setmaxnreg_inc<PARSE_PAIR_SMX_REGS>();
    // ============================ softmax (step parity wg) ============================
    // Warpgroup wg runs the steps g with g % 2 == wg on S buffer wg and writes
    // P buffer wg; thread = row = TMEM lane, all 128 key columns.  The online
    // softmax's running max is handed from each step to the next through
    // shared memory (mshare, m_ready): the step-g warpgroup posts the max in
    // use right after its max phase, the step-(g+1) one waits for it before
    // exponentiating, so both warpgroups use one max sequence and their
    // P tiles accumulate into one O.  Each keeps its own row sum (rescaled
    // when the max moves); the epilogue adds the two.
    const int wg = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;             // = TMEM lane
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    float* mshare = reinterpret_cast<float*>(smem + kMxOffP);      // [2 step parity][128]
    float* stat = reinterpret_cast<float*>(smem + kStatOffP);      // lsum [2][2][128], mlast [2][2][128]
    const uint32_t s_free_l = map_rank_p(bars.s_free(wg), 0);
    const uint32_t p_full_l = map_rank_p(bars.p_full(wg), 0);
    const uint32_t tS = tmem + lane_base + kSColP + wg * 128;
    const uint32_t tP = tmem + lane_base + kPColP + wg * 64;
    const uint32_t tO = tmem + lane_base + kOColP;
    const float sl2 = prm.scale_log2;
    uint32_t g = 0;              // global step counter (all steps, both warpgroups)
    uint32_t n_items = 0;
    auto arrive_leader = [&](uint32_t remote, uint32_t local) {
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(local);
        else mbar_arrive_remote_tc(remote);
      }
    };
    for (;; ++n_items) {
      RingEntryP e;
      if (!next_item_p(bars, ring, ring_slot, ring_phase, e, leader, leader_item_empty0)) break;
      const WorkItem& w = e.w;
      const ReqDesc& rq = e.r;
      const int ti = item_nq_p(w) == 2 ? int(rank) : 0;
      const int hpt = item_hpt_p(w);
      const int n = w.n_draft + w.n_self;
      const int t = tile_t0_p(w, ti, prm.S) + row / hpt;
      // visibility of this row: keys [0, lim) of the shared region,
      // plus own-copy keys [sbase_k, t] (or tree ancestors of sidx)
      int lim, sbase_k = 0x7fffffff, sidx = 0;
      if (t < rq.N) {
        lim = t + 1;
      } else if (t < rq.L) {
        const int k = (t - rq.N) / prm.S;
        sidx = t - rq.N - k * prm.S;
        lim = prm.bnd[rq.bnd_off + k];
        sbase_k = rq.N + k * prm.S;
      } else {
        lim = 0;
      }
      const uint64_t anc_row = prm.anc ? prm.anc[sidx] : 0ull;
      float m_last = -INFINITY, l_sum = 0.f;     // this warpgroup's max in use and row sum
      for (int j = (int(g) & 1) == wg ? 0 : 1; j < n; j += 2) {
        const uint32_t gs = g + j;
        const uint32_t u = gs >> 1;               // use index of buffers wg
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 0);
        mbar_wait(bars.s_full(wg), u & 1);
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 1);
        tc_fence_after();
        uint32_t sr[kTile];
        tmem_ld64(tS, sr);
        tmem_ld64(tS + 64, sr + 64);
        tmem_wait_ld();
        reg_fence<kTile>(sr);
        tc_fence_before();
        arrive_leader(s_free_l, bars.s_free(wg));   // S_wg may be overwritten by QK^T(gs + 2)
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 2);
        const int key0 = kv_key0_p(w, j);
        bool masked = true;
        if (j < w.n_draft) {
          const int nvis = lim - key0;           // keys [key0, lim) visible
          masked = nvis < kTile;
          if (masked) {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c >= nvis) sr[c] = 0xff800000u;   // -inf
          }
        } else {
          const int lo = sbase_k - key0;         // own copy starts at column lo
          const int hi = t - key0;               // causal: columns <= hi
          if (prm.anc) {
#pragma unroll
            for (int c = 0; c < kTile; ++c) {
              const int rel = c - lo;
              const bool vis = rel >= 0 && rel < 64 && ((anc_row >> (rel & 63)) & 1ull);
              if (!vis) sr[c] = 0xff800000u;
            }
          } else {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c < lo || c > hi) sr[c] = 0xff800000u;
          }
        }
        float mxs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float m = fmax3(__uint_as_float(sr[16 * i]), __uint_as_float(sr[16 * i + 1]), __uint_as_float(sr[16 * i + 2]));
#pragma unroll
          for (int e2 = 3; e2 < 15; e2 += 2) m = fmax3(m, __uint_as_float(sr[16 * i + e2]), __uint_as_float(sr[16 * i + e2 + 1]));
          mxs[i] = fmaxf(m, __uint_as_float(sr[16 * i + 15]));
        }
        const float m_tile =
            fmaxf(fmax3(mxs[0], mxs[1], mxs[2]), fmax3(fmax3(mxs[3], mxs[4], mxs[5]), mxs[6], mxs[7])) * sl2;
        // the max in use after step gs - 1 (the other warpgroup's step)
        float m_in = -INFINITY;
        if (gs > 0) {
          const uint32_t gp = gs - 1;
          mbar_wait(bars.m_ready(gp & 1, quad), (gp >> 1) & 1);
          if (j > 0) m_in = mshare[(gp & 1) * 128 + row];
        }
        const float m_new = m_tile > m_in + kThreshP ? m_tile : m_in;   // lazy rescale (log2 units)
        const bool rescale_o = m_new != m_in && m_in != -INFINITY;
        mshare[(gs & 1) * 128 + row] = m_new;
        __syncwarp();
        if (lane == 0) mbar_arrive(bars.m_ready(gs & 1, quad));
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 3);
        if (m_last != -INFINITY && m_new != m_last) l_sum *= ex2(m_last - m_new);
        m_last = m_new;
        const bool any_rescale = __any_sync(0xffffffffu, rescale_o);
        const float m_eff = (m_new == -INFINITY) ? 0.f : m_new;
        const float2 sl2x2 = make_float2(sl2, sl2);
        const float2 negm = make_float2(-m_eff, -m_eff);
        const bool all_full = __all_sync(0xffffffffu, !masked);
#pragma unroll
        for (int e2 = 0; e2 < kTile / 2; ++e2) {
          const float2 x = ffma2(make_float2(__uint_as_float(sr[2 * e2]), __uint_as_float(sr[2 * e2 + 1])), sl2x2, negm);
          sr[2 * e2] = __float_as_uint(x.x);
          sr[2 * e2 + 1] = __float_as_uint(x.y);
        }
        if (all_full) {
#pragma unroll
          for (int e2 = 0; e2 < kTile / 2; ++e2) {
            const float2 x = make_float2(__uint_as_float(sr[2 * e2]), __uint_as_float(sr[2 * e2 + 1]));
            const float2 pp = (e2 & 15) >= 16 - kPolyPer16P ? exp2_poly_p(x) : make_float2(ex2(x.x), ex2(x.y));
            sr[2 * e2] = __float_as_uint(pp.x);
            sr[2 * e2 + 1] = __float_as_uint(pp.y);
          }
        } else {
#pragma unroll
          for (int e2 = 0; e2 < kTile; ++e2) sr[e2] = __float_as_uint(ex2(__uint_as_float(sr[e2])));
        }
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 4);
        // P_wg may be overwritten once PV(gs - 2) has read it
        mbar_wait(bars.p_empty(wg), (u & 1) ^ 1);
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 5);
        float2 acc[4];
#pragma unroll
        for (int e0 = 0; e0 < kTile / 2; e0 += 16) {
          uint32_t pk[16];
#pragma unroll
          for (int e2 = 0; e2 < 16; ++e2) {
            const float2 pp = make_float2(__uint_as_float(sr[2 * (e0 + e2)]), __uint_as_float(sr[2 * (e0 + e2) + 1]));
            if (e0 == 0 && e2 < 4) acc[e2] = pp;
            else acc[e2 & 3] = fadd2(acc[e2 & 3], pp);
            pk[e2] = pack_bf16x2(pp.x, pp.y);
          }
          tmem_st16(tP + e0, pk);
        }
        if (any_rescale) {
          // rare: O must hold PV(gs - 1) before it is rescaled, and the rescale
          // must land before PV(gs) (p_full below)
          const uint32_t gp = gs - 1;
          mbar_wait(bars.p_empty(wg ^ 1), (gp >> 1) & 1);
          tc_fence_after();
          const float alpha = rescale_o ? ex2(m_in - m_new) : 1.f;
          const float2 al2 = make_float2(alpha, alpha);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ro[32];
            tmem_ld32(tO + c * 32, ro);
            tmem_wait_ld();
            reg_fence<32>(ro);
#pragma unroll
            for (int e2 = 0; e2 < 32; e2 += 2) {
              const float2 vv = fmul2(make_float2(__uint_as_float(ro[e2]), __uint_as_float(ro[e2 + 1])), al2);
              ro[e2] = __float_as_uint(vv.x);
              ro[e2 + 1] = __float_as_uint(vv.y);
            }
            tmem_st32(tO + c * 32, ro);
          }
        }
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        l_sum += a.x + a.y;
        tmem_wait_st();
        tc_fence_before();
        arrive_leader(p_full_l, bars.p_full(wg));
        TRP(quad == 0 && lane == 0, 1 + 2 * wg + rank, u, 6);
      }
      g += n;
      // row statistics of this item for the epilogue (double-buffered by item)
      const int ib = n_items & 1;
      mbar_wait(bars.stats_empty(ib), ((n_items >> 1) & 1) ^ 1);
      stat[(ib * 2 + wg) * 128 + row] = l_sum;
      stat[512 + (ib * 2 + wg) * 128 + row] = m_last;
      __syncwarp();
      if (lane == 0) mbar_arrive(bars.stats_full(ib));
    }
  } else {
    setmaxnreg_dec<PARSE_PAIR_EPI_REGS>();
    // ================================ epilogue ================================
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const float* stat = reinterpret_cast<const float*>(smem + kStatOffP);
    const uint32_t o_free_l = map_rank_p(bars.o_free(), 0);
    const uint64_t pol_out = make_policy_evict_first();
    uint32_t n_items = 0;
    for (;; ++n_items) {
      RingEntryP e;
      if (!next_item_p(bars, ring, ring_slot, ring_phase, e, leader, leader_item_empty0)) break;
      const WorkItem& w = e.w;
      const ReqDesc& rq = e.r;
      const bool lone = item_nq_p(w) == 1;
      const int ti = lone ? 0 : int(rank);
      const int hpt = item_hpt_p(w);
      const int t = tile_t0_p(w, ti, prm.S) + row / hpt;
      const int h = tile_h0_p(w, ti) + row % hpt;
      const bool row_valid = (leader || !lone) && t < w.t_end;
      const int ib = n_items & 1;
      mbar_wait(bars.stats_full(ib), (n_items >> 1) & 1);
      const float l0 = stat[(ib * 2) * 128 + row], l1 = stat[(ib * 2 + 1) * 128 + row];
      const float m0 = stat[512 + (ib * 2) * 128 + row], m1 = stat[512 + (ib * 2 + 1) * 128 + row];
      __syncwarp();
      if (lane == 0) mbar_arrive(bars.stats_empty(ib));
      // both halves' sums relative to the final max (the max only grows)
      const float m = fmaxf(m0, m1);
      const float l = m == -INFINITY ? 0.f
                                     : (m0 == -INFINITY ? 0.f : l0 * ex2(m0 - m)) + (m1 == -INFINITY ? 0.f : l1 * ex2(m1 - m));
      TRP(quad == 0 && lane == 0, 5 + rank, n_items, 0);
      mbar_wait(bars.o_full(), n_items & 1);
      TRP(quad == 0 && lane == 0, 5 + rank, n_items, 1);
      tc_fence_after();
      const float inv_l = l > 0.f ? prm.o_scale / l : 0.f;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.o) + rq.bcoord * prm.o_s0 +
                            int64_t(rq.q_row0 + t) * prm.o_s1 + int64_t(h) * prm.o_s2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t raw[32];
        tmem_ld32(tmem + lane_base + kOColP + c * 32, raw);
        tmem_wait_ld();
        reg_fence<32>(raw);
        if (c == 3) {
          // O may be overwritten by the next item's first PV
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(bars.o_free());
            else mbar_arrive_remote_tc(o_free_l);
          }
        }
        uint32_t pk[16];
#pragma unroll
        for (int e2 = 0; e2 < 16; ++e2)
          pk[e2] = pack_bf16x2(__uint_as_float(raw[2 * e2]) * inv_l, __uint_as_float(raw[2 * e2 + 1]) * inv_l);
        if (row_valid) {
          if (prm.o_v8) {
            st_global_v8_hint(orow + c * 32, pk, pol_out);
            st_global_v8_hint(orow + c * 32 + 16, pk + 8, pol_out);
          } else {
            uint4* d4 = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_global_v4_hint(d4 + q, make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]), pol_out);
          }
        }
      }
      TRP(quad == 0 && lane == 0, 5 + rank, n_items, 2);
      if (row_valid && prm.lse)
        prm.lse[rq.bcoord * prm.lse_sb + h * prm.lse_sh + rq.q_row0 + t] = (m + __log2f(l)) * 0.69314718055994531f;
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_p();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace

cudaError_t launch_attn_pair(const AttnParams& prm, const CUtensorMap& tm_q_tok, const CUtensorMap& tm_q_pack,
                             const CUtensorMap& tm_k64, const CUtensorMap& tm_v, int num_sms, cudaStream_t stream) {
  cudaError_t e = opt_in_smem<attn_pair_kernel>(kSmemP);
  if (e != cudaSuccess) return e;
  int clusters = num_sms / 2;
  if (prm.n_items < clusters) clusters = prm.n_items;
  if (clusters <= 0) return cudaSuccess;
  attn_pair_kernel<<<2 * clusters, kThreadsP, kSmemP, stream>>>(prm, tm_q_tok, tm_q_pack, tm_k64, tm_v);
  return cudaGetLastError();
}

}  // namespace parse
