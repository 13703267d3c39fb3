// parse_verify_attn, bf16, head_dim 128: the 2-SM (cta_group::2) variant of
// attn_sm100_kernel with a decoupled S -> P -> PV pipeline.
//
// A cluster of two CTAs runs one work item (two Q tiles of identical
// visibility): CTA r owns Q tile r.  Every tcgen05.mma is issued by the
// leader CTA with cta_group::2 (M = 256 = both CTAs' tiles); each CTA holds
// only half of every K tile (64 keys) and half of every V tile (64 of the 128
// head-dim columns), so a 32 KB stage carries a whole K/V step and six steps
// fit beside the Q tile.  TMEM per CTA: S0 | S1 | O (128 columns each) — S is
// double-buffered, so QK^T(j+2) can be queued behind PV(j) and the softmax of
// step j+1 starts as soon as it finishes step j (no wait for PV + QK^T).
//
//   warp 0      producer (both CTAs): Q tile, then K/V halves, TMA completing
//               on the leader's barriers; the leader's also fetches items and
//               writes them to both CTAs' item rings
//   warp 1      MMA issuer (leader CTA only)
//   warp 2      TMEM allocator (cta_group::2)
//   warps 4-11  softmax: 8 warps per tile, thread = 2 rows x 32 columns (the
//               16x256b TMEM shape), row max / sum over the row's 4 threads
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace parse {
using namespace parse_sm100;

namespace {

constexpr int kThreads2 = 384;
constexpr int kStages2 = 6;
constexpr int kQBytes = 128 * 128 * 2;      // one Q tile
constexpr int kKHalf = 64 * 128 * 2;        // 64 keys x 128 d
constexpr int kVHalf = 128 * 64 * 2;        // 128 keys x 64 d
constexpr int kStageBytes = kKHalf + kVHalf;
constexpr int kQOff2 = 0;
constexpr int kKVOff2 = kQBytes;
constexpr int kBarOff2 = kKVOff2 + kStages2 * kStageBytes;
constexpr int kRing2 = 4;
// barriers: q_full q_empty s_full[2] p_part[2] p_full[2] o_full o_done kv_full[S] kv_empty[S] item_full[R] item_empty[R]
constexpr int kNumBars2 = 10 + 2 * kStages2 + 2 * kRing2;
constexpr int kItemOff2 = (kBarOff2 + kNumBars2 * 8 + 15) / 16 * 16;
constexpr int kXOff2 = kItemOff2 + 64 * kRing2 + 16;            // row l / m exchange (2 x 128 floats)
constexpr int kSmem2 = kXOff2 + 2 * 128 * 4 + 1024;
constexpr int kSCol2 = 0, kOCol2 = 256;
constexpr float kThresh2 = 8.0f;
constexpr uint16_t kBoth = 3;                // multicast mask: both CTAs
#ifdef PARSE_TRACE
#define TR2(cond, role, step, e) \
  if ((cond) && blockIdx.x < 2 && prm.trace && (step) < 1024) prm.trace[((role) * 1024 + (step)) * 8 + (e)] = clock64();
#else
#define TR2(cond, role, step, e)
#endif

struct Bars2 {
  uint32_t base;
  __device__ uint32_t q_full() const { return base; }
  __device__ uint32_t q_empty() const { return base + 8; }
  __device__ uint32_t s_full(int i) const { return base + 8 * (2 + i); }
  __device__ uint32_t p_part(int i) const { return base + 8 * (4 + i); }
  __device__ uint32_t p_full(int i) const { return base + 8 * (6 + i); }
  __device__ uint32_t o_full() const { return base + 8 * 8; }
  __device__ uint32_t o_done() const { return base + 8 * 9; }
  __device__ uint32_t kv_full(int s) const { return base + 8 * (10 + s); }
  __device__ uint32_t kv_empty(int s) const { return base + 8 * (10 + kStages2 + s); }
  __device__ uint32_t item_full(int r) const { return base + 8 * (10 + 2 * kStages2 + r); }
  __device__ uint32_t item_empty(int r) const { return base + 8 * (10 + 2 * kStages2 + kRing2 + r); }
};

struct alignas(16) RingEntry2 {
  WorkItem w;
  ReqDesc r;
};

// ------------------------------ cluster PTX --------------------------------
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// wait on a local barrier that receives arrivals from the other CTA (acquire at cluster scope)
__device__ __forceinline__ void mbar_wait_cl(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  uint32_t polls = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(0x100000u)
        : "memory");
    if (ok) return;
    if ((++polls & 255u) == 0 && clock64() - t0 > (1ll << 32)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// for hand-offs whose data is ordered by tcgen05 fences (P in TMEM), not by generic memory
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
#ifdef PARSE_2SM_RELEASE
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#else
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
#endif
}
__device__ __forceinline__ void st_cluster_v4(uint32_t cluster_addr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// TMA into this CTA's shared memory, transaction bytes counted on the leader's barrier
__device__ __forceinline__ void tma_load_4d_2sm(const CUtensorMap* map, uint32_t bar, uint32_t dst, int c0, int c1,
                                                int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar & 0xFEFFFFFFu), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, %1;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar),
      "h"(kBoth)
      : "memory");
}

__device__ __forceinline__ int item_hpt2(const WorkItem& w) { return w.flags & 0xff; }
__device__ __forceinline__ int item_nq2(const WorkItem& w) { return (w.flags >> 8) & 1 ? 2 : 1; }
__device__ __forceinline__ int tile_t0_2(const WorkItem& w, int i, int S) { return w.t0 + ((w.flags >> 9) & 1 ? i * S : 0); }
__device__ __forceinline__ int tile_h0_2(const WorkItem& w, int i) { return w.h0 + ((w.flags >> 9) & 1 ? 0 : i * item_hpt2(w)); }
__device__ __forceinline__ int kv_key0_2(const WorkItem& w, int j) {
  return j < w.n_draft ? j * kTile : w.self_lo + (j - w.n_draft) * kTile;
}
__device__ __forceinline__ ReqDesc load_req2(const AttnParams& prm, int b) {
  if (prm.dense_L) return ReqDesc{prm.dense_N, prm.dense_L, prm.dense_K, b * prm.dense_K, 0, 0, b, 0};
  return prm.req[b];
}

// exp2 on the FMA pipe (see attn_sm100.cu)
__device__ __forceinline__ float2 exp2_poly2b(float2 x) {
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
template <bool kPoly, int E0, int E1>
__device__ __forceinline__ void exp_pairs2(uint32_t* sr) {
#pragma unroll
  for (int e = E0; e < E1; ++e) {
    const float2 x = make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1]));
    const float2 pp = (kPoly && (e & 15) >= 10) ? exp2_poly2b(x) : make_float2(ex2(x.x), ex2(x.y));
    sr[2 * e] = __float_as_uint(pp.x);
    sr[2 * e + 1] = __float_as_uint(pp.y);
  }
}
// P of reps k in [K0, K1) (both rows) -> bf16 pairs, 16x128b stores
template <int K0, int K1>
__device__ __forceinline__ void store_p_quads2(const uint32_t* sr, uint32_t tS, float2 (&acc)[2]) {
  uint32_t pk[2 * (K1 - K0)];
#pragma unroll
  for (int k = K0; k < K1; ++k)
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const float2 pp = make_float2(__uint_as_float(sr[4 * k + 2 * rr]), __uint_as_float(sr[4 * k + 2 * rr + 1]));
      if (k == 0) acc[rr] = pp;
      else acc[rr] = fadd2(acc[rr], pp);
      pk[2 * (k - K0) + rr] = pack_bf16x2(pp.x, pp.y);
    }
  if constexpr (K1 - K0 == 12) {
    tmem_st_16x128b_x8(tS + 4 * K0, pk);
    tmem_st_16x128b_x4(tS + 4 * K0 + 32, pk + 16);
  } else {
    tmem_st_16x128b_x4(tS + 4 * K0, pk);
  }
}

template <int kRing>
__device__ __forceinline__ bool next_item2(const Bars2& bars, const RingEntry2* ring, int& slot, uint32_t& phase,
                                           WorkItem& w, ReqDesc& r, uint32_t leader_item_empty_base, bool leader) {
  mbar_wait_cl(bars.item_full(slot), phase);
  w = ring[slot].w;
  r = ring[slot].r;
  __syncwarp();
  // release the slot on the leader's ring (only the leader's producer refills): one arrive per warp
  if ((threadIdx.x & 31) == 0) {
    if (leader) mbar_arrive(bars.item_empty(slot));
    else mbar_arrive_cluster(leader_item_empty_base + 8 * slot);
  }
  if (++slot == kRing) { slot = 0; phase ^= 1; }
  return w.n_draft >= 0;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    attn_2sm_kernel(const __grid_constant__ AttnParams prm, const __grid_constant__ CUtensorMap tm_q_tok,
                    const __grid_constant__ CUtensorMap tm_q_pack, const __grid_constant__ CUtensorMap tm_k64,
                    const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  Bars2 bars{sbase + kBarOff2};
  RingEntry2* ring = reinterpret_cast<RingEntry2*>(smem + kItemOff2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kItemOff2 + 64 * kRing2);
  float* xl = reinterpret_cast<float*>(smem + kXOff2);       // row sums
  float* xm = xl + 128;                                       // row maxima
  const uint32_t leader_item_empty = map_rank(bars.item_empty(0), 0);
  int ring_slot = 0;
  uint32_t ring_phase = 0;

  if (threadIdx.x == 0) {
    mbar_init(bars.q_full(), 1);
    mbar_init(bars.q_empty(), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bars.s_full(i), 1);
      mbar_init(bars.p_part(i), 16);        // one arrive per softmax warp, both CTAs
      mbar_init(bars.p_full(i), 16);
    }
    mbar_init(bars.o_full(), 1);
    mbar_init(bars.o_done(), 1);
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(bars.kv_full(s), 1);
      mbar_init(bars.kv_empty(s), 1);
    }
    for (int r = 0; r < kRing2; ++r) {
      mbar_init(bars.item_full(r), 1);
      // one arrive per consuming warp: the leader's MMA warp, the peer's
      // producer, both CTAs' 8 softmax warps
      mbar_init(bars.item_empty(r), 1 + 1 + 8 + 8);
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
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int r_heads = prm.Hq / prm.Hkv;

  if (warp < 4) {
    setmaxnreg_dec<72>();
    if (warp == 0) {
      // =============================== producer ===============================
      int stage = 0;
      uint32_t kv_phase = 0, q_phase = 0;
      const uint64_t pol_stream = make_policy_evict_first();
      const uint64_t pol_keep = make_policy_evict_last();
      for (;;) {
        WorkItem w;
        ReqDesc rq;
        if (leader) {
          // claim the next item and publish it to both CTAs' rings
          int it = 0;
          if (lane == 0) it = atomicAdd(prm.counter, 1);
          it = __shfl_sync(0xffffffffu, it, 0);
          if (it < prm.n_items) {
            w = prm.items[it];
            rq = load_req2(prm, w.b);
          } else {
            w = WorkItem{};
            w.n_draft = -1;
            rq = ReqDesc{};
          }
          mbar_wait_cl(bars.item_empty(ring_slot), ring_phase ^ 1);
          if (lane == 0) {
            RingEntry2 e{w, rq};
            ring[ring_slot] = e;
            const uint32_t peer = map_rank(smem_u32(&ring[ring_slot]), 1);
            const uint4* src = reinterpret_cast<const uint4*>(&e);
#pragma unroll
            for (int q = 0; q < 4; ++q) st_cluster_v4(peer + 16 * q, src[q]);
            mbar_arrive(bars.item_full(ring_slot));
            mbar_arrive_cluster(map_rank(bars.item_full(ring_slot), 1));
          }
          __syncwarp();
          if (++ring_slot == kRing2) { ring_slot = 0; ring_phase ^= 1; }
          if (w.n_draft < 0) break;
        } else {
          if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, w, rq, leader_item_empty, false)) break;
        }
        const int nq = item_nq2(w);
        const int hpt = item_hpt2(w);
        const int g = w.h0 / r_heads;
        const CUtensorMap* qm = hpt == 1 ? &tm_q_tok : &tm_q_pack;
        const int qi = (nq == 2) ? int(rank) : 0;   // single-tile items: the peer recomputes tile 0, unstored
        mbar_wait(bars.q_empty(), q_phase ^ 1);
        q_phase ^= 1;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(bars.q_full(), 2 * kQBytes);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d_2sm(qm, bars.q_full(), sbase + kQOff2 + c * 16384, c * 64, tile_h0_2(w, qi),
                            rq.q_row0 + tile_t0_2(w, qi, prm.S), rq.bcoord, pol_stream);
        }
        __syncwarp();
        const int n = w.n_draft + w.n_self;
        for (int j = 0; j < n; ++j) {
          const int key0 = kv_key0_2(w, j);
          mbar_wait(bars.kv_empty(stage), kv_phase ^ 1);
          if (elect_one()) {
            if (leader) mbar_arrive_expect_tx(bars.kv_full(stage), 2 * kStageBytes);
            const uint32_t dst = sbase + kKVOff2 + stage * kStageBytes;
            // K: keys [key0 + 64 rank, +64), both 64-column chunks of d
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_4d_2sm(&tm_k64, bars.kv_full(stage), dst + c * 8192, c * 64, g, rq.kv_row0 + key0 + 64 * int(rank),
                              rq.bcoord, pol_keep);
            // V: all 128 keys, d columns [64 rank, +64)
            tma_load_4d_2sm(&tm_v, bars.kv_full(stage), dst + kKHalf, 64 * int(rank), g, rq.kv_row0 + key0, rq.bcoord,
                            pol_keep);
          }
          __syncwarp();
          if (++stage == kStages2) { stage = 0; kv_phase ^= 1; }
        }
      }
    } else if (warp == 1 && leader) {
      // ============================== MMA issuer ==============================
      constexpr uint32_t idesc_qk = make_idesc_bf16(256, 128, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(256, 128, 1);
      const uint64_t qdesc = make_sdesc_sw128(sbase + kQOff2, 16, 1024);
      const uint64_t kdesc0 = make_sdesc_sw128(sbase + kKVOff2, 16, 1024);
      const uint64_t vdesc0 = make_sdesc_sw128(sbase + kKVOff2 + kKHalf, 8192, 1024);
      int stage = 0;
      uint32_t kv_phase = 0, q_phase = 0;
      uint32_t p_phase[2] = {0, 0};
      auto issue_qk = [&](int st, int buf) {
        const uint64_t kd = kdesc0 + uint64_t((st * kStageBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t qoff = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const uint64_t koff = uint64_t(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
          mma2_ss(tmem + kSCol2 + buf * 128, qdesc + qoff, kd + koff, idesc_qk, kk > 0);
        }
      };
      auto issue_pv = [&](int st, int buf, bool acc, int kk0, int kk1) {
        const uint64_t vd = vdesc0 + uint64_t((st * kStageBytes) >> 4);
#pragma unroll
        for (int kk = kk0; kk < kk1; ++kk)
          mma2_ts(tmem + kOCol2, tmem + kSCol2 + buf * 128 + kk * 8, vd + uint64_t((kk * 2048) >> 4), idesc_pv,
                  (acc || kk > 0) ? 1u : 0u);
      };
      int mstep = 0;
      for (;;) {
        WorkItem w;
        ReqDesc rq_unused;
        if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, w, rq_unused, leader_item_empty, true)) break;
        const int n = w.n_draft + w.n_self;
        mbar_wait(bars.q_full(), q_phase);
        q_phase ^= 1;
        // stages of this item's steps follow the ring: step j -> (stage0 + j) mod kStages2
        const int stage0 = stage;
        auto st_of = [&](int j) { return (stage0 + j) % kStages2; };
        auto ph_of = [&](int j) { return kv_phase ^ uint32_t(((stage0 + j) / kStages2) & 1); };
        // prologue: QK(0) -> S0, QK(1) -> S1
        for (int j = 0; j < 2 && j < n; ++j) {
          mbar_wait(bars.kv_full(st_of(j)), ph_of(j));
          tc_fence_after();
          if (elect_one()) {
            issue_qk(st_of(j), j);
            commit2(bars.s_full(j));
            if (j == n - 1) commit2(bars.q_empty());
          }
          __syncwarp();
        }
        for (int j = 0; j < n; ++j) {
          const int buf = j & 1;
          mbar_wait_cl(bars.p_part(buf), p_phase[buf]);
          TR2(lane == 0 && blockIdx.x == 0, 0, mstep, 0);
          tc_fence_after();
          if (elect_one()) issue_pv(st_of(j), buf, j > 0, 0, 6);
          __syncwarp();
          TR2(lane == 0 && blockIdx.x == 0, 0, mstep, 1);
          mbar_wait_cl(bars.p_full(buf), p_phase[buf]);
          TR2(lane == 0 && blockIdx.x == 0, 0, mstep, 2);
          p_phase[buf] ^= 1;
          tc_fence_after();
          if (elect_one()) {
            issue_pv(st_of(j), buf, true, 6, 8);
            commit2(bars.o_full());
            if (j == n - 1) commit2(bars.o_done());
            commit2(bars.kv_empty(st_of(j)));
          }
          __syncwarp();
          TR2(lane == 0 && blockIdx.x == 0, 0, mstep, 3);
          if (j + 2 < n) {
            mbar_wait(bars.kv_full(st_of(j + 2)), ph_of(j + 2));
            tc_fence_after();
            if (elect_one()) {
              issue_qk(st_of(j + 2), buf);
              commit2(bars.s_full(buf));
              if (j + 2 == n - 1) commit2(bars.q_empty());
            }
            __syncwarp();
            TR2(lane == 0 && blockIdx.x == 0, 0, mstep, 4);
          }
          ++mstep;
        }
        // advance the ring past this item's n stages
        const int adv = stage0 + n;
        kv_phase ^= uint32_t((adv / kStages2) & 1);
        stage = adv % kStages2;
      }
    }
  } else {
    setmaxnreg_inc<216>();
    // =============================== softmax ===============================
    const int sw = warp - 4;                 // 0..7
    const int q4 = warp & 3;
    const int hh = sw >> 2;
    const int lrow0 = q4 * 32 + hh * 16 + (lane >> 2);
    const int cq = lane & 3;
    const uint32_t lane_base = uint32_t(q4 * 32 + hh * 16) << 16;
    const uint32_t tSb = tmem + lane_base + kSCol2;
    const uint32_t p_part_l[2] = {map_rank(bars.p_part(0), 0), map_rank(bars.p_part(1), 0)};
    const uint32_t p_full_l[2] = {map_rank(bars.p_full(0), 0), map_rank(bars.p_full(1), 0)};
    uint32_t s_phase[2] = {0, 0};
    uint32_t o_count = 0, item_count = 0;
    int sstep = 0;
    const float sl2 = prm.scale_log2;
    const uint64_t pol_out = make_policy_evict_first();
    // P stored by every lane (wait::st + fence), then one arrive per warp on the leader's barrier
    auto arrive_leader = [&](uint32_t cl_addr, uint32_t local_addr) {
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(local_addr);
        else mbar_arrive_cluster_relaxed(cl_addr);
      }
    };
    for (;;) {
      WorkItem w;
      ReqDesc rq;
      if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, w, rq, leader_item_empty, leader)) break;
      const int nq = item_nq2(w);
      const int ti = nq == 2 ? int(rank) : 0;
      const bool store_tile = nq == 2 || leader;
      const int hpt = item_hpt2(w);
      const int n = w.n_draft + w.n_self;
      int tr[2], lim[2], sbk[2];
      uint64_t anc[2];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int row = lrow0 + 8 * rr;
        const int t = tile_t0_2(w, ti, prm.S) + row / hpt;
        tr[rr] = t;
        int sidx = 0;
        sbk[rr] = 0x7fffffff;
        if (t < rq.N) {
          lim[rr] = t + 1;
        } else if (t < rq.L) {
          const int k = (t - rq.N) / prm.S;
          sidx = t - rq.N - k * prm.S;
          lim[rr] = prm.bnd[rq.bnd_off + k];
          sbk[rr] = rq.N + k * prm.S;
        } else {
          lim[rr] = 0;
        }
        anc[rr] = prm.anc ? prm.anc[sidx] : 0ull;
      }
      float m_used[2] = {-INFINITY, -INFINITY}, l_sum[2] = {0.f, 0.f};
      for (int j = 0; j < n; ++j) {
        const int buf = j & 1;
        const uint32_t tS = tSb + buf * 128;
        TR2(threadIdx.x == 128, 1 + rank, sstep, 0);
        mbar_wait(bars.s_full(buf), s_phase[buf]);
        TR2(threadIdx.x == 128, 1 + rank, sstep, 1);
        s_phase[buf] ^= 1;
        tc_fence_after();
        uint32_t sr[64];
        tmem_ld_16x256b_x16(tS, sr);
        tmem_wait_ld();
        reg_fence<64>(sr);
        const int key0 = kv_key0_2(w, j);
        bool masked = false;
        if (j < w.n_draft) {
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int nvis = lim[rr] - key0;
            if (nvis < kTile) {
              masked = true;
#pragma unroll
              for (int k = 0; k < 16; ++k)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                  if (8 * k + 2 * cq + e >= nvis) sr[4 * k + 2 * rr + e] = 0xff800000u;
            }
          }
        } else {
          masked = true;
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const int lo = sbk[rr] - key0;
            const int hi = tr[rr] - key0;
#pragma unroll
            for (int k = 0; k < 16; ++k)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int c = 8 * k + 2 * cq + e;
                bool vis;
                if (prm.anc) {
                  const int rel = c - lo;
                  vis = rel >= 0 && rel < 64 && ((anc[rr] >> (rel & 63)) & 1ull);
                } else {
                  vis = c >= lo && c <= hi;
                }
                if (!vis) sr[4 * k + 2 * rr + e] = 0xff800000u;
              }
          }
        }
        float mx[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          float a = fmax3(__uint_as_float(sr[2 * rr]), __uint_as_float(sr[2 * rr + 1]), __uint_as_float(sr[4 + 2 * rr]));
          float b2 = fmax3(__uint_as_float(sr[4 + 2 * rr + 1]), __uint_as_float(sr[8 + 2 * rr]), __uint_as_float(sr[8 + 2 * rr + 1]));
#pragma unroll
          for (int k = 3; k < 16; k += 2) {
            a = fmax3(a, __uint_as_float(sr[4 * k + 2 * rr]), __uint_as_float(sr[4 * k + 2 * rr + 1]));
            if (k + 1 < 16) b2 = fmax3(b2, __uint_as_float(sr[4 * (k + 1) + 2 * rr]), __uint_as_float(sr[4 * (k + 1) + 2 * rr + 1]));
          }
          mx[rr] = fmaxf(a, b2);
          mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
          mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
        }
        float alpha[2] = {1.f, 1.f};
        bool rescale_o = false;
        float2 negm[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const float m_tile = mx[rr] * sl2;
          if (m_tile > m_used[rr] + kThresh2) {
            alpha[rr] = ex2(m_used[rr] - m_tile);
            rescale_o |= (m_used[rr] != -INFINITY);
            m_used[rr] = m_tile;
          }
          const float m_eff = (m_used[rr] == -INFINITY) ? 0.f : m_used[rr];
          negm[rr] = make_float2(-m_eff, -m_eff);
        }
        const bool any_rescale = __any_sync(0xffffffffu, rescale_o);
        const bool all_full = __all_sync(0xffffffffu, !masked);
        const float2 sl2x2 = make_float2(sl2, sl2);
        TR2(threadIdx.x == 128, 1 + rank, sstep, 2);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float2 x = ffma2(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sl2x2, negm[e & 1]);
          sr[2 * e] = __float_as_uint(x.x);
          sr[2 * e + 1] = __float_as_uint(x.y);
        }
        float2 acc[2];
        if (all_full) exp_pairs2<true, 0, 24>(sr);
        else exp_pairs2<false, 0, 24>(sr);
        store_p_quads2<0, 12>(sr, tS, acc);
        if (!any_rescale) {
          tmem_wait_st();
          tc_fence_before();
          arrive_leader(p_part_l[buf], bars.p_part(buf));
          TR2(threadIdx.x == 128, 1 + rank, sstep, 3);
        }
        if (all_full) exp_pairs2<true, 24, 32>(sr);
        else exp_pairs2<false, 24, 32>(sr);
        store_p_quads2<12, 16>(sr, tS, acc);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) l_sum[rr] = fmaf(l_sum[rr], alpha[rr], acc[rr].x + acc[rr].y);
        if (any_rescale) {
          // rare: O must hold PV(j-1) before the rescale, which must land before PV(j)
          mbar_wait(bars.o_full(), (o_count + j - 1) & 1);
          tc_fence_after();
          const float2 al0 = make_float2(alpha[0], alpha[0]), al1 = make_float2(alpha[1], alpha[1]);
          const uint32_t tO = tmem + lane_base + kOCol2;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t ro[32];
            tmem_ld_16x256b_x8(tO + c * 64, ro);
            tmem_wait_ld();
            reg_fence<32>(ro);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float2 v = fmul2(make_float2(__uint_as_float(ro[2 * e]), __uint_as_float(ro[2 * e + 1])), (e & 1) ? al1 : al0);
              ro[2 * e] = __float_as_uint(v.x);
              ro[2 * e + 1] = __float_as_uint(v.y);
            }
            tmem_st_16x256b_x8(tO + c * 64, ro);
          }
          tmem_wait_st();
          tc_fence_before();
          arrive_leader(p_part_l[buf], bars.p_part(buf));
        }
        tmem_wait_st();
        tc_fence_before();
        arrive_leader(p_full_l[buf], bars.p_full(buf));
        TR2(threadIdx.x == 128, 1 + rank, sstep, 4);
        ++sstep;
      }
      // ------------------------------ epilogue ------------------------------
      // row sums and maxima to shared memory (layout: this thread holds rows
      // lrow0, lrow0 + 8), then warp (q4, hh) writes columns [64 hh, +64) of
      // its quarter's 32 rows with 32x32b loads (thread = row) and 32-byte stores
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        float l = l_sum[rr];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        if (cq == 0) {
          xl[lrow0 + 8 * rr] = l;
          xm[lrow0 + 8 * rr] = m_used[rr];
        }
      }
      named_bar_sync(1, 256);
      mbar_wait(bars.o_done(), item_count & 1);
      ++item_count;
      o_count += n;
      tc_fence_after();
      const int er = q4 * 32 + lane;                       // row of this thread in the 32x32b shape
      const float l_row = xl[er], m_row = xm[er];
      const float inv_l = l_row > 0.f ? prm.o_scale / l_row : 0.f;
      const int t_row = tile_t0_2(w, ti, prm.S) + er / hpt;
      const int h_row = tile_h0_2(w, ti) + er % hpt;
      const bool valid = store_tile && t_row < w.t_end;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.o) + rq.bcoord * prm.o_s0 +
                            int64_t(rq.q_row0 + t_row) * prm.o_s1 + int64_t(h_row) * prm.o_s2;
      const uint32_t tO32 = tmem + (uint32_t(q4 * 32) << 16) + kOCol2 + 64 * hh;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t raw[32];
        tmem_ld32(tO32 + 32 * c, raw);
        tmem_wait_ld();
        reg_fence<32>(raw);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[e] = pack_bf16x2(__uint_as_float(raw[2 * e]) * inv_l, __uint_as_float(raw[2 * e + 1]) * inv_l);
        if (valid) {
          __nv_bfloat16* dst = orow + 64 * hh + 32 * c;
          if (prm.o_v8) {
            st_global_v8_hint(dst, pk, pol_out);
            st_global_v8_hint(dst + 16, pk + 8, pol_out);
          } else {
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              st_global_v4_hint(d4 + e, make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]), pol_out);
          }
        }
      }
      if (valid && hh == 0 && prm.lse)
        prm.lse[rq.bcoord * prm.lse_sb + h_row * prm.lse_sh + rq.q_row0 + t_row] =
            (m_row + __log2f(l_row)) * 0.69314718055994531f;
      named_bar_sync(1, 256);     // xl / xm are reused by the next item
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace

cudaError_t launch_attn_sm100_2sm(const AttnParams& prm, const CUtensorMap& tm_q_tok, const CUtensorMap& tm_q_pack,
                                  const CUtensorMap& tm_k64, const CUtensorMap& tm_v, int num_sms, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int clusters = num_sms / 2;
  if (prm.n_items < clusters) clusters = prm.n_items;
  if (clusters <= 0) return cudaSuccess;
  attn_2sm_kernel<<<2 * clusters, kThreads2, kSmem2, stream>>>(prm, tm_q_tok, tm_q_pack, tm_k64, tm_v);
  return cudaGetLastError();
}

}  // namespace parse
