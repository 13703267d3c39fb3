// parse_verify_attn, bf16, head_dim 128: the 2-SM (cta_group::2) variant of
// attn_sm100_kernel with a decoupled S -> P -> PV pipeline.
//
// A cluster of two CTAs runs a pair of work items with the same request, KV
// group and K/V sequence (build_pairs): CTA r owns the two Q tiles of item r.
// Every tcgen05.mma is issued by the leader CTA with cta_group::2 (M = 256 =
// tile t of both CTAs); each CTA holds only half of every K tile (64 keys) and
// half of every V tile (64 of the 128 head-dim columns), so a 32 KB stage
// carries a whole K/V step.  The freed shared memory holds P (bf16, SW128),
// so PV reads P from shared memory and QK^T(j+1) overwrites S_t as soon as
// both CTAs' softmax have loaded S_t(j): each softmax runs step after step,
// never waiting for PV + QK^T.  TMEM per CTA: S0 | S1 | O0 | O1 (round 1's layout;
// the one-CTA kernel now shares one S buffer between its two tiles).
//
//   warp 0      producer (both CTAs): Q tile, then K/V halves, TMA completing
//               on the leader's barriers; the leader's also fetches items and
//               writes them to both CTAs' item rings
//   warps 1, 3  MMA issuers for tiles 0 / 1 (leader CTA only)
//   warp 2      TMEM allocator (cta_group::2)
//   warps 4-11  softmax: one warpgroup per tile, thread = row (as the one-CTA
//               kernel), P written to shared memory
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace parse {
using namespace parse_sm100;

namespace {

constexpr int kThreads2 = 384;
constexpr int kStages2 = 3;                  // K/V steps in flight (half tiles: 32 KB per step)
constexpr int kQBytes = 128 * 128 * 2;      // one Q tile (also one P tile)
constexpr int kKHalf = 64 * 128 * 2;        // 64 keys x 128 d
constexpr int kVHalf = 128 * 64 * 2;        // 128 keys x 64 d
constexpr int kStageBytes = kKHalf + kVHalf;
constexpr int kQOff2 = 0;                    // Q tiles 0, 1
constexpr int kPOff2 = 2 * kQBytes;          // P tiles 0, 1 (bf16, K-major SW128)
constexpr int kKVOff2 = 4 * kQBytes;
constexpr int kBarOff2 = kKVOff2 + kStages2 * kStageBytes;
constexpr int kRing2 = 4;
// barriers: q_full q_empty s_full[2] s_used[2] p_full[2] p_empty[2] o_full[2] o_done[2] kv_full[S] kv_empty[S]
//           item_full[R] item_empty[R]
constexpr int kNumBars2 = 14 + 2 * kStages2 + 2 * kRing2;
constexpr int kItemOff2 = (kBarOff2 + kNumBars2 * 8 + 15) / 16 * 16;
constexpr int kSmem2 = kItemOff2 + 96 * kRing2 + 16 + 1024;
constexpr int kSCol2 = 0, kOCol2 = 256;
constexpr float kThresh2 = 8.0f;
constexpr uint16_t kBoth = 3;                // multicast mask: both CTAs
static_assert(kSmem2 <= 232448, "shared memory budget");
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
  __device__ uint32_t s_used(int i) const { return base + 8 * (4 + i); }
  __device__ uint32_t p_full(int i) const { return base + 8 * (6 + i); }
  __device__ uint32_t p_empty(int i) const { return base + 8 * (8 + i); }
  __device__ uint32_t o_full(int i) const { return base + 8 * (10 + i); }
  __device__ uint32_t o_done(int i) const { return base + 8 * (12 + i); }
  __device__ uint32_t kv_full(int s) const { return base + 8 * (14 + s); }
  __device__ uint32_t kv_empty(int s) const { return base + 8 * (14 + kStages2 + s); }
  __device__ uint32_t item_full(int r) const { return base + 8 * (14 + 2 * kStages2 + r); }
  __device__ uint32_t item_empty(int r) const { return base + 8 * (14 + 2 * kStages2 + kRing2 + r); }
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
#ifndef PARSE_CL_HINT
constexpr uint32_t kClHint = 0x100000u;
#else
constexpr uint32_t kClHint = PARSE_CL_HINT;
#endif
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
        : "r"(bar), "r"(parity), "r"(kClHint)
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

// Ring entry: the two items of a work unit (w1 = w0 when it runs alone) and
// their request.
struct alignas(16) RingEntry2 {
  WorkItem w0, w1;
  ReqDesc r;
};
static_assert(sizeof(RingEntry2) == 96, "ring entry is 96 bytes");

template <int kRing>
__device__ __forceinline__ bool next_item2(const Bars2& bars, const RingEntry2* ring, int& slot, uint32_t& phase,
                                           RingEntry2& e, uint32_t leader_item_empty_base, bool leader) {
  mbar_wait_cl(bars.item_full(slot), phase);
  e = ring[slot];
  __syncwarp();
  // release the slot on the leader's ring (only the leader's producer refills): one arrive per warp
  if ((threadIdx.x & 31) == 0) {
    if (leader) mbar_arrive(bars.item_empty(slot));
    else mbar_arrive_cluster(leader_item_empty_base + 8 * slot);
  }
  if (++slot == kRing) { slot = 0; phase ^= 1; }
  return e.w0.n_draft >= 0;
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
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kItemOff2 + sizeof(RingEntry2) * kRing2);
  const uint32_t leader_item_empty = map_rank(bars.item_empty(0), 0);
  int ring_slot = 0;
  uint32_t ring_phase = 0;

  if (threadIdx.x == 0) {
    mbar_init(bars.q_full(), 1);
    mbar_init(bars.q_empty(), 2);            // both MMA warps
    for (int i = 0; i < 2; ++i) {
      mbar_init(bars.s_full(i), 1);
      mbar_init(bars.s_used(i), 8);          // one arrive per softmax warp of tile i, both CTAs
      mbar_init(bars.p_full(i), 8);
      mbar_init(bars.p_empty(i), 1);
      mbar_init(bars.o_full(i), 1);
      mbar_init(bars.o_done(i), 1);
    }
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(bars.kv_full(s), 1);
      mbar_init(bars.kv_empty(s), 2);        // both MMA warps
    }
    for (int r = 0; r < kRing2; ++r) {
      mbar_init(bars.item_full(r), 1);
      // one arrive per consuming warp: both MMA warps, the peer's producer, 8 + 8 softmax warps
      mbar_init(bars.item_empty(r), 2 + 1 + 8 + 8);
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
        RingEntry2 e;
        if (leader) {
          int it = 0;
          if (lane == 0) it = atomicAdd(prm.counter, 1);
          it = __shfl_sync(0xffffffffu, it, 0);
          if (it < prm.n_work) {
            const int2 pr = prm.work[it];
            e.w0 = prm.items[pr.x];
            e.w1 = pr.y >= 0 ? prm.items[pr.y] : e.w0;
            if (pr.y < 0) e.w1.flags |= 1 << 16;     // alone: the peer recomputes w0, unstored
            e.r = load_req2(prm, e.w0.b);
          } else {
            e.w0 = WorkItem{};
            e.w0.n_draft = -1;
            e.w1 = e.w0;
            e.r = ReqDesc{};
          }
          mbar_wait_cl(bars.item_empty(ring_slot), ring_phase ^ 1);
          if (lane == 0) {
            ring[ring_slot] = e;
            const uint32_t peer = map_rank(smem_u32(&ring[ring_slot]), 1);
            const uint4* src = reinterpret_cast<const uint4*>(&e);
#pragma unroll
            for (int q = 0; q < 6; ++q) st_cluster_v4(peer + 16 * q, src[q]);
            mbar_arrive(bars.item_full(ring_slot));
            mbar_arrive_cluster(map_rank(bars.item_full(ring_slot), 1));
          }
          __syncwarp();
          if (++ring_slot == kRing2) { ring_slot = 0; ring_phase ^= 1; }
          if (e.w0.n_draft < 0) break;
        } else {
          if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, e, leader_item_empty, false)) break;
        }
        const WorkItem& w = rank == 0 ? e.w0 : e.w1;
        const ReqDesc& rq = e.r;
        const int nq = item_nq2(w);
        const int hpt = item_hpt2(w);
        const int g = w.h0 / r_heads;
        const CUtensorMap* qm = hpt == 1 ? &tm_q_tok : &tm_q_pack;
        mbar_wait(bars.q_empty(), q_phase ^ 1);
        q_phase ^= 1;
        if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(bars.q_full(), 2 * nq * kQBytes);
          for (int i = 0; i < nq; ++i)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_4d_2sm(qm, bars.q_full(), sbase + kQOff2 + i * kQBytes + c * 16384, c * 64, tile_h0_2(w, i),
                              rq.q_row0 + tile_t0_2(w, i, prm.S), rq.bcoord, pol_stream);
        }
        __syncwarp();
        const int n = w.n_draft + w.n_self;
        for (int j = 0; j < n; ++j) {
          const int key0 = kv_key0_2(w, j);
          mbar_wait(bars.kv_empty(stage), kv_phase ^ 1);
          if (elect_one()) {
            if (leader) mbar_arrive_expect_tx(bars.kv_full(stage), 2 * kStageBytes);
            const uint32_t dst = sbase + kKVOff2 + stage * kStageBytes;
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_4d_2sm(&tm_k64, bars.kv_full(stage), dst + c * 8192, c * 64, g, rq.kv_row0 + key0 + 64 * int(rank),
                              rq.bcoord, pol_keep);
            tma_load_4d_2sm(&tm_v, bars.kv_full(stage), dst + kKHalf, 64 * int(rank), g, rq.kv_row0 + key0, rq.bcoord,
                            pol_keep);
          }
          __syncwarp();
          if (++stage == kStages2) { stage = 0; kv_phase ^= 1; }
        }
      }
    } else if ((warp == 1 || warp == 3) && leader) {
      // ===================== MMA issuers (leader CTA): tile t =====================
      const int t = warp == 1 ? 0 : 1;
      constexpr uint32_t idesc_qk = make_idesc_bf16(256, 128, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(256, 128, 1);
      const uint64_t qdesc = make_sdesc_sw128(sbase + kQOff2 + t * kQBytes, 16, 1024);
      const uint64_t pdesc = make_sdesc_sw128(sbase + kPOff2 + t * kQBytes, 16, 1024);
      const uint64_t kdesc0 = make_sdesc_sw128(sbase + kKVOff2, 16, 1024);
      const uint64_t vdesc0 = make_sdesc_sw128(sbase + kKVOff2 + kKHalf, 8192, 1024);
      const uint32_t s_tm = tmem + kSCol2 + t * 128;
      const uint32_t o_tm = tmem + kOCol2 + t * 128;
      int stage = 0, mstep = 0;
      uint32_t kv_phase = 0, q_phase = 0, u_phase = 0, p_phase = 0;
      auto issue_qk = [&](int st) {
        const uint64_t kd = kdesc0 + uint64_t((st * kStageBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t qoff = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const uint64_t koff = uint64_t(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
          mma2_ss(s_tm, qdesc + qoff, kd + koff, idesc_qk, kk > 0);
        }
      };
      auto issue_pv = [&](int st, bool acc) {
        const uint64_t vd = vdesc0 + uint64_t((st * kStageBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t poff = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          mma2_ss(o_tm, pdesc + poff, vd + uint64_t((kk * 2048) >> 4), idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };
      for (;;) {
        RingEntry2 e;
        if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, e, leader_item_empty, true)) break;
        const WorkItem& w = e.w0;
        const int n = w.n_draft + w.n_self;
        const int nq = item_nq2(w);
        const int stage0 = stage;
        auto st_of = [&](int j) { return (stage0 + j) % kStages2; };
        auto ph_of = [&](int j) { return kv_phase ^ uint32_t(((stage0 + j) / kStages2) & 1); };
        if (t >= nq) {
          // tile 1 absent: release this warp's share of the Q buffer and every stage once landed
          for (int j = 0; j < n; ++j) {
            mbar_wait(bars.kv_full(st_of(j)), ph_of(j));
            if (lane == 0) {
              mbar_arrive(bars.kv_empty(st_of(j)));
              mbar_arrive_cluster(map_rank(bars.kv_empty(st_of(j)), 1));
            }
            __syncwarp();
          }
          mbar_wait(bars.q_full(), q_phase);
          q_phase ^= 1;
          if (lane == 0) {
            mbar_arrive(bars.q_empty());
            mbar_arrive_cluster(map_rank(bars.q_empty(), 1));
          }
          __syncwarp();
        } else {
          mbar_wait(bars.q_full(), q_phase);
          q_phase ^= 1;
          mbar_wait(bars.kv_full(st_of(0)), ph_of(0));
          tc_fence_after();
          if (elect_one()) {
            issue_qk(st_of(0));
            commit2(bars.s_full(t));
            if (n == 1) commit2(bars.q_empty());
          }
          __syncwarp();
          for (int j = 0; j < n; ++j) {
            if (j + 1 < n) {
              // QK(j+1) into S_t as soon as both CTAs' softmax have read S_t(j)
              mbar_wait_cl(bars.s_used(t), u_phase);
              TR2(lane == 0 && blockIdx.x == 0 && t == 0, 0, mstep, 0);
              u_phase ^= 1;
              mbar_wait(bars.kv_full(st_of(j + 1)), ph_of(j + 1));
              TR2(lane == 0 && blockIdx.x == 0 && t == 0, 0, mstep, 1);
              tc_fence_after();
              if (elect_one()) {
                issue_qk(st_of(j + 1));
                commit2(bars.s_full(t));
                if (j + 1 == n - 1) commit2(bars.q_empty());
              }
              __syncwarp();
            } else {
              mbar_wait_cl(bars.s_used(t), u_phase);
              u_phase ^= 1;
            }
            TR2(lane == 0 && blockIdx.x == 0 && t == 0, 0, mstep, 2);
            mbar_wait_cl(bars.p_full(t), p_phase);
            TR2(lane == 0 && blockIdx.x == 0 && t == 0, 0, mstep, 3);
            p_phase ^= 1;
            tc_fence_after();
            if (elect_one()) {
              issue_pv(st_of(j), j > 0);
              commit2(bars.o_full(t));
              commit2(bars.p_empty(t));
              commit2(bars.kv_empty(st_of(j)));
              if (j == n - 1) commit2(bars.o_done(t));
            }
            __syncwarp();
            TR2(lane == 0 && blockIdx.x == 0 && t == 0, 0, mstep, 4);
            if (t == 0) ++mstep;
          }
        }
        const int adv = stage0 + n;
        kv_phase ^= uint32_t((adv / kStages2) & 1);
        stage = adv % kStages2;
      }
    }
  } else {
    setmaxnreg_inc<216>();
    // ============================ softmax (tile wg) ============================
    const int wg = (warp - 4) >> 2;
    const int row = threadIdx.x & 127;
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + kSCol2 + wg * 128;
    const uint32_t tO = tmem + lane_base + kOCol2 + wg * 128;
    const uint32_t s_used_l = map_rank(bars.s_used(wg), 0);
    const uint32_t p_full_l = map_rank(bars.p_full(wg), 0);
    // P tile of this row in shared memory: K-major SW128 (2 x 64-key atoms of 128 rows x 128 B)
    const uint32_t p_row = sbase + kPOff2 + wg * kQBytes + row * 128;
    uint32_t s_phase = 0;
    uint32_t steps = 0, items_done = 0;   // p_empty / o_full phases: one per step; o_done: one per item
    const float sl2 = prm.scale_log2;
    const uint64_t pol_out = make_policy_evict_first();
    auto arrive_leader = [&](uint32_t cl_addr, uint32_t local_addr) {
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(local_addr);
        else mbar_arrive_cluster_relaxed(cl_addr);
      }
    };
    for (;;) {
      RingEntry2 e;
      if (!next_item2<kRing2>(bars, ring, ring_slot, ring_phase, e, leader_item_empty, leader)) break;
      const WorkItem& w = rank == 0 ? e.w0 : e.w1;
      const ReqDesc& rq = e.r;
      const bool store_ok = leader || !((e.w1.flags >> 16) & 1);
      const int nq = item_nq2(w);
      if (wg >= nq) continue;
      const int hpt = item_hpt2(w);
      const int n = w.n_draft + w.n_self;
      const int t = tile_t0_2(w, wg, prm.S) + row / hpt;
      const int h = tile_h0_2(w, wg) + row % hpt;
      const bool row_valid = store_ok && t < w.t_end;
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
      float m_used = -INFINITY, l_sum = 0.f;
      for (int j = 0; j < n; ++j, ++steps) {
        TR2(row == 0 && wg == 0, 1 + rank, steps, 0);
        mbar_wait(bars.s_full(wg), s_phase);
        TR2(row == 0 && wg == 0, 1 + rank, steps, 1);
        s_phase ^= 1;
        tc_fence_after();
        uint32_t sr[kTile];
        tmem_ld64(tS, sr);
        tmem_ld64(tS + 64, sr + 64);
        tmem_wait_ld();
        reg_fence<kTile>(sr);
        tc_fence_before();
        arrive_leader(s_used_l, bars.s_used(wg));     // S_t may be overwritten by QK(j+1)
        TR2(row == 0 && wg == 0, 1 + rank, steps, 2);
        const int key0 = kv_key0_2(w, j);
        bool masked = true;
        if (j < w.n_draft) {
          const int nvis = lim - key0;
          masked = nvis < kTile;
          if (masked) {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c >= nvis) sr[c] = 0xff800000u;
          }
        } else {
          const int lo = sbase_k - key0;
          const int hi = t - key0;
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
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float m = fmax3(__uint_as_float(sr[16 * i]), __uint_as_float(sr[16 * i + 1]), __uint_as_float(sr[16 * i + 2]));
#pragma unroll
          for (int e2 = 3; e2 < 15; e2 += 2) m = fmax3(m, __uint_as_float(sr[16 * i + e2]), __uint_as_float(sr[16 * i + e2 + 1]));
          mx[i] = fmaxf(m, __uint_as_float(sr[16 * i + 15]));
        }
        const float mt = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float m_tile = mt * sl2;
        float alpha = 1.f;
        bool rescale_o = false;
        if (m_tile > m_used + kThresh2) {
          alpha = ex2(m_used - m_tile);
          rescale_o = (m_used != -INFINITY);
          m_used = m_tile;
        }
        const bool any_rescale = __any_sync(0xffffffffu, rescale_o);
        const float m_eff = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2x2 = make_float2(sl2, sl2);
        const float2 negm = make_float2(-m_eff, -m_eff);
        const bool all_full = __all_sync(0xffffffffu, !masked);
#pragma unroll
        for (int e2 = 0; e2 < kTile / 2; ++e2) {
          const float2 x = ffma2(make_float2(__uint_as_float(sr[2 * e2]), __uint_as_float(sr[2 * e2 + 1])), sl2x2, negm);
          sr[2 * e2] = __float_as_uint(x.x);
          sr[2 * e2 + 1] = __float_as_uint(x.y);
        }
        if (all_full) exp_pairs2<true, 0, kTile / 2>(sr);
        else exp_pairs2<false, 0, kTile / 2>(sr);
        // P(j) may overwrite P(j-1) once PV(j-1) has read it
        TR2(row == 0 && wg == 0, 1 + rank, steps, 3);
        if (steps > 0) mbar_wait(bars.p_empty(wg), (steps - 1) & 1);
        TR2(row == 0 && wg == 0, 1 + rank, steps, 4);
        float2 acc[4];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          uint32_t pk[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e2 = 4 * v + q;
            const float2 pp = make_float2(__uint_as_float(sr[2 * e2]), __uint_as_float(sr[2 * e2 + 1]));
            if (e2 < 4) acc[e2] = pp;
            else acc[e2 & 3] = fadd2(acc[e2 & 3], pp);
            pk[q] = pack_bf16x2(pp.x, pp.y);
          }
          const uint32_t addr = p_row + (v >> 3) * 16384 + ((uint32_t((v & 7) ^ (row & 7))) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[0]), "r"(pk[1]), "r"(pk[2]),
                       "r"(pk[3])
                       : "memory");
        }
        const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
        const float2 a = fadd2(a01, a23);
        l_sum = fmaf(l_sum, alpha, a.x + a.y);
        if (any_rescale) {
          // rare: O must hold PV(j-1) before the rescale, which must land before PV(j)
          mbar_wait(bars.o_full(wg), (steps - 1) & 1);
          tc_fence_after();
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
          tmem_wait_st();
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // P visible to the tensor core
        tc_fence_before();
        arrive_leader(p_full_l, bars.p_full(wg));
        TR2(row == 0 && wg == 0, 1 + rank, steps, 5);
      }
      // ------------------------------ epilogue ------------------------------
      mbar_wait(bars.o_done(wg), items_done & 1);
      ++items_done;
      tc_fence_after();
      const float inv_l = l_sum > 0.f ? prm.o_scale / l_sum : 0.f;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.o) + rq.bcoord * prm.o_s0 +
                            int64_t(rq.q_row0 + t) * prm.o_s1 + int64_t(h) * prm.o_s2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t raw[32];
        tmem_ld32(tO + c * 32, raw);
        tmem_wait_ld();
        reg_fence<32>(raw);
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
      if (row_valid && prm.lse)
        prm.lse[rq.bcoord * prm.lse_sb + h * prm.lse_sh + rq.q_row0 + t] = (m_used + __log2f(l_sum)) * 0.69314718055994531f;
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
  cudaError_t e = opt_in_smem<attn_2sm_kernel>(kSmem2);
  if (e != cudaSuccess) return e;
  int clusters = num_sms / 2;
  if (prm.n_work < clusters) clusters = prm.n_work;
  if (clusters <= 0) return cudaSuccess;
  attn_2sm_kernel<<<2 * clusters, kThreads2, kSmem2, stream>>>(prm, tm_q_tok, tm_q_pack, tm_k64, tm_v);
  return cudaGetLastError();
}

}  // namespace parse
