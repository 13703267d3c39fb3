// parse_verify_attn, bf16 path: persistent warp-specialised tcgen05 kernel for
// sm_100a.
//
// What it computes (§3.2): masked attention over the packed sequence
// [shared region (N rows) | K appended suffix copies (S rows each)] where
// shared rows are causal, suffix copy k sees shared keys [0, b_k) plus itself
// causally (or its tree ancestors), and copies never see each other.
//
// Structure (one CTA per SM, 384 threads):
//   warp 0      TMA producer: Q tiles, then K_j / V_j tiles into an smem ring
//   warp 1      MMA issuer (one thread): S_i = Q_i K_j^T (SS, fp32 in TMEM);
//               O_i += P_i V_j (TS: P from TMEM, V from smem)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax warpgroup for Q tile 0 (thread = row = TMEM lane)
//   warps 8-11  softmax warpgroup for Q tile 1
// A work item holds up to two Q tiles with the same rows' visibility (two
// q heads, or two head-packs, of one KV group), so every K/V tile brought
// into shared memory is used by both (north_star: "Each draft K/V tile is
// loaded once and shared by every suffix whose boundary covers it").
// The softmax is online with a lazy rescale: O is rescaled in TMEM only when
// a row max grows by more than 2^8 (log2 units) over the max in use.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"

namespace parse {
using namespace parse_sm100;

namespace {

constexpr int kThreads = 384;
constexpr float kRescaleThresh = 8.0f;  // log2 units

template <int D>
struct Cfg {
  static constexpr int kChunks = D / 64;          // 128-byte swizzle atoms along d
  static constexpr int kChunkBytes = 128 * 128;   // 128 rows x 128 B
  static constexpr int kTileBytes = 128 * D * 2;  // one Q / K / V tile (bf16)
  static constexpr int kStages = D == 128 ? 4 : 8;
  static constexpr int kQOff = 0;
  static constexpr int kKVOff = 2 * kTileBytes;
  static constexpr int kBarOff = kKVOff + kStages * kTileBytes;
  // barriers: q_full[2] q_empty[2] s_full[2] p_full[2] o_full[2] kv_full[S] kv_empty[S]
  static constexpr int kNumBars = 10 + 2 * kStages;
  static constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;  // + tmem slot + align slack
  static constexpr int kTmemCols = 512;
  static constexpr int kSCol = 0;    // S_i at i*128
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
};

__device__ __forceinline__ int item_hpt(const WorkItem& w) { return w.flags & 0xff; }
__device__ __forceinline__ int item_nq(const WorkItem& w) { return (w.flags >> 8) & 1 ? 2 : 1; }
__device__ __forceinline__ int kv_key0(const WorkItem& w, int j) {
  return j < w.n_draft ? j * kTile : w.self_lo + (j - w.n_draft) * kTile;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    attn_sm100_kernel(const __grid_constant__ AttnParams prm,
                      const __grid_constant__ CUtensorMap tm_q_tok,
                      const __grid_constant__ CUtensorMap tm_q_pack,
                      const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  Bars bars{sbase + C::kBarOff};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kBarOff + C::kNumBars * 8);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bars.q_full(i), 1);
      mbar_init(bars.q_empty(i), 1);
      mbar_init(bars.s_full(i), 1);
      mbar_init(bars.p_full(i), 128);
      mbar_init(bars.o_full(i), 1);
    }
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(bars.kv_full(s), 1);
      mbar_init(bars.kv_empty(s, C::kStages), 1);
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
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int r_heads = prm.Hq / prm.Hkv;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t kv_phase = 0;
      uint32_t q_phase[2] = {0, 0};
      for (int it = blockIdx.x; it < prm.n_items; it += gridDim.x) {
        const WorkItem w = prm.items[it];
        const int hpt = item_hpt(w), nq = item_nq(w);
        const int g = w.h0 / r_heads;
        const CUtensorMap* qm = hpt == 1 ? &tm_q_tok : &tm_q_pack;
        for (int i = 0; i < nq; ++i) {
          mbar_wait(bars.q_empty(i), q_phase[i] ^ 1);
          q_phase[i] ^= 1;
          mbar_arrive_expect_tx(bars.q_full(i), C::kTileBytes);
          const uint32_t dst = sbase + C::kQOff + i * C::kTileBytes;
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_4d(qm, bars.q_full(i), dst + c * C::kChunkBytes, c * 64, w.h0 + i * hpt, w.t0, w.b);
        }
        const int n = w.n_draft + w.n_self;
        for (int j = 0; j < n; ++j) {
          const int key0 = kv_key0(w, j);
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {
            mbar_wait(bars.kv_empty(stage, C::kStages), kv_phase ^ 1);
            mbar_arrive_expect_tx(bars.kv_full(stage), C::kTileBytes);
            const uint32_t dst = sbase + C::kKVOff + stage * C::kTileBytes;
            for (int c = 0; c < C::kChunks; ++c)
              tma_load_4d(kv == 0 ? &tm_k : &tm_v, bars.kv_full(stage), dst + c * C::kChunkBytes, c * 64, g,
                          key0, w.b);
            if (++stage == C::kStages) { stage = 0; kv_phase ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================= MMA issuer =============================
    if (lane == 0) {
      constexpr uint32_t idesc_qk = make_idesc_bf16(128, 128, 0);
      constexpr uint32_t idesc_pv = make_idesc_bf16(128, D, 1);
      int stage = 0;
      uint32_t kv_phase = 0;
      uint32_t q_phase[2] = {0, 0}, p_phase[2] = {0, 0};
      auto issue_qk = [&](int i, int kst) {
        const uint32_t qa = sbase + C::kQOff + i * C::kTileBytes;
        const uint32_t ka = sbase + C::kKVOff + kst * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::kChunkBytes + (kk & 3) * 32;
          mma_ss(tmem + C::kSCol + i * 128, make_sdesc_sw128(qa + off, 16, 1024),
                 make_sdesc_sw128(ka + off, 16, 1024), idesc_qk, kk > 0);
        }
      };
      auto issue_pv = [&](int i, int vst, bool acc) {
        const uint32_t va = sbase + C::kKVOff + vst * C::kTileBytes;
#pragma unroll
        for (int kk = 0; kk < kTile / 16; ++kk) {
          mma_ts(tmem + C::kOCol + i * D, tmem + C::kSCol + i * 128 + kk * 8,
                 make_sdesc_sw128(va + kk * 2048, C::kChunkBytes, 1024), idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };
      auto next_stage = [&](int& st) {
        st = stage;
        mbar_wait(bars.kv_full(stage), kv_phase);
        if (++stage == C::kStages) { stage = 0; kv_phase ^= 1; }
      };
      for (int it = blockIdx.x; it < prm.n_items; it += gridDim.x) {
        const WorkItem w = prm.items[it];
        const int nq = item_nq(w);
        const int n = w.n_draft + w.n_self;
        for (int i = 0; i < nq; ++i) {
          mbar_wait(bars.q_full(i), q_phase[i]);
          q_phase[i] ^= 1;
        }
        int kst, vst;
        next_stage(kst);
        tc_fence_after();
        for (int i = 0; i < nq; ++i) {
          issue_qk(i, kst);
          mma_commit(bars.s_full(i));
        }
        mma_commit(bars.kv_empty(kst, C::kStages));
        if (n == 1)
          for (int i = 0; i < nq; ++i) mma_commit(bars.q_empty(i));
        for (int j = 0; j < n; ++j) {
          const bool more = j + 1 < n;
          next_stage(vst);
          if (more) next_stage(kst);
          tc_fence_after();
          for (int i = 0; i < nq; ++i) {
            mbar_wait(bars.p_full(i), p_phase[i]);
            p_phase[i] ^= 1;
            tc_fence_after();
            issue_pv(i, vst, j > 0);
            mma_commit(bars.o_full(i));
            if (more) {
              issue_qk(i, kst);
              mma_commit(bars.s_full(i));
            }
          }
          mma_commit(bars.kv_empty(vst, C::kStages));
          if (more) {
            mma_commit(bars.kv_empty(kst, C::kStages));
            if (j + 2 == n)
              for (int i = 0; i < nq; ++i) mma_commit(bars.q_empty(i));
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ========================== softmax warpgroups ==========================
    const int wg = (warp - 4) >> 2;             // Q tile index
    const int row = threadIdx.x & 127;          // = TMEM lane
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_base + C::kSCol + wg * 128;
    const uint32_t tO = tmem + lane_base + C::kOCol + wg * D;
    uint32_t s_phase = 0;
    uint32_t pv_count = 0;                      // # PV MMAs committed to o_full[wg] so far
    const float sl2 = prm.scale_log2;
    for (int it = blockIdx.x; it < prm.n_items; it += gridDim.x) {
      const WorkItem w = prm.items[it];
      const int nq = item_nq(w);
      if (wg >= nq) continue;
      const int hpt = item_hpt(w);
      const int n = w.n_draft + w.n_self;
      const int t = w.t0 + row / hpt;
      const int h = w.h0 + wg * hpt + row % hpt;
      const bool row_valid = t < w.t_end;
      // visibility of this row: keys [0, lim) of the shared region,
      // plus own-copy keys [sbase, t] (or tree ancestors of sidx)
      int lim, sbase_k = 0x7fffffff, sidx = 0;
      if (t < prm.N) {
        lim = t + 1;
      } else if (t < prm.L) {
        const int k = (t - prm.N) / prm.S;
        sidx = t - prm.N - k * prm.S;
        lim = prm.bnd[w.b * prm.K + k];
        sbase_k = prm.N + k * prm.S;
      } else {
        lim = 0;
      }
      const uint64_t anc_row = prm.anc ? prm.anc[sidx] : 0ull;
      float m_used = -INFINITY, l_sum = 0.f;
      for (int j = 0; j < n; ++j) {
        mbar_wait(bars.s_full(wg), s_phase);
        s_phase ^= 1;
        tc_fence_after();
        float s[kTile];
        {
          uint32_t raw[32];
#pragma unroll
          for (int c = 0; c < kTile / 32; ++c) {
            tmem_ld32(tS + c * 32, raw);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) s[c * 32 + e] = __uint_as_float(raw[e]);
          }
        }
        const int key0 = kv_key0(w, j);
        if (j < w.n_draft) {
          const int nvis = lim - key0;           // keys [key0, lim) visible
          if (nvis < kTile) {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c >= nvis) s[c] = -INFINITY;
          }
        } else {
          const int lo = sbase_k - key0;         // own copy starts at column lo
          const int hi = t - key0;               // causal: columns <= hi
          if (prm.anc) {
#pragma unroll
            for (int c = 0; c < kTile; ++c) {
              const int rel = c - lo;
              const bool vis = rel >= 0 && rel < 64 && ((anc_row >> (rel & 63)) & 1ull);
              if (!vis) s[c] = -INFINITY;
            }
          } else {
#pragma unroll
            for (int c = 0; c < kTile; ++c)
              if (c < lo || c > hi) s[c] = -INFINITY;
          }
        }
        float mt = s[0];
#pragma unroll
        for (int c = 1; c < kTile; ++c) mt = fmaxf(mt, s[c]);
        const float m_tile = mt * sl2;
        float alpha = 1.f;
        bool rescale_o = false;
        if (m_tile > m_used + kRescaleThresh) {
          alpha = ex2(m_used - m_tile);
          rescale_o = (m_used != -INFINITY);
          m_used = m_tile;
        }
        const float m_eff = (m_used == -INFINITY) ? 0.f : m_used;
        float rs = 0.f;
#pragma unroll
        for (int half = 0; half < kTile / 64; ++half) {
          // P (bf16, packed in pairs: even key in the low half) overwrites
          // columns [32*half, 32*half+32) of S_i; the PV MMA reads it as A.
          uint32_t packed[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const int c = half * 64 + 2 * e;
            const float p0 = ex2(fmaf(s[c], sl2, -m_eff));
            const float p1 = ex2(fmaf(s[c + 1], sl2, -m_eff));
            rs += p0 + p1;
            __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            packed[e] = *reinterpret_cast<uint32_t*>(&b2);
          }
          tmem_st32(tS + half * 32, packed);
        }
        l_sum = l_sum * alpha + rs;
        if (__any_sync(0xffffffffu, rescale_o)) {
          // O_i must hold PV(j-1) before it is rescaled in place.
          mbar_wait(bars.o_full(wg), (pv_count + j - 1) & 1);
          tc_fence_after();
          uint32_t raw[32];
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            tmem_ld32(tO + c * 32, raw);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) raw[e] = __float_as_uint(__uint_as_float(raw[e]) * alpha);
            tmem_st32(tO + c * 32, raw);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(bars.p_full(wg));
      }
      // ------------------------------ epilogue ------------------------------
      mbar_wait(bars.o_full(wg), (pv_count + n - 1) & 1);
      pv_count += n;
      tc_fence_after();
      const float inv_l = l_sum > 0.f ? 1.f / l_sum : 0.f;
      __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(prm.o) + w.b * prm.o_s0 +
                            int64_t(t) * prm.o_s1 + int64_t(h) * prm.o_s2;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t raw[32];
        tmem_ld32(tO + c * 32, raw);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(raw[2 * e]) * inv_l,
                                                    __uint_as_float(raw[2 * e + 1]) * inv_l);
          pk[e] = *reinterpret_cast<uint32_t*>(&b2);
        }
        if (row_valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
        }
      }
      if (row_valid && prm.lse)
        prm.lse[(int64_t(w.b) * prm.Hq + h) * prm.L + t] = (m_used + __log2f(l_sum)) * 0.69314718055994531f;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

template <int D>
cudaError_t launch_impl(const AttnParams& prm, const CUtensorMap& a, const CUtensorMap& b,
                        const CUtensorMap& c, const CUtensorMap& d, int num_sms, cudaStream_t stream) {
  using Cf = Cfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int grid = prm.n_items < num_sms ? prm.n_items : num_sms;
  if (grid <= 0) return cudaSuccess;
  attn_sm100_kernel<D><<<grid, kThreads, Cf::kSmem, stream>>>(prm, a, b, c, d);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_sm100(const AttnParams& prm, int D, const CUtensorMap& tm_q_tok,
                              const CUtensorMap& tm_q_pack, const CUtensorMap& tm_k,
                              const CUtensorMap& tm_v, int num_sms, cudaStream_t stream) {
  if (D == 128) return launch_impl<128>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream);
  return launch_impl<64>(prm, tm_q_tok, tm_q_pack, tm_k, tm_v, num_sms, stream);
}

}  // namespace parse
