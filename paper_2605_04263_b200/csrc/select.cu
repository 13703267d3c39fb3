// parse_select_prefix: verdict readout + maximal-valid-prefix scan, one warp
// per request.
//
//   p_k  = exp(l_C)/(exp(l_C)+exp(l_I))                 Eq. (p2way)
//   v_k  = raw Correct and p_k >= tau  (d_k >= theta)
//   k*   = leading run of Correct - 1                   App. A.3
//          or max{k : v_k Correct}                       §3.2
//   L*   = t_m, m = floor(max(0, k*+1-eta))              Eq. (adopted)
//
// The pass bits of 32 consecutive prefixes are one __ballot_sync word; the
// first zero bit (leading run) / last one bit (max rule) comes from
// __ffs / __clz across words — the warp prefix scan of the pass bits.  The
// threshold decision is one fp64 compare in logit space, so it is bit-exact
// with the fp64 oracle.
#include <cuda_bf16.h>

#include "internal.h"
#include "verdict_row.cuh"

namespace parse {
namespace {

__device__ __forceinline__ float load_logit(const void* base, int bf16, int64_t idx) {
  if (bf16) return __uint_as_float(uint32_t(reinterpret_cast<const uint16_t*>(base)[idx]) << 16);
  return reinterpret_cast<const float*>(base)[idx];
}
// fused verdict + selection: logits another CTA wrote in this launch (L2, not L1)
__device__ __forceinline__ float load_logit_cg(const void* base, int64_t idx) {
  return __ldcg(reinterpret_cast<const float*>(base) + idx);
}

__device__ __forceinline__ double two_way(double d) {
  // exp(l_C)/(exp(l_C)+exp(l_I)) with x = l_I - l_C = -d, scaled by exp(-max)
  const double x = -d;
  if (x != x) return x;
  if (x < 0.0) return 1.0 / (1.0 + exp(x));
  const double e = exp(-x);
  return e / (1.0 + e);
}

constexpr int kWarps = 4;

// Fused mode: store one 32-bit result word of this rank into slot `rank` of
// every rank's gather buffer (peer memory over NVLink / IPC mappings).
__device__ __forceinline__ void put_all(const SelectParams& p, int64_t word, uint32_t v) {
  const int64_t off = int64_t(p.set * p.world + p.rank) * p.slot_words + word;
  for (int q = 0; q < p.world; ++q)
    reinterpret_cast<uint32_t*>(p.peers[q] + kPeerHeader)[off] = v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* ptr, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* ptr) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
  return v;
}

// After every block's peer stores: the last block to finish raises this
// rank's flag (= epoch) in every peer's header, then waits until every rank's
// flag in its own header has reached the epoch (flags only grow, so a rank
// that is already one call ahead also satisfies the wait).
__device__ void gather_complete(const SelectParams& p) {
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    uint32_t* counter = reinterpret_cast<uint32_t*>(p.peers[p.rank] + 128) + p.set;
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < p.world) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(p.peers[threadIdx.x]) + p.rank, p.epoch);
  }
  if (threadIdx.x == 0) reinterpret_cast<uint32_t*>(p.peers[p.rank] + 128)[p.set] = 0;   // next use of this set
  if (threadIdx.x < p.world) {
    const uint32_t* flag = reinterpret_cast<const uint32_t*>(p.peers[p.rank]) + threadIdx.x;
    const long long t0 = clock64();
    uint32_t polls = 0;
    while (int32_t(ld_acquire_sys(flag) - p.epoch) < 0) {
      if ((++polls & 1023u) == 0 && clock64() - t0 > (1ll << 34)) __trap();   // a peer never arrived
    }
  }
  __syncthreads();
}

// The selection of request b by one warp (lanes over 32 prefixes at a time).
// kCg: the logits were written by other CTAs of the same launch (fused
// verdict + selection) and are read from L2.
template <bool kCg>
__device__ void select_request(const SelectParams& p, int b, int lane, bool fused) {
  int first_fail = -1, last_pass = -1, n_incorrect = 0, trail = 0, n_below = 0;
  bool nonfinite = false;
  float min_sc = __int_as_float(0x7fc00000);  // NaN: ignored by fminf
  for (int k0 = 0; k0 < p.K; k0 += 32) {
    const int k = k0 + lane;
    const bool in = k < p.K;
    bool pass = false, below = false, bad = false;
    if (in) {
      const int64_t base = int64_t(b) * p.ls_b + int64_t(k) * p.ls_k;
      const float lc = kCg ? load_logit_cg(p.logits, base) : load_logit(p.logits, p.bf16, base);
      const float li = kCg ? load_logit_cg(p.logits, base + p.ls_pair) : load_logit(p.logits, p.bf16, base + p.ls_pair);
      const bool fin = isfinite(lc) && isfinite(li);
      const double d = double(lc) - double(li);
      const bool raw = (d > 0.0) || (d == 0.0 && p.tie);
      pass = fin && raw && d >= p.theta;
      below = p.use_aux && !(fin && d >= p.theta_aux);
      bad = !fin;
      const float sc = float(two_way(d));
      if (fused) put_all(p, 2 * int64_t(p.B) + int64_t(b) * p.K + k, __float_as_uint(sc));
      else p.scores[int64_t(b) * p.K + k] = sc;
      min_sc = fminf(min_sc, sc);
    }
    const unsigned pw = __ballot_sync(0xffffffffu, pass);
    const unsigned vw = __ballot_sync(0xffffffffu, in);
    const unsigned fails = vw & ~pw;
    if (first_fail < 0 && fails) first_fail = k0 + __ffs(fails) - 1;
    if (pw) {
      const int lp = 31 - __clz(pw);
      last_pass = k0 + lp;
      trail = __popc(fails & ~((lp == 31) ? 0xffffffffu : ((2u << lp) - 1u)));
    } else {
      trail += __popc(fails);
    }
    n_incorrect += __popc(fails);
    n_below += __popc(__ballot_sync(0xffffffffu, below));
    nonfinite |= __any_sync(0xffffffffu, bad);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) min_sc = fminf(min_sc, __shfl_xor_sync(0xffffffffu, min_sc, o));
  if (lane == 0) {
    int ks;
    if (p.rule == PARSE_RULE_LEADING_RUN) ks = first_fail < 0 ? p.K - 1 : first_fail - 1;
    else ks = last_pass;
    const double mm = floor(fmax(0.0, double(ks) + 1.0 - p.eta));
    const int m = int(mm);
    const int acc = m >= 1 ? p.bnd[int64_t(b) * p.bnd_s + (m - 1)] : 0;
    if (fused) {
      put_all(p, b, uint32_t(acc));
      put_all(p, p.B + b, uint32_t(ks));
    } else {
      p.kstar[b] = ks;
      p.accepted[b] = acc;
    }
    if (p.stats) {
      parse_prefix_stats_t st;
      st.n_incorrect = n_incorrect;
      st.trailing_incorrect_run = trail;
      st.n_below_aux = n_below;
      st.min_score = min_sc;
      p.stats[b] = st;
    }
    if (p.status && nonfinite) atomicOr(p.status, 1);
  }
}

__global__ void __launch_bounds__(kWarps * 32) select_kernel(const SelectParams p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kWarps + warp;
  const bool fused = p.peers != nullptr;
  if (b < p.B) select_request<false>(p, b, lane, fused);
  if (fused) gather_complete(p);
}

// Hidden states -> verdict logits -> selection in one launch: one CTA per
// judgment row computes (l_C, l_I) (verdict_row, reading R17) and writes
// them to the fp32 logits buffer the selection reads (sp.logits); the CTA
// that completes the last row of request b (per-request arrival counter)
// then runs that request's selection with one warp and resets the counter.
__global__ void __launch_bounds__(kHeadThreads) verdict_select_kernel(const VerdictHeadParams hp,
                                                                      const SelectParams sp, uint32_t* counters) {
  const int row = blockIdx.x;
  const int b = row / hp.K;
  const float2 l = verdict_row(hp, row);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    hp.out[2 * row] = l.x;
    hp.out[2 * row + 1] = l.y;
    __threadfence();                                      // this row's logits before the arrival
    last = atomicAdd(counters + b, 1u) == uint32_t(hp.K - 1);
    if (last) {
      __threadfence();                                    // every row's logits visible to this CTA
      counters[b] = 0;                                    // ready for the next call
    }
  }
  __syncthreads();
  if (last && threadIdx.x < 32) select_request<true>(sp, b, threadIdx.x, false);
}

}  // namespace

cudaError_t launch_select(const SelectParams& p, cudaStream_t stream) {
  const int blocks = (p.B + kWarps - 1) / kWarps;
  select_kernel<<<blocks, kWarps * 32, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_verdict_select(const VerdictHeadParams& hp, const SelectParams& sp, uint32_t* counters,
                                  cudaStream_t stream) {
  verdict_select_kernel<<<hp.B * hp.K, kHeadThreads, 0, stream>>>(hp, sp, counters);
  return cudaGetLastError();
}

}  // namespace parse
