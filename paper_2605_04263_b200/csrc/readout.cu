// Verdict readout kernels, both HBM-bound streaming passes.
//
// verdict_head_kernel: one warp per judgment row; one pass over the bf16
//   hidden state computes sum(h^2), sum(h*g*w_C), sum(h*g*w_I) in fp32; then
//   l = dot * rsqrt(mean(h^2) + eps) (the RMSNorm scale factors out of both
//   dots).  gamma and the two W_U rows stay in L1/L2 across rows.
// vocab_readout_kernel: one CTA per judgment row streams the V logits with
//   16-byte loads, keeps a per-thread online (max, sum 2^x) pair, reduces it
//   over the CTA, and reads z_C, z_I.
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"
#include "verdict_row.cuh"

namespace parse {
using namespace parse_sm100;
namespace {

__global__ void __launch_bounds__(kHeadThreads) verdict_head_kernel(const VerdictHeadParams p) {
  const int row = blockIdx.x;
  const float2 l = verdict_row(p, row);
  if (threadIdx.x == 0) {
    p.out[2 * row] = l.x;
    p.out[2 * row + 1] = l.y;
  }
}

constexpr int kVocabThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;

// online log-sum-exp state in base 2: value = m + log2(s)
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * ex2(m - mn) + s2 * ex2(m2 - mn);
  m = mn;
}

template <bool kBf16>
__global__ void __launch_bounds__(kVocabThreads) vocab_readout_kernel(const VocabReadoutParams p) {
  __shared__ float sm[kVocabThreads / 32], ssum[kVocabThreads / 32];
  const int row = blockIdx.x;
  const int b = row / p.K, k = row - b * p.K;
  const int64_t off = int64_t(b) * p.s_b + int64_t(k) * p.s_k;
  float m = -INFINITY, s = 0.f;  // base-2 running max of z*log2e and sum of 2^(x - m)
  constexpr int kPer = kBf16 ? 8 : 4;
  const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(p.z) + off * (kBf16 ? 2 : 4));
  const int nvec = p.V / kPer;
#pragma unroll 4
  for (int q = threadIdx.x; q < nvec; q += kVocabThreads) {
    const uint4 v = __ldcs(src + q);  // streamed once
    float x[kPer];
    if constexpr (kBf16) {
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) { x[2 * e] = bf_lo(w[e]) * kLog2e; x[2 * e + 1] = bf_hi(w[e]) * kLog2e; }
    } else {
      x[0] = __uint_as_float(v.x) * kLog2e; x[1] = __uint_as_float(v.y) * kLog2e;
      x[2] = __uint_as_float(v.z) * kLog2e; x[3] = __uint_as_float(v.w) * kLog2e;
    }
    float mx = x[0];
#pragma unroll
    for (int e = 1; e < kPer; ++e) mx = fmaxf(mx, x[e]);
    if (mx > m) {
      s *= ex2(m - mx);
      m = mx;
    }
    // masked entries (-inf) before any finite one: m = -inf would make
    // x - m = -inf - -inf = NaN; they add exactly 0 instead
    const float m_eff = m == -INFINITY ? 0.f : m;
#pragma unroll
    for (int e = 0; e < kPer; ++e) s += ex2(x[e] - m_eff);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, m2, s2);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sm[warp] = m; ssum[warp] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], Ssum = ssum[0];
    for (int w = 1; w < kVocabThreads / 32; ++w) lse_merge(M, Ssum, sm[w], ssum[w]);
    const float lse = (M + __log2f(Ssum)) * 0.69314718055994531f;  // natural log
    float zc, zi;
    if constexpr (kBf16) {
      const uint16_t* zz = reinterpret_cast<const uint16_t*>(p.z) + off;
      zc = __uint_as_float(uint32_t(zz[p.id_c]) << 16);
      zi = __uint_as_float(uint32_t(zz[p.id_i]) << 16);
    } else {
      const float* zz = reinterpret_cast<const float*>(p.z) + off;
      zc = zz[p.id_c];
      zi = zz[p.id_i];
    }
    p.pair[2 * row] = zc;
    p.pair[2 * row + 1] = zi;
    if (p.lse) p.lse[row] = lse;
    if (p.mass) p.mass[row] = __expf(zc - lse) + __expf(zi - lse);
  }
}

}  // namespace

cudaError_t launch_verdict_head(const VerdictHeadParams& p, cudaStream_t stream) {
  const int rows = p.B * p.K;
  verdict_head_kernel<<<rows, kHeadThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_vocab_readout(const VocabReadoutParams& p, cudaStream_t stream) {
  const int rows = p.B * p.K;
  if (p.bf16) vocab_readout_kernel<true><<<rows, kVocabThreads, 0, stream>>>(p);
  else vocab_readout_kernel<false><<<rows, kVocabThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace parse
