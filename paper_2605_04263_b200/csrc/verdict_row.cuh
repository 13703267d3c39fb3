// Verdict logits of one judgment row (reading R17): one pass
// over the bf16 hidden state accumulates sum(h^2), sum(h*g*w_C), sum(h*g*w_I)
// in fp32; l = dot * rsqrt(mean(h^2) + eps) (the RMSNorm scale factors out of
// both dots).  Called by every thread of a 128-thread CTA; thread 0 returns
// (l_C, l_I).  Shared by verdict_head_kernel (readout.cu) and the fused
// verdict + selection kernel (select.cu).
#pragma once
#include "internal.h"

namespace parse {

constexpr int kHeadThreads = 128;   // one CTA per judgment row: a row's loads all in flight at once

__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

__device__ __forceinline__ float2 verdict_row(const VerdictHeadParams& p, int row) {
  __shared__ float red[3][kHeadThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = row / p.K, k = row - b * p.K;
  const uint16_t* h = p.h + int64_t(b) * p.hs_b + int64_t(k) * p.hs_k;
  const uint4* h4 = reinterpret_cast<const uint4*>(h);
  const uint4* g4 = reinterpret_cast<const uint4*>(p.g);
  const uint4* c4 = reinterpret_cast<const uint4*>(p.w);
  const uint4* i4 = reinterpret_cast<const uint4*>(p.w + p.H);
  float ss = 0.f, dc = 0.f, di = 0.f;
  const int n8 = p.H / 8;
#pragma unroll 4
  for (int q = threadIdx.x; q < n8; q += kHeadThreads) {
    const uint4 hv = __ldcs(h4 + q), gv = __ldg(g4 + q), cv = __ldg(c4 + q), iv = __ldg(i4 + q);
    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, gw[4] = {gv.x, gv.y, gv.z, gv.w};
    const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w}, iw[4] = {iv.x, iv.y, iv.z, iv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float h0 = bf_lo(hw[e]), h1 = bf_hi(hw[e]);
      const float hg0 = h0 * bf_lo(gw[e]), hg1 = h1 * bf_hi(gw[e]);
      ss = fmaf(h0, h0, fmaf(h1, h1, ss));
      dc = fmaf(hg0, bf_lo(cw[e]), fmaf(hg1, bf_hi(cw[e]), dc));
      di = fmaf(hg0, bf_lo(iw[e]), fmaf(hg1, bf_hi(iw[e]), di));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    dc += __shfl_xor_sync(0xffffffffu, dc, o);
    di += __shfl_xor_sync(0xffffffffu, di, o);
  }
  if (lane == 0) { red[0][warp] = ss; red[1][warp] = dc; red[2][warp] = di; }
  __syncthreads();
  float2 l = make_float2(0.f, 0.f);
  if (threadIdx.x == 0) {
    ss = dc = di = 0.f;
#pragma unroll
    for (int w = 0; w < kHeadThreads / 32; ++w) { ss += red[0][w]; dc += red[1][w]; di += red[2][w]; }
    const float r = rsqrtf(ss / float(p.H) + p.eps);
    l = make_float2(dc * r, di * r);
  }
  return l;
}

}  // namespace parse
