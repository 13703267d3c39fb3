// parse_verify_attn, PARSE_PREC_FP32_DEBUG path: a plain SIMT kernel with the
// same visibility (§3.2) as the tcgen05 path, fp32 scores, fp32 softmax
// weights and fp32 output.  It exists as the on-GPU parity mode (<= 1e-5 vs
// the fp64 oracle) — not as a fallback; it is only used when the
// caller asks for precision = PARSE_PREC_FP32_DEBUG.
#include <cuda_bf16.h>

#include "internal.h"

namespace parse {
namespace {

constexpr int kRows = 64;   // query rows per block (one q head)
constexpr int kKeys = 32;   // keys per smem tile

__device__ __forceinline__ float bf2f(uint16_t x) { return __uint_as_float(uint32_t(x) << 16); }

template <int D>
__global__ void __launch_bounds__(kRows) attn_fp32_kernel(const AttnFp32Params p) {
  extern __shared__ float sm[];
  float* qs = sm;                          // [kRows][D+1]
  float* ks = qs + kRows * (D + 1);        // [kKeys][D]
  float* vs = ks + kKeys * D;              // [kKeys][D]
  __shared__ int s_maxlim, s_selflo, s_selfhi;

  const int b = blockIdx.z, h = blockIdx.y, tid = threadIdx.x;
  const ReqDesc rq = p.req[b];
  const int t = blockIdx.x * kRows + tid;
  if (blockIdx.x * kRows >= rq.L) return;       // ragged batch: past this request's rows
  const int g = h / (p.Hq / p.Hkv);
  int lim = 0, sbase = 0x7fffffff, sidx = 0;
  const bool valid = t < rq.L;
  if (valid) {
    if (t < rq.N) {
      lim = t + 1;
    } else {
      const int k = (t - rq.N) / p.S;
      sidx = t - rq.N - k * p.S;
      lim = p.bnd[rq.bnd_off + k];
      sbase = rq.N + k * p.S;
    }
  }
  const uint64_t anc = p.anc ? p.anc[sidx] : 0ull;
  if (tid == 0) { s_maxlim = 0; s_selflo = 0x7fffffff; s_selfhi = 0; }
  __syncthreads();
  atomicMax(&s_maxlim, lim);
  if (valid && t >= rq.N) { atomicMin(&s_selflo, sbase); atomicMax(&s_selfhi, t + 1); }
  for (int i = tid; i < kRows * D; i += kRows) {
    const int rr = i / D, c = i % D, tt = blockIdx.x * kRows + rr;
    qs[rr * (D + 1) + c] =
        tt < rq.L ? bf2f(p.q[rq.bcoord * p.q_s0 + int64_t(rq.q_row0 + tt) * p.q_s1 + int64_t(h) * p.q_s2 + c]) : 0.f;
  }
  __syncthreads();
  const int maxlim = s_maxlim, selflo = s_selflo, selfhi = s_selfhi;

  float acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.f;
  float m = -INFINITY, l = 0.f;
  const float* qrow = qs + tid * (D + 1);

  // segment 0: shared keys [0, maxlim); segment 1: own-copy keys [selflo, selfhi)
  for (int seg = 0; seg < 2; ++seg) {
    const int lo = seg == 0 ? 0 : selflo;
    const int hi = seg == 0 ? maxlim : selfhi;
    for (int k0 = lo; k0 < hi; k0 += kKeys) {
      __syncthreads();
      for (int i = tid; i < kKeys * D; i += kRows) {
        const int kk = i / D, c = i % D, j = k0 + kk;
        float kv = 0.f, vv = 0.f;
        if (j < hi) {
          // contiguous: (batch, row); paged: (page, row in page) from the block table
          int64_t outer = rq.bcoord, row = rq.kv_row0 + j;
          if (p.page_log2) {
            outer = p.block_table[int64_t(b) * p.bt_stride + (j >> p.page_log2)];
            row = j & ((1 << p.page_log2) - 1);
          }
          if (outer >= 0 && (!p.page_log2 || outer < p.num_pages)) {
            kv = bf2f(p.k[outer * p.k_s0 + row * p.k_s1 + int64_t(g) * p.k_s2 + c]);
            vv = bf2f(p.v[outer * p.v_s0 + row * p.v_s1 + int64_t(g) * p.v_s2 + c]);
          }
        }
        ks[kk * D + c] = kv;
        vs[kk * D + c] = vv;
      }
      __syncthreads();
      if (!valid) continue;
      for (int kk = 0; kk < kKeys; ++kk) {
        const int j = k0 + kk;
        if (j >= hi) break;
        bool vis;
        if (seg == 0) {
          vis = j < lim;
        } else {
          const int rel = j - sbase;
          vis = p.anc ? (rel >= 0 && rel < 64 && ((anc >> rel) & 1ull)) : (j >= sbase && j <= t);
        }
        if (!vis) continue;
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) dot = fmaf(qrow[c], ks[kk * D + c], dot);
        const float s = dot * p.scale;
        if (s > m) {
          const float corr = expf(m - s);
          l *= corr;
#pragma unroll
          for (int c = 0; c < D; ++c) acc[c] *= corr;
          m = s;
        }
        const float w = expf(s - m);
        l += w;
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = fmaf(w, vs[kk * D + c], acc[c]);
      }
    }
  }
  if (!valid) return;
  float* orow = p.o + rq.bcoord * p.o_s0 + int64_t(rq.q_row0 + t) * p.o_s1 + int64_t(h) * p.o_s2;
  const float inv = 1.f / l;
#pragma unroll
  for (int c = 0; c < D; ++c) orow[c] = acc[c] * inv;
  if (p.lse) p.lse[rq.bcoord * p.lse_sb + h * p.lse_sh + rq.q_row0 + t] = m + logf(l);
}

template <int D>
cudaError_t launch_impl(const AttnFp32Params& p, cudaStream_t stream) {
  const size_t smem = sizeof(float) * (kRows * (D + 1) + 2 * kKeys * D);
  cudaError_t e = opt_in_smem<attn_fp32_kernel<D>>(int(smem));
  if (e != cudaSuccess) return e;
  dim3 grid((p.Lmax + kRows - 1) / kRows, p.Hq, p.B);
  attn_fp32_kernel<D><<<grid, kRows, smem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fp32(const AttnFp32Params& p, cudaStream_t stream) {
  return p.D == 128 ? launch_impl<128>(p, stream) : launch_impl<64>(p, stream);
}

}  // namespace parse
