// Microbenchmark: tcgen05.mma (kind::f16, M=128, N=128, K=16, 128B swizzle)
// throughput under the traffic the attention kernel puts beside it:
//   pattern 0: SS (A and B from shared memory, the QK^T form)
//   pattern 1: TS (A from TMEM, B from shared memory, the PV form)
//   pattern 2: groups of 8 SS then 8 TS, alternating (one QK^T + one PV per step)
//   extra bit 1: 8 warps stream tcgen05.ld (32x32b.x64, two per 128 columns)
//                like the softmax's S loads
//   extra bit 2: one warp streams 32 KB TMA bulk copies global -> shared
//                (the K/V tile loads)
//   extra bit 8: Q / K / V tiles filled with random N(0,1) bf16 (else whatever is there)
//   extra bit 4: 8 warps run softmax-like FFMA2 / MUFU.EX2 / F2FP work and
//                tcgen05.st 64 columns per round (P stores) on all SMSPs
// Patterns and extras are template parameters: a runtime SS/TS branch in the
// issue loop compiles to predicated UTCHMMA pairs, which cost ~10-40 cycles
// per MMA by themselves (tools/mma_offsets.cu measures that artefact).
// One CTA per SM, 384 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_contend.cu -o build/mma_contend && build/mma_contend
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 256;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int pattern, int extra>
__global__ void __launch_bounds__(384, 1) bench(long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  const uint32_t sb = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    done = 0;
    fence_mbar_init();
  }
  if (warp == 1) { tmem_alloc(smem_u32(&tslot), 512); tmem_relinquish(); }
  if (extra & 8) {
    // operand tiles filled with the bf16 data the kernel multiplies (random normal)
    const uint4* src = reinterpret_cast<const uint4*>(gsrc);
    uint4* dst = reinterpret_cast<uint4*>(smem + (sb - smem_u32(smem)));
    for (int i = threadIdx.x; i < 98304 / 16; i += blockDim.x) dst[i] = src[i];
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc_ss = make_idesc_bf16(128, 128, 0);
    const uint32_t idesc_ts = make_idesc_bf16(128, 128, 1);
    const uint64_t ad = make_sdesc_sw128(sb, 16, 1024);              // Q tile at 0
    const uint64_t bd = make_sdesc_sw128(sb + 32768, 16, 1024);      // K tile at 32 KB
    const uint64_t vd = make_sdesc_sw128(sb + 65536, 16384, 1024);   // V tile at 64 KB (MN-major)
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; ++it) {
        const bool ss = pattern == 0 || (pattern == 2 && (it & 1) == 0);   // compile-time for 0 / 1
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (ss) {
            const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            mma_ss(tmem + 0, ad + off, bd + off, idesc_ss, kk > 0);
          } else {
            const uint64_t voff = uint64_t((kk * 2 * 1024) >> 4);
            mma_ts(tmem + 256, tmem + 128 + kk * 8, vd + voff, idesc_ts, 1);
          }
        }
      }
      mma_commit(smem_u32(&bar[0]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar[0]), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; done = 1; }
  } else if (warp == 2 && (extra & 2)) {
    // K/V tile loads: 32 KB bulk copies into [96 KB, 128 KB), one at a time
    uint32_t ph = 0;
    for (int r = 0; r < 4096 && !done; ++r) {
      if (elect_one()) {
        mbar_arrive_expect_tx(smem_u32(&bar[1]), 32768);
        bulk_g2s(sb + 98304, gsrc + (size_t(blockIdx.x) % 64) * 32768, 32768, smem_u32(&bar[1]));
      }
      __syncwarp();
      mbar_wait(smem_u32(&bar[1]), ph);
      ph ^= 1;
    }
  } else if (warp >= 4 && (extra & 4)) {
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    float x[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int r = 0; r < 4096 && !done; ++r) {
#pragma unroll
      for (int i = 0; i < 64; i += 2) {
        float2 v = ffma2(make_float2(x[i], x[i + 1]), make_float2(0.5f, 0.5f), make_float2(-1.f, -1.f));
        x[i] = ex2(v.x);
        x[i + 1] = v.y;
      }
      uint32_t pk[16];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(x[(16 * c + e) & 63], x[(16 * c + e + 1) & 63]);
        tmem_st16(tmem + lane_base + 384 + 16 * c, pk);
      }
      tmem_wait_st();
    }
    if (x[5] == 1234.5f) out[1001] = 1;
  } else if (warp >= 4 && (extra & 1)) {
    // softmax-like S loads: each warp its 32 lanes x 128 columns
    const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    for (int r = 0; r < 4096 && !done; ++r) {
      uint32_t sr[128];
      tmem_ld64(tmem + lane_base, sr);
      tmem_ld64(tmem + lane_base + 64, sr + 64);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 128; ++i) acc += sr[i];
    }
    if (acc == 0x12345678u) out[1000] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int pattern, int extra>
void run(const char* name, const uint8_t* g) {
  long long* d;
  cudaMalloc(&d, 2048 * sizeof(long long));
  auto k = bench<pattern, extra>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<148, 384, 140 * 1024>>>(d, g);
  k<<<148, 384, 140 * 1024>>>(d, g);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (kIters * 8);
  printf("%-26s tmem_ld=%d tma=%d alu+sttm=%d: %6.1f cycles/MMA -> %5.1f%% of peak  [%s]\n", name, extra & 1,
         (extra >> 1) & 1, (extra >> 2) & 1, per, 100.0 * 64.0 / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  uint8_t* g;
  cudaMalloc(&g, 64 * 32768);
  {
    // bf16 ~ N(0, 1) (Box-Muller on the host), the kernel's operand distribution
    static unsigned short h[64 * 16384];
    unsigned s = 12345u;
    for (int i = 0; i < 64 * 16384; i += 2) {
      s = s * 1664525u + 1013904223u; float u1 = ((s >> 8) + 1) / 16777217.f;
      s = s * 1664525u + 1013904223u; float u2 = (s >> 8) / 16777216.f;
      float r = sqrtf(-2.f * logf(u1)), a = 6.2831853f * u2;
      float v[2] = {r * cosf(a), r * sinf(a)};
      for (int e = 0; e < 2; ++e) { unsigned b; memcpy(&b, &v[e], 4); h[i + e] = (unsigned short)((b + 0x8000u) >> 16); }
    }
    cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  }
  run<0, 0>("SS N128 zeros", g);
  run<0, 8>("SS N128 random bf16", g);
  run<1, 0>("TS N128 zeros", g);
  run<1, 8>("TS N128 random bf16 (A: TMEM junk)", g);
  run<0, 12>("SS random + alu/sttm", g);
  run<0, 15>("SS random + all", g);
  return 0;
}
