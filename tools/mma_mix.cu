// Microbenchmark: tensor-pipe throughput when SS (QK^T form) and TS (PV form)
// groups of 8 tcgen05.mma (M=128, N=128, K=16) alternate, from one warp or
// from two warps issuing concurrently (the attention kernel's two MMA warps).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_mix.cu -o build/mma_mix && build/mma_mix
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 128;   // groups per stream

// MODE 0: one warp, SS groups only; 1: one warp, TS only; 2: one warp, SS/TS
// alternating; 3: warp 0 SS groups + warp 1 TS groups concurrently;
// 4: warp 0 SS + warp 1 SS (two QK streams); 5: two warps each alternating SS/TS
template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x / 32;
  const uint32_t sb = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar[0]), 1); mbar_init(smem_u32(&bar[1]), 1); fence_mbar_init(); }
  if (warp == 2) { tmem_alloc(smem_u32(&tslot), 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const bool active = warp == 0 || (warp == 1 && MODE >= 3);
  if (active) {
    const uint32_t idesc_ss = make_idesc_bf16(128, 128, 0);
    const uint32_t idesc_ts = make_idesc_bf16(128, 128, 1);
    const uint64_t qd = make_sdesc_sw128(sb + warp * 32768, 16, 1024);
    const uint64_t kd = make_sdesc_sw128(sb + 65536, 16, 1024);
    const uint64_t vd = make_sdesc_sw128(sb + 98304 + warp * 32768, 16384, 1024);
    const uint32_t s_t = tmem + (warp == 0 ? 0 : 128);   // separate S columns per warp
    const uint32_t p_t = tmem + 256 + warp * 64;
    const uint32_t o_t = tmem + 384;   // junk accumulate target shared by both
    auto ss = [&]() {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
        mma_ss(s_t, qd + off, kd + off, idesc_ss, kk > 0);
      }
    };
    auto ts = [&]() {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) mma_ts(o_t, p_t + kk * 8, vd + uint64_t((kk * 2048) >> 4), idesc_ts, 1);
    };
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; it += 2) {
        if (MODE == 0 || MODE == 4 || (MODE == 3 && warp == 0)) { ss(); ss(); }
        else if (MODE == 1 || (MODE == 3 && warp == 1)) { ts(); ts(); }
        else { ss(); ts(); }
      }
      mma_commit(smem_u32(&bar[warp]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar[warp]), 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 2 + warp] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaMemset(d, 0, 2 * 148 * sizeof(long long));
  auto k = bench<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, 128, 200 * 1024>>>(d);
  k<<<148, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (h[2 * i] > h[2 * i + 1] ? h[2 * i] : h[2 * i + 1]);
  avg /= 148;
  const int groups = kIters * (MODE >= 3 ? 2 : 1);
  printf("%-44s %7.1f cycles per group of 8 (ideal 512) -> %5.1f%%  [%s]\n", name, avg / groups,
         100.0 * 512.0 * groups / avg, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("one warp: SS groups");
  run<1>("one warp: TS groups");
  run<2>("one warp: SS/TS alternating");
  run<3>("warp 0 SS groups + warp 1 TS groups");
  run<4>("warp 0 SS groups + warp 1 SS groups");
  run<5>("two warps, each SS/TS alternating");
  return 0;
}
