// Microbenchmark: when two warps (on different SMSPs) each issue one group of
// 8 tcgen05.mma (M=128, N=128, K=16) at the same time, does the tensor core
// run the groups one after the other (completions ~512 and ~1024 cycles
// after the start) or interleave them (both complete at ~1024)?  A third warp
// timestamps both commits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_interleave.cu -o build/mma_interleave && build/mma_interleave
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok != 0;
}

// MODE 0: only warp 1 issues; 1: warps 1 and 3 issue together (SS + SS);
// 2: warps 1 (SS) and 3 (TS) together; 3: warp 1 issues both groups back to back
template <int MODE>
__global__ void __launch_bounds__(128, 1) bench(long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[3];
  __shared__ volatile int go;
  const int warp = threadIdx.x / 32;
  const uint32_t sb = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) { for (int i = 0; i < 3; ++i) mbar_init(smem_u32(&bar[i]), 1); go = 0; fence_mbar_init(); }
  if (warp == 2) { tmem_alloc(smem_u32(&tslot), 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc_ss = make_idesc_bf16(128, 128, 0), idesc_ts = make_idesc_bf16(128, 128, 1);
  const uint64_t qd = make_sdesc_sw128(sb, 16, 1024), kd = make_sdesc_sw128(sb + 65536, 16, 1024);
  const uint64_t vd = make_sdesc_sw128(sb + 98304, 16384, 1024);
  auto ss = [&](uint32_t d) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
      mma_ss(tmem + d, qd + off, kd + off, idesc_ss, kk > 0);
    }
  };
  auto ts = [&](uint32_t d) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + d, tmem + 128 + kk * 8, vd + uint64_t((kk * 2048) >> 4), idesc_ts, 1);
  };
  long long t0 = 0;
  if (warp == 0) {
    // observer: release the issuers, then timestamp both completions
    uint32_t done[2] = {0, 0};
    long long tc[2] = {0, 0};
    __syncwarp();
    t0 = clock64();
    if (threadIdx.x == 0) go = 1;
    const int need = MODE == 0 ? 1 : 2;
    int got = 0;
    while (got < need) {
      for (int i = 0; i < 2; ++i)
        if (!done[i] && test_wait(smem_u32(&bar[i]), 0)) { done[i] = 1; tc[i] = clock64(); ++got; }
    }
    if (threadIdx.x == 0) { out[blockIdx.x * 2] = tc[0] - t0; out[blockIdx.x * 2 + 1] = tc[1] - t0; }
  } else if (warp == 1 || (warp == 3 && (MODE == 1 || MODE == 2))) {
    while (!go) {}
    if (elect_one()) {
      if (warp == 1) { ss(0); mma_commit(smem_u32(&bar[0])); if (MODE == 3) { ss(256); mma_commit(smem_u32(&bar[1])); } }
      else { if (MODE == 1) ss(256); else ts(256); mma_commit(smem_u32(&bar[1])); }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  auto k = bench<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int r = 0; r < 3; ++r) k<<<148, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double a = 0, b = 0;
  for (int i = 0; i < 148; ++i) { a += h[2 * i]; b += h[2 * i + 1]; }
  printf("%-46s group A done at %6.0f, group B at %6.0f cycles  [%s]\n", name, a / 148, b / 148, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0>("one warp, one SS group");
  run<3>("one warp, two SS groups back to back");
  run<1>("warps 1 and 3 (two SMSPs), one SS group each");
  run<2>("warp 1 SS group + warp 3 TS group");
  return 0;
}
