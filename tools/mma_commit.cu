// Microbenchmark: cost of tcgen05.commit (mbarrier::arrive::one) placed after
// every group of 8 tcgen05.mma (M=128, N=128, K=16; SS), from one warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_commit.cu -o build/mma_commit && build/mma_commit
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kGroups = 256;

// NC commits per group (to distinct barriers nobody waits on); GAP: clock64
// timestamps around the commits of group 100 are written to out2
template <int NC>
__global__ void __launch_bounds__(128, 1) bench(long long* out, long long* out2) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x / 32;
  const uint32_t sb = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&bar[i]), 1);
    fence_mbar_init();
  }
  if (warp == 1) { tmem_alloc(smem_u32(&tslot), 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 128, 0);
    const uint64_t ad = make_sdesc_sw128(sb, 16, 1024);
    const uint64_t bd = make_sdesc_sw128(sb + 65536, 16, 1024);
    long long t0 = clock64(), ta = 0, tb = 0, tc = 0;
    if (elect_one()) {
      for (int g = 0; g < kGroups; ++g) {
        if (g == 100) ta = clock64();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          mma_ss(tmem + (g & 1) * 128, ad + off, bd + off, idesc, kk > 0);
        }
        if (g == 100) tb = clock64();
#pragma unroll
        for (int c = 0; c < NC; ++c) mma_commit(smem_u32(&bar[1 + c]));
        if (g == 100) tc = clock64();
      }
      mma_commit(smem_u32(&bar[0]));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar[0]), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (elect_one() && blockIdx.x == 0) { out2[0] = tb - ta; out2[1] = tc - tb; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int NC>
void run() {
  long long *d, *d2;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&d2, 4 * sizeof(long long));
  auto k = bench<NC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<148, 128, 140 * 1024>>>(d, d2);
  k<<<148, 128, 140 * 1024>>>(d, d2);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148], h2[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%d commit(s) per group: %6.1f cycles per group (ideal 512) -> %5.1f%%; group 100: 8 MMAs issued in %lld, "
         "commits in %lld cycles  [%s]\n", NC, avg / kGroups, 100.0 * 512 * kGroups / avg, h2[0], h2[1], cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(d2);
}

int main() {
  run<0>();
  run<1>();
  run<2>();
  run<3>();
  return 0;
}
