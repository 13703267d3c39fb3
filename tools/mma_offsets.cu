// Microbenchmark: SS tcgen05.mma (kind::f16, M=128, N=128, K=16, 128B swizzle,
// both operands K-major) throughput against the shared-memory offsets of A
// and B.  The attention kernel keeps Q tiles at 0 / 32 KB and K/V stages at
// 64 KB + s * 32 KB; this checks which relative placements run at full rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_offsets.cu -o build/mma_offsets && build/mma_offsets
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 256;

__global__ void __launch_bounds__(128, 1) bench(long long* out, int a_off, int b_off, int ts) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  const uint32_t sb = (smem_u32(smem) + 1023) & ~1023u;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 1) { tmem_alloc(smem_u32(&tslot), 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 128, ts);
    const uint64_t ad = make_sdesc_sw128(sb + a_off, 16, 1024);
    const uint64_t bd = ts ? make_sdesc_sw128(sb + b_off, 16384, 1024) : make_sdesc_sw128(sb + b_off, 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (ts) {
            mma_ts(tmem + 256, tmem + 128 + kk * 8, bd + uint64_t((kk * 2048) >> 4), idesc, 1);
          } else {
            const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
            mma_ss(tmem, ad + off, bd + off, idesc, kk > 0);
          }
        }
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

double run(int a_off, int b_off, int ts) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 231424);
  bench<<<148, 128, 231424>>>(d, a_off, b_off, ts);
  bench<<<148, 128, 231424>>>(d, a_off, b_off, ts);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  cudaFree(d);
  return avg / 148 / (kIters * 8);
}

int main() {
  const int K = 1024;
  int as[] = {0, 32 * K};
  for (int a : as) {
    printf("A at %3d KB:", a / K);
    for (int b = 64 * K; b <= 192 * K; b += 32 * K) printf("  B@%3dK %5.1f", b / K, run(a, b, 0));
    printf("\n");
  }
  printf("A at 0, B at A + d (KB):");
  int ds[] = {1, 2, 4, 8, 16, 17, 24, 32, 33, 40, 48, 64, 65, 80, 96, 112, 128};
  for (int d : ds) printf(" %d:%.1f", d, run(0, 64 * K + (d - 64) * K > 0 ? d * K : d * K, 0));
  printf("\n");
  printf("A at 0, B at 64 KB + s*32 KB + skew (KB), s = 0..4:\n");
  int skews[] = {0, 1, 2, 4, 8, 16};
  for (int sk : skews) {
    printf("  skew %2d:", sk);
    for (int s = 0; s < 4; ++s) printf("  %5.1f/%5.1f", run(0, 64 * K + s * 33 * K + sk * K, 0), run(32 * K + sk * K, 64 * K + s * 33 * K, 0));
    printf("\n");
  }
  printf("TS (PV form), B at 64 KB + s*32 KB:");
  for (int s = 0; s < 5; ++s) printf("  %5.1f", run(0, 64 * K + s * 32 * K, 1));
  printf("\n");
  return 0;
}
