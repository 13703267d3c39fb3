// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128) for SS / TS
// operand sources and several N, optionally with other warps streaming
// st.shared traffic (a stand-in for TMA writes).  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_bench.cu -o build/mma_bench && build/mma_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 256;

template <int N, bool TS, int MN = 0>
__global__ void __launch_bounds__(256, 1) mma_bench(long long* out, int smem_writers) {
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
    const uint32_t idesc = make_idesc_bf16(128, N, MN);
    const uint64_t ad = make_sdesc_sw128(sb, 16, 1024);
    const uint64_t bd = MN ? make_sdesc_sw128(sb + 65536, 16384, 1024) : make_sdesc_sw128(sb + 65536, 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = MN ? uint64_t((kk * 2048) >> 4) : uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          if (TS) mma_ts(tmem + 256, tmem + kk * 8, bd + off, idesc, 1);
          else mma_ss(tmem + 256, ad + off, bd + off, idesc, 1);
        }
      }
      mma_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  } else if (warp >= 4 && smem_writers) {
    // stream 16-byte stores over a 32 KB region (~TMA write traffic)
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    volatile uint4* dst = reinterpret_cast<volatile uint4*>(smem + 131072);
    for (int r = 0; r < kIters * 8; ++r)
      for (int i = threadIdx.x - 128; i < 2048; i += 128) const_cast<uint4*>(dst)[i] = v;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, int MN = 0>
void run(const char* name, int writers) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = mma_bench<N, TS, MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, 256, 200 * 1024>>>(d, writers);
  k<<<148, 256, 200 * 1024>>>(d, writers);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (kIters * 8);
  const double ideal = 128.0 * N / 256.0;
  printf("%-28s writers=%d: %7.1f cycles/MMA (ideal %5.1f) -> %5.1f%% of peak  [%s]\n", name, writers, per, ideal,
         100.0 * ideal / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int w = 0; w < 2; ++w) {
    run<128, false>("SS M128 N128", w);
    run<64, false>("SS M128 N64", w);
    run<256, false>("SS M128 N256", w);
    run<128, true>("TS M128 N128", w);
    run<64, true>("TS M128 N64", w);
    run<256, true>("TS M128 N256", w);
    run<128, true, 1>("TS M128 N128 B MN-major", w);
  }
  return 0;
}
