// Microbenchmark: does the accumulate flag, the D column or the TMEM A column
// change tcgen05.mma (kind::f16, M=128, N=128, K=16) throughput?  Groups of 8
// K-steps; compile-time variants only (no predicated MMAs in the issue loop).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/mma_modes.cu -o build/mma_modes && build/mma_modes
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 256;

// TS: A from TMEM; FIRST0: the first K-step of each group overwrites D; DCOL / ACOL: TMEM columns
template <bool TS, bool FIRST0, int DCOL, int ACOL, bool MN>
__global__ void __launch_bounds__(128, 1) bench(long long* out) {
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
    const uint32_t idesc = make_idesc_bf16(128, 128, MN ? 1 : 0);
    const uint64_t ad = make_sdesc_sw128(sb, 16, 1024);
    const uint64_t bd = MN ? make_sdesc_sw128(sb + 65536, 16384, 1024) : make_sdesc_sw128(sb + 65536, 16, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = MN ? uint64_t((kk * 2048) >> 4) : uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          const uint32_t acc = (FIRST0 && kk == 0) ? 0u : 1u;
          if (TS) mma_ts(tmem + DCOL, tmem + ACOL + kk * 8, bd + off, idesc, acc);
          else mma_ss(tmem + DCOL, ad + off, bd + off, idesc, acc);
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

template <bool TS, bool FIRST0, int DCOL, int ACOL, bool MN>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = bench<TS, FIRST0, DCOL, ACOL, MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  k<<<148, 128, 140 * 1024>>>(d);
  k<<<148, 128, 140 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (kIters * 8);
  printf("%-44s %6.1f cycles/MMA -> %5.1f%% of peak  [%s]\n", name, per, 100.0 * 64.0 / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<false, false, 256, 0, false>("SS D@256 always accumulate");
  run<false, true, 256, 0, false>("SS D@256 first K-step overwrites");
  run<false, false, 0, 0, false>("SS D@0 always accumulate");
  run<false, true, 0, 0, false>("SS D@0 first K-step overwrites");
  run<true, false, 256, 0, true>("TS A@0 D@256 MN-major B");
  run<true, false, 256, 128, true>("TS A@128 D@256 MN-major B");
  run<true, true, 256, 128, true>("TS A@128 D@256 first overwrites");
  run<true, false, 384, 192, true>("TS A@192 D@384 MN-major B");
  return 0;
}
