// Does a tcgen05.mma that overwrites TMEM columns read (as the A operand) by
// the previous MMAs cost a pipeline drain?  Loop of [8 TS MMAs reading A from
// TMEM columns 0-63 into D at 256] + [8 SS MMAs writing D = columns 0-127
// (overlap) or 128-255 (no overlap)], cycles per MMA.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 256;

template <bool kOverlap>
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
    const uint32_t id_qk = make_idesc_bf16(128, 128, 0);
    const uint32_t id_pv = make_idesc_bf16(128, 128, 1);
    const uint64_t ad = make_sdesc_sw128(sb, 16, 1024);
    const uint64_t bd = make_sdesc_sw128(sb + 32768, 16, 1024);
    const uint64_t vd = make_sdesc_sw128(sb + 65536, 16384, 1024);
    long long t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ts(tmem + 256, tmem + kk * 8, vd + uint64_t((kk * 2048) >> 4), id_pv, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t off = uint64_t(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4);
          mma_ss(tmem + (kOverlap ? 0 : 128), ad + off, bd + off, id_qk, kk > 0);
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

template <bool kOverlap>
void run(const char* name) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  auto k = bench<kOverlap>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<148, 128, 200 * 1024>>>(d);
  k<<<148, 128, 200 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-40s %6.1f cycles per MMA (ideal 64) [%s]\n", name, avg / (kIters * 16), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<true>("PV(A from S cols 0-63) -> QK into cols 0-127");
  run<false>("PV(A from S cols 0-63) -> QK into cols 128-255");
  return 0;
}
