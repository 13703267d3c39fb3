// Probe of the 2-SM tensor-core path (groundwork for the cta_group::2 kernel,
// DESIGN "Next"): a cluster of 2 CTAs computes D[256 x 128] = A[256 x 64] *
// B[128 x 64]^T with ONE tcgen05.mma.cta_group::2 stream issued by the leader
// CTA.  Each CTA holds its 128 rows of A and one half (64 rows) of B in shared
// memory (SW128, K-major), TMEM is allocated with cta_group::2, the commit
// multicasts to both CTAs' barriers, and each CTA reads its own 128 rows of D
// from TMEM.  The host checks D against an fp64 reference, and also reports
// which B half each CTA must hold.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/cta2_probe.cu -o build/cta2_probe && build/cta2_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kM = 256, kN = 128, kK = 64;

// byte offset of element (r, k) in a K-major SW128 tile with 128-byte rows
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  const uint32_t off = uint32_t(r) * 128u + uint32_t(k) * 2u;
  const uint32_t chunk = ((off >> 4) & 7u) ^ (uint32_t(r) & 7u);
  return (off & ~0x70u) | (chunk << 4);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int b_half_of_rank) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];   // 128 rows x 64 bf16
  __shared__ __align__(1024) uint8_t sb[64 * 128];    // 64 rows x 64 bf16
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = cluster_rank();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // fill this CTA's operands (generic stores in the swizzled layout)
  for (int i = threadIdx.x; i < 128 * kK; i += 128) {
    const int r = i / kK, k = i % kK;
    *reinterpret_cast<__nv_bfloat16*>(sa + sw128(r, k)) = A[(rank * 128 + r) * kK + k];
  }
  const int bh = b_half_of_rank ? int(rank) : 0;      // which 64-row half of B this CTA holds
  for (int i = threadIdx.x; i < 64 * kK; i += 128) {
    const int r = i / kK, k = i % kK;
    *reinterpret_cast<__nv_bfloat16*>(sb + sw128(r, k)) = B[(bh * 64 + r) * kK + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(smem_u32(&bar), 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (rank == 0 && warp == 0) {
    // M = 256 (both CTAs' A), N = 128 (both CTAs' B halves), kind::f16 bf16 -> fp32
    const uint32_t idesc = make_idesc_bf16(kM, kN, 0);
    const uint64_t ad = make_sdesc_sw128(smem_u32(sa), 16, 1024);
    const uint64_t bd = make_sdesc_sw128(smem_u32(sb), 16, 1024);
    if (elect_one()) {
#pragma unroll
      for (int kk = 0; kk < kK / 16; ++kk) {
        const uint64_t off = uint64_t((kk * 32) >> 4);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad + off), "l"(bd + off), "r"(idesc), "r"(kk > 0 ? 1 : 0)
            : "memory");
      }
      asm volatile(
          "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
              smem_u32(&bar))
          : "memory");
    }
    __syncwarp();
  }
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  // each warp reads its 32 TMEM lanes (= rows of this CTA's half of D)
  for (int c = 0; c < kN; c += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) D[(rank * 128 + warp * 32 + lane) * kN + c + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128) : "memory");
}

int main() {
  __nv_bfloat16 *hA = new __nv_bfloat16[kM * kK], *hB = new __nv_bfloat16[kN * kK];
  srand(1);
  for (int i = 0; i < kM * kK; ++i) hA[i] = __float2bfloat16(float(rand() % 17 - 8) / 8.f);
  for (int i = 0; i < kN * kK; ++i) hB[i] = __float2bfloat16(float(rand() % 17 - 8) / 8.f);
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(__nv_bfloat16) * kM * kK);
  cudaMalloc(&dB, sizeof(__nv_bfloat16) * kN * kK);
  cudaMalloc(&dD, sizeof(float) * kM * kN);
  cudaMemcpy(dA, hA, sizeof(__nv_bfloat16) * kM * kK, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(__nv_bfloat16) * kN * kK, cudaMemcpyHostToDevice);
  float* hD = new float[kM * kN];
  for (int mode = 1; mode >= 0; --mode) {
    cudaMemset(dD, 0, sizeof(float) * kM * kN);
    probe<<<2, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, sizeof(float) * kM * kN, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < kM; ++m)
      for (int n = 0; n < kN; ++n) {
        double ref = 0;
        for (int k = 0; k < kK; ++k) ref += double(__bfloat162float(hA[m * kK + k])) * __bfloat162float(hB[n * kK + k]);
        maxerr = fmax(maxerr, fabs(ref - hD[m * kN + n]));
      }
    printf("B half per CTA rank = %s: %s, max |D - ref| = %.3e -> %s\n", mode ? "rank" : "0 (both hold rows 0-63)",
           cudaGetErrorString(e), maxerr, maxerr < 1e-3 ? "MATCH" : "mismatch");
  }
  return 0;
}
