// Probe the thread <-> (lane, column) mapping of tcgen05.ld shapes 16x256b,
// 16x128b, 16x64b: fill TMEM with value = lane*1024 + col via 32x32b stores,
// load with the probed shape, print which (lane, col) each thread receives.
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace parse_sm100;

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 32); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  // each warp (4) writes its 32 lanes x 32 columns
  uint32_t v[32];
  for (int c = 0; c < 32; ++c) v[c] = (warp * 32 + lane) * 1024 + c;
  tmem_st32(tm + ((warp * 32) << 16), v);
  tmem_wait_st();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 1) {
    // lane base 48 = second 16-lane half of warp 1's quarter
    uint32_t a[4];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(tm + (48u << 16)));
    uint32_t b[4];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]) : "r"(tm + (48u << 16)));
    tmem_wait_ld();
    for (int i = 0; i < 4; ++i) out[512 + lane * 8 + i] = a[i];
    for (int i = 0; i < 4; ++i) out[512 + lane * 8 + 4 + i] = b[i];
  }
  if (warp == 0) {
    uint32_t a[4], b[2], c1;
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(tm));
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(tm));
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(c1) : "r"(tm));
    tmem_wait_ld();
    for (int i = 0; i < 4; ++i) out[lane * 8 + i] = a[i];
    out[lane * 8 + 4] = b[0]; out[lane * 8 + 5] = b[1]; out[lane * 8 + 6] = c1;
    // x2 of 16x256b: second repetition columns
    uint32_t d[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]) : "r"(tm));
    tmem_wait_ld();
    out[256 + lane * 8 + 0] = d[4]; out[256 + lane * 8 + 1] = d[5]; out[256 + lane * 8 + 2] = d[6]; out[256 + lane * 8 + 3] = d[7];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tm, 32); }
}
int main() {
  uint32_t* d; cudaMalloc(&d, 1024 * 4); cudaMemset(d, 0xff, 1024 * 4);
  probe<<<1, 128>>>(d);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  uint32_t h[1024]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  auto f = [](uint32_t x) { static char buf[32]; snprintf(buf, 32, "(%u,%u)", x / 1024, x % 1024); return buf; };
  for (int t = 0; t < 32; ++t) {
    printf("t%2d 16x256b:", t);
    for (int i = 0; i < 4; ++i) printf(" %s", f(h[t * 8 + i]));
    printf(" | x2 rep1:");
    for (int i = 0; i < 4; ++i) printf(" %s", f(h[256 + t * 8 + i]));
    printf(" | 16x128b: %s", f(h[t * 8 + 4])); printf(" %s", f(h[t * 8 + 5]));
    printf(" | 16x64b: %s\n", f(h[t * 8 + 6]));
  }
  for (int t = 0; t < 32; ++t) {
    printf("w1 base48 t%2d 16x256b.x1:", t);
    for (int i = 0; i < 4; ++i) printf(" %s", f(h[512 + t * 8 + i]));
    printf(" | 16x128b.x2:");
    for (int i = 0; i < 4; ++i) printf(" %s", f(h[512 + t * 8 + 4 + i]));
    printf("\n");
  }
}
