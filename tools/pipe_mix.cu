// Microbenchmark: which sm_100 pipes the softmax's instructions share.
// Each kernel runs a fixed mix of instructions over 8 independent chains per
// thread, 16 warps per CTA (4 per SMSP); the printed figure is cycles per
// iteration per warp per SMSP, so a mix of two instruction kinds that costs
// the SUM of their single costs shares a pipe, one that costs the MAX does not.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/pipe_mix.cu -o build/pipe_mix
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

__device__ __forceinline__ void ffma2(uint64_t& a, uint64_t b) {
  asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a) : "l"(b));
}
__device__ __forceinline__ void fadd2(uint64_t& a, uint64_t b) {
  asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(b));
}
__device__ __forceinline__ void f2fp(uint32_t& d, float a, float b) {
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b));
}
__device__ __forceinline__ void mnmx3(float& a, float b, float c) {
  asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(b), "f"(c));
}
__device__ __forceinline__ void ex2f(float& a) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a)); }
__device__ __forceinline__ void hfma2bf(uint32_t& a, uint32_t b) {
  asm volatile("fma.rn.bf16x2 %0, %0, %1, %1;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void hfma2h(uint32_t& a, uint32_t b) {
  asm volatile("fma.rn.f16x2 %0, %0, %1, %1;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void hadd2h(uint32_t& a, uint32_t b) {
  asm volatile("add.rn.f16x2 %0, %0, %1;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void prmt(uint32_t& a, uint32_t b) {
  asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void lea(uint32_t& a, uint32_t b) {
  asm volatile("{\n\t.reg .u32 t;\n\tshl.b32 t, %1, 7;\n\tadd.u32 %0, %0, t;\n\t}" : "+r"(a) : "r"(b));
}
__device__ __forceinline__ void iadd(uint32_t& a, uint32_t b) { asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b)); }
__device__ __forceinline__ void shl(uint32_t& a) { asm volatile("shl.b32 %0, %0, 3;" : "+r"(a)); }
__device__ __forceinline__ void cvt_f32_bf16(float& d, uint32_t a) {
  asm volatile("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %1;\n\tcvt.f32.bf16 %0, hi;\n\t}" : "=f"(d) : "r"(a));
}
__device__ __forceinline__ void ex2bf2(uint32_t& a) { asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a)); }
__device__ __forceinline__ void ex2h2(uint32_t& a) { asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a)); }
__device__ __forceinline__ void e4m3(uint32_t& d, float a, float b) {
  asm volatile("{\n\t.reg .b16 t;\n\tcvt.rn.satfinite.e4m3x2.f32 t, %1, %2;\n\tcvt.u32.u16 %0, t;\n\t}" : "=r"(d) : "f"(a), "f"(b));
}

// mask bits: 1 FFMA2, 2 FADD2, 4 F2FP, 8 FMNMX3, 16 MUFU.EX2, 32 HFMA2.BF16, 64 HFMA2.F16,
// 128 PRMT, 256 SHL+ADD, 512 IADD, 1024 SHL, 2048 HADD2.F16, 4096 cvt f32<-bf16, 8192 e4m3x2
template <int MASK>
__global__ void __launch_bounds__(512, 1) bench(float* out, long long* cyc, float seed) {
  uint64_t a[8];
  uint32_t u[8];
  float f[8];
  const uint64_t b = 0x3f0000003f000000ull;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (uint64_t(__float_as_uint(seed + i)) << 32) | __float_as_uint(seed * 0.5f + threadIdx.x * 1e-3f);
    u[i] = 0x3f803f80u + i + threadIdx.x * 3u;
    f[i] = seed * 1e-3f * i - 1.f;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MASK & 1) ffma2(a[i], b);
      if (MASK & 2) fadd2(a[i], b);
      if (MASK & 4) f2fp(u[i], __uint_as_float(u[i]), f[i]);
      if (MASK & 8) mnmx3(f[i], f[(i + 1) & 7], f[(i + 2) & 7]);
      if (MASK & 16) ex2f(f[i]);
      if (MASK & 32) hfma2bf(u[i], 0x3f003f00u);
      if (MASK & 64) hfma2h(u[i], 0x38003800u);
      if (MASK & 128) prmt(u[i], u[(i + 1) & 7]);
      if (MASK & 256) lea(u[i], u[(i + 1) & 7]);
      if (MASK & 512) iadd(u[i], u[(i + 1) & 7]);
      if (MASK & 1024) shl(u[i]);
      if (MASK & 2048) hadd2h(u[i], 0x38003800u);
      if (MASK & 4096) cvt_f32_bf16(f[i], __float_as_uint(f[i]));
      if (MASK & 8192) e4m3(u[i], __uint_as_float(u[i]), f[i]);
      if (MASK & 16384) ex2bf2(u[i]);
      if (MASK & 32768) ex2h2(u[i]);
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(uint32_t(a[i])) + __uint_as_float(u[i]) + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MASK>
void run(const char* name) {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 512 * 4);
  cudaMalloc(&c, 148 * 8);
  bench<MASK><<<148, 512>>>(o, c, 1.f);
  bench<MASK><<<148, 512>>>(o, c, 1.f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  // 4 warps per SMSP, 8 instructions of each kind per iteration per warp
  printf("%-28s %6.2f cycles per 8-instruction group per warp (4 warps / SMSP)\n", name, avg / (4.0 * kIters));
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<16>("MUFU.EX2 f32");
  run<16384>("ex2.approx.ftz.bf16x2");
  run<32768>("ex2.approx.f16x2");
  run<16 | 16384>("EX2 f32 + ex2 bf16x2");
  run<1 | 16384>("FFMA2 + ex2 bf16x2");
  run<4 | 16384>("F2FP + ex2 bf16x2");
  return 0;
}
