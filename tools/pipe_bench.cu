// Microbenchmark: per-SM-sub-partition throughput of the instructions the
// softmax uses.  16 warps per CTA (4 per SMSP), 8 independent chains each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_04263_b200/csrc \
//        tools/pipe_bench.cu -o build/pipe_bench && build/pipe_bench
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace parse_sm100;

constexpr int kIters = 4096;

template <int OP>
__global__ void __launch_bounds__(512, 1) bench(float* out, long long* cyc, float seed) {
  float a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed + threadIdx.x * 1e-3f + i; b[i] = 0.5f + i * 1e-2f; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      if (OP == 0) {  // FFMA2
        float2 r = ffma2(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]), make_float2(b[i + 1], b[i]));
        a[i] = r.x; a[i + 1] = r.y;
      } else if (OP == 1) {  // FADD2
        float2 r = fadd2(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]));
        a[i] = r.x; a[i + 1] = r.y;
      } else if (OP == 2) {  // FFMA scalar x2
        a[i] = fmaf(a[i], b[i], b[i + 1]);
        a[i + 1] = fmaf(a[i + 1], b[i + 1], b[i]);
      } else if (OP == 3) {  // MUFU.EX2 x2
        a[i] = ex2(a[i]);
        a[i + 1] = ex2(a[i + 1]);
      } else if (OP == 4) {  // F2FP pack (one per pair)
        uint32_t p = pack_bf16x2(a[i], a[i + 1]);
        a[i] = __uint_as_float(p);
      } else if (OP == 5) {  // FMNMX3 (two per pair)
        a[i] = fmax3(a[i], b[i], a[i + 1]);
        a[i + 1] = fmax3(a[i + 1], b[i + 1], a[i]);
      } else if (OP == 6) {  // shift (two per pair)
        a[i] = __uint_as_float(__float_as_uint(a[i]) << 1);
        a[i + 1] = __uint_as_float(__float_as_uint(a[i + 1]) << 1);
      } else if (OP == 7) {  // FMUL2
        float2 r = fmul2(make_float2(a[i], a[i + 1]), make_float2(b[i], b[i + 1]));
        a[i] = r.x; a[i + 1] = r.y;
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int instr_per_iter_per_warp) {
  float* o;
  long long* c;
  cudaMalloc(&o, 148 * 512 * 4);
  cudaMalloc(&c, 148 * 8);
  bench<OP><<<148, 512>>>(o, c, 1.f);
  bench<OP><<<148, 512>>>(o, c, 1.f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  // 16 warps per CTA, 4 per SMSP
  const double per_smsp_instr = 4.0 * kIters * instr_per_iter_per_warp;
  printf("%-10s %6.2f cycles per warp-instruction per SMSP\n", name, avg / per_smsp_instr);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  run<0>("FFMA2", 4);
  run<1>("FADD2", 4);
  run<7>("FMUL2", 4);
  run<2>("FFMA", 8);
  run<3>("MUFU.EX2", 8);
  run<4>("F2FP", 4);
  run<5>("FMNMX3", 8);
  run<6>("SHL", 8);
  return 0;
}
