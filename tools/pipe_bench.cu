// Per-SMSP issue rates of the instructions in the score kernel's chunk loop (development aid):
// 1 CTA per SM, W warps, each warp runs a loop of independent chains of one instruction kind;
// prints cycles per warp-instruction per SM sub-partition.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sqrtap(float x) {
  float r;
  asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

constexpr int CH = 8, IT = 4096;

template <int K>
__global__ void bench(float* out, long long* cyc) {
  unsigned long long a[CH];
  float f[CH];
  uint32_t u[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = 0x3f8000003f800000ull + threadIdx.x + i;
    f[i] = 1.0f + 1e-3f * (threadIdx.x + i);
    u[i] = threadIdx.x * 7 + i;
  }
  const unsigned long long m = 0x3f8000013f800001ull, c = 0x3a0000003a000000ull;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (K == 0) a[i] = ffma2(a[i], m, c);
      if (K == 1) a[i] = fmul2(a[i], m);
      if (K == 2) f[i] = fmaf(f[i], 1.0001f, f[(i + 1) % CH]);
      if (K == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u[i]) : "r"(u[(i + 1) % CH]), "r"(u[(i + 3) % CH]));
      if (K == 4) f[i] = ex2(f[i]);
      if (K == 5) f[i] = sqrtap(f[i]);
      if (K == 6) {  // chunk-loop mix: 4 FFMA2 per MUFU
        a[i] = ffma2(a[i], m, c);
        a[i] = ffma2(a[i], m, c);
        a[i] = ffma2(a[i], m, c);
        a[i] = ffma2(a[i], m, c);
        f[i] = ex2(f[i]);
      }
      if (K == 7) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[i]) : "r"(u[(i + 1) % CH]), "r"(u[(i + 3) % CH]));
      if (K == 8) f[i] = f[i] + f[(i + 1) % CH];
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += __uint_as_float(static_cast<uint32_t>(a[i])) + f[i] + u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int K>
void run(const char* name, int warps, int per_iter_instr) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  bench<K><<<148, warps * 32>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const double instr_per_smsp = static_cast<double>(IT) * CH * per_iter_instr * warps / 4.0;
  printf("%-14s warps %2d  cycles/warp-instr/SMSP %.3f\n", name, warps, h[0] / instr_per_smsp);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("FFMA2", w, 1);
    run<1>("FMUL2", w, 1);
    run<2>("FFMA", w, 1);
    run<3>("IMAD", w, 1);
    run<4>("MUFU.EX2", w, 1);
    run<5>("MUFU.SQRT", w, 1);
    run<6>("4FFMA2+EX2", w, 5);
    run<7>("LOP3", w, 1);
    run<8>("FADD", w, 1);
  }
  return 0;
}
