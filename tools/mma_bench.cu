// Microbenchmark (not part of the library): cycles per tcgen05.mma kind::f16 (M = 128, K = 16, SS)
// for N in {16, 32, 64, 128, 256}, issued back to back into one accumulator ("chain") or
// alternating between two ("2 acc"), and kind::tf32 with A from TMEM (the L^-1 k contraction).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_bench tools/mma_bench.cu && ./mma_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2603_11603_b200/csrc/tc_ptx.cuh"

using namespace as::tc;

__global__ void bench(int N, int nmma, int mode, long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3C003C00u;
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  if (warp == 0) {
    const uint32_t sA = smem_u32(sm), sB = sA + 32 * 1024;
    const uint64_t da = sdesc(sA, 128, 256), db = sdesc(sB, 128, 256);
    const uint32_t id16 = idesc_f16(128, N), id32 = idesc_tf32(128, N);
    long long t0 = clock64();
    for (int r = 0; r < 2; ++r) {   // r = 0 warm-up
      if (r == 1) t0 = clock64();
      if (mode == 0) {
        for (int i = 0; i < nmma; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_f16_w(tm, da + 16 * u, db + 16 * u, id16, 1u);
        }
      } else if (mode == 1) {
        for (int i = 0; i < nmma; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_f16_w(tm + (u & 1) * 256, da + 16 * u, db + 16 * u, id16, 1u);
        }
      } else {
        for (int i = 0; i < nmma; i += 8) {
#pragma unroll
          for (int u = 0; u < 8; ++u) mma_tf32_ts_w(tm, tm + 256 + 8 * u, db + 16 * u, id32, 1u);
        }
      }
      mma_commit_w(&bar);
      mbar_wait(&bar, r);
    }
    const long long t1 = clock64();
    if (tid == 0) *out = t1 - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char* names[3] = {"f16 SS chain ", "f16 SS 2 acc ", "tf32 TS chain"};
  for (int mode = 0; mode < 3; ++mode)
    for (int N : {16, 32, 64, 128, 256}) {
      if (mode == 1 && N > 256) continue;
      for (int nmma : {8, 64, 256}) {
        bench<<<1, 128, 64 * 1024>>>(N, nmma, mode, d);
        long long h = 0;
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("CUDA error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%s N=%3d nmma=%3d  cycles %7lld  per MMA %.1f\n", names[mode], N, nmma, h, double(h) / nmma);
      }
    }
  return 0;
}
