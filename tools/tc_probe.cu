// Standalone probe of the tcgen05 plumbing used by the tensor-core posterior (not part of the
// library): D[128 x N] (at TMEM column offset `coff`) = A[128 x 32] * B[N x 32]^T with 3xTF32,
// A written to SMEM by threads, B brought in by a bulk async copy completing an mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tools/tc_probe.cu && ./tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2603_11603_b200/csrc/tc_ptx.cuh"

using namespace as::tc;

constexpr int KC = 32;  // K extent of one chunk

__global__ void probe(const float* A, const float* Bhi_g, const float* Blo_g, int N, int coff, int ksteps_mask,
                      float* D, int mode) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* Ahi = reinterpret_cast<float*>(sm);
  float* Alo = Ahi + 128 * KC;
  float* Bhi = Alo + 128 * KC;
  float* Blo = Bhi + 256 * KC;
  __shared__ __align__(8) uint64_t bar_b, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar_b, 1);
    mbar_init(&bar_mma, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  // A: thread t owns row t
  for (int k = 0; k < KC; ++k) {
    float h, l;
    split_tf32(A[tid * KC + k], h, l);
    const uint32_t off = kmajor_off(tid, k, KC / 4) / 4;
    Ahi[off] = h;
    Alo[off] = l;
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t bytes = N * KC * 4;
    mbar_arrive_expect_tx(&bar_b, 2 * bytes);
    bulk_g2s(Bhi, Bhi_g, bytes, &bar_b);
    bulk_g2s(Blo, Blo_g, bytes, &bar_b);
    mbar_wait(&bar_b, 0);
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t sbo = (KC / 4) * 128;
    for (int s = 0; s < KC / 8; ++s) {
      if (!((ksteps_mask >> s) & 1)) continue;
      const uint64_t ah = sdesc(smem_u32(Ahi) + 256 * s, 128, sbo);
      const uint64_t al = sdesc(smem_u32(Alo) + 256 * s, 128, sbo);
      const uint64_t bh = sdesc(smem_u32(Bhi) + 256 * s, 128, sbo);
      const uint64_t bl = sdesc(smem_u32(Blo) + 256 * s, 128, sbo);
      const uint32_t acc = (s > 0 && (ksteps_mask & ((1 << s) - 1))) ? 1u : 0u;
      mma_tf32(tm + coff, ah, bh, idesc, acc);
      if (mode == 3) {
        mma_tf32(tm + coff, ah, bl, idesc, 1);
        mma_tf32(tm + coff, al, bh, idesc, 1);
      }
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  fence_after_sync();
  // each warp reads its 32 lanes (rows), N columns in chunks of 16
  const int row = (warp & 3) * 32 + lane;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + (static_cast<uint32_t>((warp & 3) * 32) << 16) + coff + c, v);
    for (int i = 0; i < 16; ++i) D[row * N + c + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

// A written into TMEM columns [acol, acol+32) by tcgen05.st (hi 0..15? no: hi at acol.., lo at acol+32..)
__global__ void probe_ts(const float* A, const float* Bhi_g, const float* Blo_g, int N, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* Bhi = reinterpret_cast<float*>(sm);
  float* Blo = Bhi + 256 * KC;
  __shared__ __align__(8) uint64_t bar_b, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar_b, 1);
    mbar_init(&bar_mma, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  const uint32_t acol = 256;  // A hi at columns [256, 288), lo at [288, 320)
  for (int k4 = 0; k4 < KC / 4; ++k4) {
    float h[4], l[4];
    for (int q = 0; q < 4; ++q) split_tf32(A[tid * KC + 4 * k4 + q], h[q], l[q]);
    const uint32_t lanebase = tm + (static_cast<uint32_t>(warp * 32) << 16);
    tmem_st4(lanebase + acol + 4 * k4, h[0], h[1], h[2], h[3]);
    tmem_st4(lanebase + acol + KC + 4 * k4, l[0], l[1], l[2], l[3]);
  }
  tmem_st_wait();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t bytes = N * KC * 4;
    mbar_arrive_expect_tx(&bar_b, 2 * bytes);
    bulk_g2s(Bhi, Bhi_g, bytes, &bar_b);
    bulk_g2s(Blo, Blo_g, bytes, &bar_b);
    mbar_wait(&bar_b, 0);
    const uint32_t idesc = idesc_tf32(128, N);
    const uint32_t sbo = (KC / 4) * 128;
    for (int s = 0; s < KC / 8; ++s) {
      const uint64_t bh = sdesc(smem_u32(Bhi) + 256 * s, 128, sbo);
      const uint64_t bl = sdesc(smem_u32(Blo) + 256 * s, 128, sbo);
      mma_tf32_ts(tm, tm + acol + 8 * s, bh, idesc, s > 0 ? 1u : 0u);
      mma_tf32_ts(tm, tm + acol + 8 * s, bl, idesc, 1u);
      mma_tf32_ts(tm, tm + acol + KC + 8 * s, bh, idesc, 1u);
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  fence_after_sync();
  const int row = warp * 32 + lane;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[row * N + c + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

static void split_host(float x, float& hi, float& lo) {
  // round-to-nearest-away to 10 mantissa bits (matches cvt.rna.tf32.f32 for finite values)
  uint32_t u;
  memcpy(&u, &x, 4);
  uint32_t h = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&hi, &h, 4);
  float r = x - hi;
  memcpy(&u, &r, 4);
  h = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&lo, &h, 4);
}

int main() {
  int fails = 0;
  for (int mode : {1, 3})
    for (int N : {64, 256, 144})
      for (int coff : {0, 64, 256}) {
        if (coff + N > 512) continue;
        std::vector<float> A(128 * KC), B(N * KC), Bhi(N * KC), Blo(N * KC), D(128 * N);
        srand(N * 7 + coff + mode);
        for (auto& x : A) x = (rand() / float(RAND_MAX) - 0.5f) * 2.0f;
        for (auto& x : B) x = (rand() / float(RAND_MAX) - 0.5f) * 30.0f;
        // B host-prepared in the K-major core-matrix layout
        for (int n = 0; n < N; ++n)
          for (int k = 0; k < KC; ++k) {
            float h, l;
            split_host(B[n * KC + k], h, l);
            const uint32_t off = kmajor_off(n, k, KC / 4) / 4;
            Bhi[off] = h;
            Blo[off] = l;
          }
        float *dA, *dBh, *dBl, *dD;
        cudaMalloc(&dA, A.size() * 4);
        cudaMalloc(&dBh, Bhi.size() * 4);
        cudaMalloc(&dBl, Blo.size() * 4);
        cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dBh, Bhi.data(), Bhi.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dBl, Blo.data(), Blo.size() * 4, cudaMemcpyHostToDevice);
        const size_t smem = (2 * 128 + 2 * 256) * KC * 4;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe<<<1, 128, smem>>>(dA, dBh, dBl, N, coff, 0xF, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("CUDA error %s\n", cudaGetErrorString(e));
          return 2;
        }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, maxabs = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < N; ++n) {
            double ref = 0, mag = 0;
            for (int k = 0; k < KC; ++k) {
              ref += double(A[m * KC + k]) * double(B[n * KC + k]);
              mag += fabs(double(A[m * KC + k]) * double(B[n * KC + k]));
            }
            const double err = fabs(D[m * N + n] - ref);
            maxabs = fmax(maxabs, err);
            maxrel = fmax(maxrel, err / mag);
          }
        const double bar = mode == 3 ? 1e-6 : 2e-3;
        const bool ok = maxrel < bar;
        fails += !ok;
        printf("mode %dxTF32 N=%3d coff=%3d  max|err|/sum|ab| = %.3e  %s\n", mode, N, coff, maxrel, ok ? "OK" : "FAIL");
        cudaFree(dA);
        cudaFree(dBh);
        cudaFree(dBl);
        cudaFree(dD);
      }
  // A-from-TMEM variant (3xTF32), N = 256 and 64
  for (int N : {64, 256}) {
    std::vector<float> A(128 * KC), B(N * KC), Bhi(N * KC), Blo(N * KC), D(128 * N);
    srand(N + 99);
    for (auto& x : A) x = (rand() / float(RAND_MAX) - 0.5f) * 2.0f;
    for (auto& x : B) x = (rand() / float(RAND_MAX) - 0.5f) * 30.0f;
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < KC; ++k) {
        float h, l;
        split_host(B[n * KC + k], h, l);
        const uint32_t off = kmajor_off(n, k, KC / 4) / 4;
        Bhi[off] = h;
        Blo[off] = l;
      }
    float *dA, *dBh, *dBl, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dBh, Bhi.size() * 4);
    cudaMalloc(&dBl, Blo.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBh, Bhi.data(), Bhi.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBl, Blo.data(), Blo.size() * 4, cudaMemcpyHostToDevice);
    const size_t smem = 2 * 256 * KC * 4;
    cudaFuncSetAttribute(probe_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_ts<<<1, 128, smem>>>(dA, dBh, dBl, N, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < KC; ++k) { ref += double(A[m * KC + k]) * B[n * KC + k]; mag += fabs(double(A[m * KC + k]) * B[n * KC + k]); }
        maxrel = fmax(maxrel, fabs(D[m * N + n] - ref) / mag);
      }
    const bool ok = maxrel < 1e-6;
    fails += !ok;
    printf("A-from-TMEM 3xTF32 N=%3d  max|err|/sum|ab| = %.3e  %s\n", N, maxrel, ok ? "OK" : "FAIL");
  }
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails ? 1 : 0;
}
