// Standalone probe (not part of the library): kind::f16 MMA with A from TMEM (packed f16x2
// columns written by tcgen05.st) and B from SMEM, 3-term FP16 split (hi.hi + hi.lo + lo.hi) of
// FP32 data with power-of-two scaling -- the layout and accuracy of the L^-1 k contraction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o f16ts_probe tools/f16ts_probe.cu && ./f16ts_probe
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2603_11603_b200/csrc/tc_ptx.cuh"

using namespace as::tc;
constexpr int KC = 32;   // K extent (2 MMA k-steps)

__global__ void probe(const float* A, float sa, const uint16_t* Bhi_g, const uint16_t* Blo_g, int N, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* Bhi = sm;
  unsigned char* Blo = sm + 256 * KC * 2;
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
  const uint32_t acol = 256;   // A hi at [256, 256 + KC/2), lo at [256 + KC/2, 256 + KC)
  const uint32_t lb = tm + (static_cast<uint32_t>(warp * 32) << 16);
  for (int k4 = 0; k4 < KC / 4; ++k4) {
    float x[4], h[4];
    uint32_t hp[2], lp[2];
    for (int q = 0; q < 4; ++q) x[q] = A[tid * KC + 4 * k4 + q] * sa;
    for (int q = 0; q < 2; ++q) {
      hp[q] = pack_f16x2(x[2 * q], x[2 * q + 1]);
      unpack_f16x2(hp[q], h[2 * q], h[2 * q + 1]);
      lp[q] = pack_f16x2(x[2 * q] - h[2 * q], x[2 * q + 1] - h[2 * q + 1]);
    }
    tmem_st2(lb + acol + 2 * k4, hp[0], hp[1]);
    tmem_st2(lb + acol + KC / 2 + 2 * k4, lp[0], lp[1]);
  }
  tmem_st_wait();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  if (tid == 0) {
    const uint32_t bytes = N * KC * 2;
    mbar_arrive_expect_tx(&bar_b, 2 * bytes);
    bulk_g2s(Bhi, Bhi_g, bytes, &bar_b);
    bulk_g2s(Blo, Blo_g, bytes, &bar_b);
    mbar_wait(&bar_b, 0);
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t idesc = idesc_f16(128, N);
    const uint32_t sbo = (KC / 8) * 128;
    for (int s = 0; s < KC / 16; ++s) {
      const uint64_t bh = sdesc(smem_u32(Bhi) + 256 * s, 128, sbo), bl = sdesc(smem_u32(Blo) + 256 * s, 128, sbo);
      mma_f16_ts_w(tm, tm + acol + 8 * s, bh, idesc, s > 0 ? 1u : 0u);
      mma_f16_ts_w(tm, tm + acol + 8 * s, bl, idesc, 1u);
      mma_f16_ts_w(tm, tm + acol + KC / 2 + 8 * s, bh, idesc, 1u);
    }
    mma_commit_w(&bar_mma);
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

static uint16_t h16(double x) {
  __half h = __double2half(x);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static double v16(uint16_t u) {
  __half h;
  memcpy(&h, &u, 2);
  return __half2float(h);
}

int main() {
  int fails = 0;
  for (int N : {16, 64, 256}) {
    std::vector<float> A(128 * KC);
    std::vector<double> B(N * KC);
    srand(N);
    for (auto& x : A) x = 0.1f * std::exp(-10.0 * rand() / RAND_MAX);   // k-like: (0, 0.1]
    for (auto& x : B) x = (rand() / double(RAND_MAX) - 0.5) * 60.0 * std::exp(-5.0 * rand() / RAND_MAX);
    double amax = 0.1, bmax = 0;
    for (double x : B) bmax = fmax(bmax, fabs(x));
    const int ea = (int)floor(log2(32768.0 / amax)), eb = (int)floor(log2(32768.0 / bmax));
    const float sa = std::ldexp(1.0f, ea);
    std::vector<uint16_t> Bh(N * KC), Bl(N * KC);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < KC; ++k) {
        const double x = std::ldexp(B[n * KC + k], eb);
        const uint16_t hi = h16(x);
        const uint32_t o = kmajor_off16(n, k, KC / 8) / 2;
        Bh[o] = hi;
        Bl[o] = h16(x - v16(hi));
      }
    float *dA, *dD;
    uint16_t *dBh, *dBl;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dBh, Bh.size() * 2);
    cudaMalloc(&dBl, Bl.size() * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dBh, Bh.data(), Bh.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dBl, Bl.data(), Bl.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = 2 * 256 * KC * 2;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<1, 128, smem>>>(dA, sa, dBh, dBl, N, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 2;
    }
    std::vector<float> D(128 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0, mag = 0;
        for (int k = 0; k < KC; ++k) {
          ref += double(A[m * KC + k]) * B[n * KC + k];
          mag += fabs(double(A[m * KC + k]) * B[n * KC + k]);
        }
        const double got = std::ldexp(double(D[m * N + n]), -(ea + eb));
        maxrel = fmax(maxrel, fabs(got - ref) / mag);
      }
    const bool ok = maxrel < 1e-6;
    fails += !ok;
    printf("f16 TS 3-term N=%3d  max|err|/sum|ab| = %.3e  %s\n", N, maxrel, ok ? "OK" : "FAIL");
  }
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails ? 1 : 0;
}
