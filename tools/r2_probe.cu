// Standalone probe (not part of the library) of the one-hot squared-distance contraction:
//   R2[m][j] = sum_k E[m][k] * T[j][k],  E = one-hot digit encoding of candidate m (BF16, exact),
//   T[j][(f,v)] = (xt_f[v] - xt_f[d_jf])^2 split into three BF16 pieces (hi + mid + lo),
// as tcgen05.mma kind::f16 (M = 128, N = 16 / 32 / 64, K = 16 per instruction) with E written to SMEM by
// threads and T brought in by a bulk async copy.  Reports max |R2 - r2_exact| / r2_exact.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o r2_probe tools/r2_probe.cu && ./r2_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2603_11603_b200/csrc/tc_ptx.cuh"

using namespace as::tc;

static uint16_t bf16_rn(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t r = u + 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(r >> 16);
}
#include <cuda_fp16.h>
static uint16_t f16_rn(double x) {
  __half h = __double2half(x);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}
static double f16_val(uint16_t u) {
  __half h;
  memcpy(&h, &u, 2);
  return static_cast<double>(__half2float(h));
}
static double bf16_val(uint16_t h) {
  uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

__global__ void probe(const uint16_t* ecols, int nfeat, const uint16_t* T_g, int N, int Kp, int np, int f16, float* D) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* E = sm;                                   // 128 x Kp bf16
  unsigned char* T = sm + 128 * Kp * 2;                    // 3 x N x Kp bf16
  __shared__ __align__(8) uint64_t bar_b, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bar_b, 1);
    mbar_init(&bar_mma, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 512);
  const uint32_t kcore = Kp / 8;
  for (int k = 0; k < Kp; k += 8)
    *reinterpret_cast<uint4*>(E + kmajor_off16(tid, k, kcore)) = make_uint4(0, 0, 0, 0);
  for (int f = 0; f < nfeat; ++f) {
    const int k = ecols[tid * nfeat + f];
    *reinterpret_cast<uint16_t*>(E + kmajor_off16(tid, k, kcore)) = f16 ? 0x3C00 : 0x3F80;   // 1.0
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t bytes = np * N * Kp * 2;
    mbar_arrive_expect_tx(&bar_b, bytes);
    bulk_g2s(T, T_g, bytes, &bar_b);
    mbar_wait(&bar_b, 0);
    const uint32_t idesc = f16 ? idesc_f16(128, N) : idesc_bf16(128, N);
    const uint32_t sbo = kcore * 128;
    const uint32_t piece = N * Kp * 2;
    for (int s = 0; s < Kp / 16; ++s) {
      const uint64_t ad = sdesc(smem_u32(E) + 256 * s, 128, sbo);
      for (int p = 0; p < np; ++p) {
        const uint64_t bd = sdesc(smem_u32(T) + p * piece + 256 * s, 128, sbo);
        mma_f16(tm, ad, bd, idesc, (s | p) ? 1u : 0u);
      }
    }
    mma_commit(&bar_mma);
  }
  __syncwarp();
  mbar_wait(&bar_mma, 0);
  fence_after_sync();
  const int row = (warp & 3) * 32 + lane;
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tm + (static_cast<uint32_t>((warp & 3) * 32) << 16) + c, v);
    for (int i = 0; i < 16; ++i) D[row * N + c + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

int main() {
  const int nf[16] = {7, 4, 4, 9, 4, 4, 3, 4, 2, 2, 33, 2, 2, 2, 64, 9};   // C4 feature cardinalities
  const int nfeat = 16;
  int off[17];
  off[0] = 0;
  for (int f = 0; f < nfeat; ++f) off[f + 1] = off[f] + nf[f];
  const int K = off[nfeat], Kp = (K + 15) / 16 * 16;
  int fails = 0;
  for (int cfg = 0; cfg < 6; ++cfg) {
    const int N = (cfg % 3 == 0) ? 16 : (cfg % 3 == 1 ? 32 : 64);
    const int f16 = cfg >= 3, np = f16 ? 2 : 3;
    srand(N);
    std::vector<std::vector<double>> xt(nfeat);
    for (int f = 0; f < nfeat; ++f)
      for (int v = 0; v < nf[f]; ++v) xt[f].push_back(2.0 * rand() / RAND_MAX);
    std::vector<int> dm(128 * nfeat), dj(N * nfeat);
    for (int m = 0; m < 128; ++m)
      for (int f = 0; f < nfeat; ++f) dm[m * nfeat + f] = rand() % nf[f];
    for (int j = 0; j < N; ++j)
      for (int f = 0; f < nfeat; ++f) dj[j * nfeat + f] = (j < 4) ? dm[j * nfeat + f] : rand() % nf[f];
    // a few candidates differ from observed point 4 in one digit only (small r^2)
    for (int m = 8; m < 12; ++m) {
      for (int f = 0; f < nfeat; ++f) dm[m * nfeat + f] = dj[4 * nfeat + f];
      dm[m * nfeat + 14] = (dm[m * nfeat + 14] + 1) % nf[14];
    }
    std::vector<uint16_t> ecols(128 * nfeat), Tg(3 * N * Kp, 0);
    double tmax = 0;
    for (int f = 0; f < nfeat; ++f)
      for (double a : xt[f])
        for (double b : xt[f]) tmax = fmax(tmax, (a - b) * (a - b));
    int sc = 0;   // fp16: scale by 2^sc (sc even) so the largest entry lies in [2^13, 2^15]
    if (f16) while (tmax * std::ldexp(1.0, sc + 2) <= 32768.0) sc += 2;
    for (int m = 0; m < 128; ++m)
      for (int f = 0; f < nfeat; ++f) ecols[m * nfeat + f] = off[f] + dm[m * nfeat + f];
    const uint32_t piece = N * Kp;   // elements
    for (int j = 0; j < N; ++j)
      for (int f = 0; f < nfeat; ++f)
        for (int v = 0; v < nf[f]; ++v) {
          const double d = xt[f][v] - xt[f][dj[j * nfeat + f]];
          const double t = d * d;
          const uint32_t o = kmajor_off16(j, off[f] + v, Kp / 8) / 2;
          if (f16) {
            const double ts = std::ldexp(t, sc);
            const uint16_t h = f16_rn(ts);
            Tg[o] = h;
            Tg[piece + o] = f16_rn(ts - f16_val(h));
            continue;
          }
          const uint16_t h = bf16_rn(static_cast<float>(t));
          const double r1 = t - bf16_val(h);
          const uint16_t md = bf16_rn(static_cast<float>(r1));
          const uint16_t lo = bf16_rn(static_cast<float>(r1 - bf16_val(md)));
          Tg[o] = h;
          Tg[piece + o] = md;
          Tg[2 * piece + o] = lo;
        }
    uint16_t *dE, *dT;
    float* dD;
    cudaMalloc(&dE, ecols.size() * 2);
    cudaMalloc(&dT, Tg.size() * 2);
    cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dE, ecols.data(), ecols.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dT, Tg.data(), Tg.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = 128 * Kp * 2 + np * N * Kp * 2;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<<<1, 128, smem>>>(dE, nfeat, dT, N, Kp, np, f16, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 2;
    }
    std::vector<float> D(128 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxrel = 0, maxabs0 = 0;
    int nzero = 0;
    for (int m = 0; m < 128; ++m)
      for (int j = 0; j < N; ++j) {
        double r2 = 0;
        for (int f = 0; f < nfeat; ++f) {
          const double d = xt[f][dm[m * nfeat + f]] - xt[f][dj[j * nfeat + f]];
          r2 += d * d;
        }
        if (r2 == 0) {
          ++nzero;
          maxabs0 = fmax(maxabs0, fabs(D[m * N + j]));
        } else {
          maxrel = fmax(maxrel, fabs(std::ldexp(static_cast<double>(D[m * N + j]), -sc) - r2) / r2);
        }
      }
    const bool ok = maxrel < 4e-6 && maxabs0 == 0;
    fails += !ok;
    printf("one-hot R2 %s K=%d N=%2d  max rel err %.3e (%.1f ulp32)  exact zeros %d (max |R2| %.1e)  %s\n", f16 ? "f16x2 " : "bf16x3", Kp, N,
           maxrel, maxrel / 5.96e-8, nzero, maxabs0, ok ? "OK" : "FAIL");
    cudaFree(dE);
    cudaFree(dT);
    cudaFree(dD);
  }
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails ? 1 : 0;
}
