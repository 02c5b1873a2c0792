// GP hyper-parameter evidence, batched (R21): the log marginal
// likelihood of the observed residuals r = y - m0 - b under N(0, K_h), K_h = k_h(x_i, x_j) + sn2_h I,
// for many hyper-parameter settings h in one launch (ML-II search).  One CTA per setting (grid-
// stride), FP64 throughout: K_h is built in a per-CTA L2-resident work matrix, factorised by a
// right-looking Cholesky (column q final -> rank-1 update of the trailing lower triangle, one warp
// per row, lanes over columns: coalesced), with the forward solve z = L^-1 r fused into the same
// column steps; lml = -1/2 z.z - sum_q ln L_qq - M/2 ln(2 pi).  Not positive definite -> -INF.
#pragma once
#include "common.cuh"

namespace as {

constexpr int LML_THREADS = 256;

__global__ void __launch_bounds__(LML_THREADS)
lml_kernel(const double* __restrict__ phi, const double* __restrict__ r, int M, int d, int kind,
           const double* __restrict__ hyp, int n_set, double* __restrict__ work, double* __restrict__ out) {
  extern __shared__ double lml_sm[];                   // [M] column q, [M] z / r, [d] 1/l^2
  double* colq = lml_sm;
  double* z = colq + M;
  double* il2 = z + M;
  __shared__ double s_logdet;
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = LML_THREADS / 32;
  double* A = work + static_cast<size_t>(blockIdx.x) * M * M;
  for (int h = blockIdx.x; h < n_set; h += gridDim.x) {
    const double* hp = hyp + static_cast<size_t>(h) * (d + 2);
    const double sf2 = hp[d], sn2 = hp[d + 1];
    for (int j = tid; j < d; j += LML_THREADS) il2[j] = 1.0 / (hp[j] * hp[j]);
    for (int i = tid; i < M; i += LML_THREADS) z[i] = r[i];
    if (tid == 0) {
      s_logdet = 0.0;
      s_fail = 0;
    }
    __syncthreads();
    // K (lower triangle, row-major M x M)
    for (int i = warp; i < M; i += nw)
      for (int j = lane; j <= i; j += 32) {
        double r2 = 0.0;
        for (int q = 0; q < d; ++q) {
          const double df = phi[i * d + q] - phi[j * d + q];
          r2 += df * df * il2[q];
        }
        A[static_cast<size_t>(i) * M + j] = kernel64(kind, sf2, r2) + (i == j ? sn2 : 0.0);
      }
    __syncthreads();
    for (int q = 0; q < M; ++q) {
      if (tid == 0) {
        const double dq = A[static_cast<size_t>(q) * M + q];
        if (!(dq > 0.0)) s_fail = 1;
        const double lqq = dq > 0.0 ? sqrt(dq) : 1.0;
        colq[q] = lqq;
        s_logdet += log(lqq);
        z[q] = z[q] / lqq;
      }
      __syncthreads();
      const double lqq = colq[q], zq = z[q];
      for (int i = q + 1 + tid; i < M; i += LML_THREADS) {
        const double liq = A[static_cast<size_t>(i) * M + q] / lqq;
        colq[i] = liq;
        z[i] -= liq * zq;                               // fused forward solve
      }
      __syncthreads();
      for (int i = q + 1 + warp; i < M; i += nw) {     // trailing update, one warp per row
        const double liq = colq[i];
        double* ai = A + static_cast<size_t>(i) * M;
        for (int j = q + 1 + lane; j <= i; j += 32) ai[j] -= liq * colq[j];
      }
      __syncthreads();
    }
    // 1/2 z.z (block reduction)
    double part = 0.0;
    for (int i = tid; i < M; i += LML_THREADS) part += z[i] * z[i];
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __shared__ double red[LML_THREADS / 32];
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (tid == 0) {
      double zz = 0.0;
      for (int w = 0; w < nw; ++w) zz += red[w];
      out[h] = s_fail ? -INFINITY : -0.5 * zz - s_logdet - 0.5 * M * 1.8378770664093454836;   // ln(2 pi)
    }
    __syncthreads();
  }
}

}  // namespace as
