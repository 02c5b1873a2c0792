// sm_100a kernels of the scoring path.
//   score_kernel   persistent; candidates generated from indices in registers; decode + mask +
//                  simulator (FP64) -> SMEM queue of valid candidates -> GP batches of 32:
//                  cross-covariance (SIMT FP32) -> posterior  v = L^-1 k  (register-blocked SIMT
//                  over 4x4 W blocks in SMEM) -> FP64 acquisition + error bound -> CTA top-k'
//   merge_kernel   one CTA: CTA lists + running pool -> running pool (top k'), drop bound
//   refine_kernel  one CTA per pool entry: exact FP64 re-score (same formulas, FP64 GP)
//   mask_kernel    validity bit per raw index (parity path)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace as {

constexpr int SCORE_THREADS = 256;
constexpr int QCAP = 288;                // 31 leftover + 256 new valid candidates per tile
constexpr uint64_t KEY_NONE = ~0ull;
constexpr float U32 = 5.9604644775390625e-08f;  // 2^-24 (unit roundoff, FP32)

struct DevSpace {
  int d, n_prefix, n_comp, n_struct;
  uint64_t n_cvi, n_raw, tail_span;
  const uint64_t* prefix;  // [n_struct+1]
  const uint32_t* bucket;  // [n_bucket+1]: structure of position b << bshift (SMEM-resident decode, gen kernel)
  int n_bucket, bshift;
  const uint64_t* s_raw;   // [n_struct]
  const uint32_t* s_act;   // [n_struct]
  const DV* s_dv;          // [n_struct]
  const uint4* s_oc;       // [n_struct*n_comp] (offset, count, magic, sh1 | sh2 << 8): t / count by multiply
  const Tuple* tuples;
  const double* val;       // [d*VMAX]
  const double* inv;       // [d*VMAX] 1/val   (simulator cost terms)
  const double* lg2;       // [d*VMAX] log2(val)
  const float* xt32;       // [d*VMAX]
  const double* xt64;      // [d*VMAX]
  uint64_t stride[DMAX];
  int nval[DMAX];
  int comp_first[DMAX];
  int comp_width[DMAX];
  SimParams sim;
  // GP prior mean (R9 / R20): ln cost_sim, or the regression-simulator ensemble (NEXT-1)
  int ens_on;
  double ens_c0;
  const double* ens_tab;   // [d * VMAX]
  // derived-mode partial evaluation per structure (gen kernel fast path; srec == nullptr: off)
  const SimRec* srec;      // [n_struct]
  SimFast sf;
};

// out of line: keeps the ensemble loop out of the register allocation of the hot kernels
__device__ __noinline__ double ensemble_m0_dev(const double* tab, double c0, int d, uint64_t w0, uint64_t w1,
                                               uint64_t w2) {
  DV dv;
  dv.w[0] = w0;
  dv.w[1] = w1;
  dv.w[2] = w2;
  double m = c0;
  for (int f = 0; f < d; ++f) m += __ldg(tab + f * VMAX + dv_get(dv, f));
  return m;
}
__device__ __forceinline__ double prior_m0(const DevSpace& S, const DV& dv, double cost) {
  if (!S.ens_on) return log(cost);
  return ensemble_m0_dev(S.ens_tab, S.ens_c0, S.d, dv.w[0], dv.w[1], dv.w[2]);
}

struct DevGP {
  int M, Mp, DP, kernel;   // Mp: M padded to 4; DP: d padded to 4
  float sf2f;
  double sf2, b, fstar;
  double eps;              // (d + 8 + M) * 2^-24   : relative error coefficient of the FP32 screen
  double w_fro;            // ||L^-1||_F
  const float* O;          // [Mp][DP]
  const float* alpha;      // [Mp]
  const float* aabs;       // [Mp]
  const float* Wblk;       // 4x4 blocks of L^-1, lower block-triangle, block (q,a) at (q(q+1)/2+a)*16, [b][r]
  const double* O64;       // [M][d]
  const double* alpha64;   // [M]
  const double* W64;       // [M][M] row-major
};

struct BatchArgs {
  int mode, acq;
  uint64_t begin, count;
  FeistelKey fk;
  double kappa, xi;
  float* d_scores;
  uint64_t* d_raw;
  uint64_t* d_valid_count;
  const uint64_t* list;   // LIST mode: CVI positions (entries >= n_cvi are masked)
  uint64_t n_cvi;
  float* d_screen;        // nullable [4 count]: mu, s2, screen, upper bound of the FP32 screen
};

// a0: candidate j of the batch -> CVI position.  A LIST entry outside [0, n_cvi) is
// replaced by position 0 and reported through `in` = false: the caller decodes unconditionally
// (keeps the hot RANGE / SAMPLE code straight-line) and scores the candidate as masked.
__device__ __forceinline__ uint64_t assign_pos(const BatchArgs& A, uint64_t j, bool& in) {
  in = true;
  if (A.mode == 2) {
    const uint64_t p = __ldg(A.list + A.begin + j);
    in = p < A.n_cvi;
    return in ? p : 0;
  }
  return (A.mode == 0) ? A.begin + j : feistel_pi(A.fk, A.begin + j);
}

struct CtaOut {
  uint64_t* lists;     // [grid][KC]
  int* counts;         // [grid]
  uint64_t* drop;      // [grid] best (smallest) key that the CTA did not keep
  uint64_t* valid;     // total valid counter
  int KC;
  int P;               // pow2 >= KC + SCORE_THREADS
};

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ uint32_t f32_order(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// ascending key = better: (score desc, cvi asc); cvi order = raw order (R11)
__device__ __forceinline__ uint64_t make_key(float score_ub, uint32_t cvi) {
  return (static_cast<uint64_t>(~f32_order(score_ub)) << 32) | cvi;
}

__device__ __forceinline__ void decode_dev(const DevSpace& S, uint64_t p, DV& dv, uint32_t& act, uint64_t& raw) {
  int lo = 0, hi = S.n_struct;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(S.prefix + mid) <= p) lo = mid; else hi = mid;
  }
  uint32_t t = static_cast<uint32_t>(p - __ldg(S.prefix + lo));
  const DV* sd = S.s_dv + lo;
  dv.w[0] = __ldg(&sd->w[0]);
  dv.w[1] = __ldg(&sd->w[1]);
  dv.w[2] = __ldg(&sd->w[2]);
  act = __ldg(S.s_act + lo);
  raw = __ldg(S.s_raw + lo);
  for (int c = S.n_comp - 1; c >= 0; --c) {
    const uint4 oc = __ldg(S.s_oc + static_cast<size_t>(lo) * S.n_comp + c);
    const uint32_t hi = __umulhi(oc.z, t);
    const uint32_t q = (hi + ((t - hi) >> (oc.w & 0xFFu))) >> (oc.w >> 8);
    const uint32_t r = t - q * oc.y;
    t = q;
    const Tuple* tu = S.tuples + oc.x + r;
    dv.w[0] |= __ldg(&tu->dv.w[0]);
    dv.w[1] |= __ldg(&tu->dv.w[1]);
    dv.w[2] |= __ldg(&tu->dv.w[2]);
    act |= __ldg(&tu->act);
    raw += __ldg(&tu->raw);
  }
}

// Tail of the CVI decode: structure record, then one mixed-radix digit (multiply-shift division)
// and one tuple per gating group, OR-ed into the digit vector.  (Issuing every group's loads ahead
// of use was tried: with the unrolled register footprint the 3-block generation kernel spills and
// the 2-block one loses latency hiding -- 5.56 -> 7.40 / 6.94 ms on C4.)
__device__ __forceinline__ void decode_tail(const DevSpace& S, int lo, uint32_t t, DV& dv, uint32_t& act, uint64_t& raw) {
  const DV* sd = S.s_dv + lo;
  dv.w[0] = __ldg(&sd->w[0]);
  dv.w[1] = __ldg(&sd->w[1]);
  dv.w[2] = __ldg(&sd->w[2]);
  act = __ldg(S.s_act + lo);
  raw = __ldg(S.s_raw + lo);
  for (int c = S.n_comp - 1; c >= 0; --c) {
    const uint4 oc = __ldg(S.s_oc + static_cast<size_t>(lo) * S.n_comp + c);
    const uint32_t hi = __umulhi(oc.z, t);
    const uint32_t q = (hi + ((t - hi) >> (oc.w & 0xFFu))) >> (oc.w >> 8);
    const uint32_t r = t - q * oc.y;
    t = q;
    const Tuple* tu = S.tuples + oc.x + r;
    dv.w[0] |= __ldg(&tu->dv.w[0]);
    dv.w[1] |= __ldg(&tu->dv.w[1]);
    dv.w[2] |= __ldg(&tu->dv.w[2]);
    act |= __ldg(&tu->act);
    raw += __ldg(&tu->raw);
  }
}

// Decode with a coarse SMEM index of the structure prefix array: cidx[k] = prefix[k * n_struct / ci_n]
// (k < ci_n) brackets the structure before a short binary search in global memory; with
// ci_n == n_struct the whole search runs in shared memory.
constexpr int CI = 256;
__device__ __forceinline__ void decode_dev_ci(const DevSpace& S, const uint64_t* cidx, int ci_n, uint64_t p, DV& dv,
                                              uint32_t& act, uint64_t& raw, int* sidx = nullptr) {
  int a = 0, b = ci_n;                       // largest k with cidx[k] <= p
  while (b - a > 1) {
    const int mid = (a + b) >> 1;
    if (cidx[mid] <= p) a = mid; else b = mid;
  }
  int lo = static_cast<int>((static_cast<long long>(a) * S.n_struct) / ci_n);
  int hi = (b >= ci_n) ? S.n_struct : static_cast<int>((static_cast<long long>(b) * S.n_struct) / ci_n);
  if (hi <= lo) hi = lo + 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(S.prefix + mid) <= p) lo = mid; else hi = mid;
  }
  if (sidx) *sidx = lo;
  decode_tail(S, lo, static_cast<uint32_t>(p - __ldg(S.prefix + lo)), dv, act, raw);
}
// Structure lookup from SMEM copies of the whole prefix table and of the bucket index: the
// position's bucket brackets its structure, then a short binary search (typically 0-2 probes).
__device__ __forceinline__ void decode_dev_bucket(const DevSpace& S, const uint64_t* pre, const uint32_t* bkt,
                                                  uint64_t p, DV& dv, uint32_t& act, uint64_t& raw, int* sidx = nullptr) {
  const int b = static_cast<int>(p >> S.bshift);
  int lo = static_cast<int>(bkt[b]), hi = static_cast<int>(bkt[b + 1]) + 1;
  if (hi > S.n_struct) hi = S.n_struct;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= p) lo = mid; else hi = mid;
  }
  if (sidx) *sidx = lo;
  decode_tail(S, lo, static_cast<uint32_t>(p - pre[lo]), dv, act, raw);
}
// Generation kernel variant with a compile-time component count NC: the (offset, count, magic,
// shift) records of all NC tail groups are loaded as soon as the structure is known, so the
// mixed-radix chain and the tuple loads no longer wait for one record load per group in turn.
template <int NC>
__device__ __forceinline__ void decode_tail_nc(const DevSpace& S, int lo, uint32_t t, DV& dv, uint32_t& act, uint64_t& raw) {
  if (NC == 0) {
    decode_tail(S, lo, t, dv, act, raw);
    return;
  }
  uint4 oc[NC > 0 ? NC : 1];
  const uint4* ob = S.s_oc + static_cast<size_t>(lo) * (NC > 0 ? NC : 1);
#pragma unroll
  for (int c = 0; c < NC; ++c) oc[c] = __ldg(ob + c);
  const DV* sd = S.s_dv + lo;
  dv.w[0] = __ldg(&sd->w[0]);
  dv.w[1] = __ldg(&sd->w[1]);
  dv.w[2] = __ldg(&sd->w[2]);
  act = __ldg(S.s_act + lo);
  raw = __ldg(S.s_raw + lo);
#pragma unroll
  for (int c = NC - 1; c >= 0; --c) {
    const uint32_t hi = __umulhi(oc[c].z, t);
    const uint32_t q = (hi + ((t - hi) >> (oc[c].w & 0xFFu))) >> (oc[c].w >> 8);
    const uint32_t r = t - q * oc[c].y;
    t = q;
    const Tuple* tu = S.tuples + oc[c].x + r;
    dv.w[0] |= __ldg(&tu->dv.w[0]);
    dv.w[1] |= __ldg(&tu->dv.w[1]);
    dv.w[2] |= __ldg(&tu->dv.w[2]);
    act |= __ldg(&tu->act);
    raw += __ldg(&tu->raw);
  }
}
// structure of CVI position p from the SMEM prefix table + bucket index
__device__ __forceinline__ int find_struct_bucket(const DevSpace& S, const uint64_t* pre, const uint32_t* bkt, uint64_t p) {
  const int b = static_cast<int>(p >> S.bshift);
  int lo = static_cast<int>(bkt[b]), hi = static_cast<int>(bkt[b + 1]) + 1;
  if (hi > S.n_struct) hi = S.n_struct;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}
template <int NC>
__device__ __forceinline__ void decode_dev_bucket_nc(const DevSpace& S, const uint64_t* pre, const uint32_t* bkt,
                                                     uint64_t p, DV& dv, uint32_t& act, uint64_t& raw, int* sidx) {
  const int b = static_cast<int>(p >> S.bshift);
  int lo = static_cast<int>(bkt[b]), hi = static_cast<int>(bkt[b + 1]) + 1;
  if (hi > S.n_struct) hi = S.n_struct;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pre[mid] <= p) lo = mid; else hi = mid;
  }
  *sidx = lo;
  decode_tail_nc<NC>(S, lo, static_cast<uint32_t>(p - pre[lo]), dv, act, raw);
}
__device__ __forceinline__ void decode_dev_idx(const DevSpace& S, const uint64_t* cidx, uint64_t p, DV& dv,
                                               uint32_t& act, uint64_t& raw) {
  decode_dev_ci(S, cidx, S.n_struct < CI ? S.n_struct : CI, p, dv, act, raw);
}
__device__ __forceinline__ void load_cidx_n(const DevSpace& S, uint64_t* cidx, int ci_n, int tid, int nthreads) {
  for (int k = tid; k < ci_n; k += nthreads)
    cidx[k] = __ldg(S.prefix + static_cast<int>((static_cast<long long>(k) * S.n_struct) / ci_n));
}
__device__ __forceinline__ void load_cidx(const DevSpace& S, uint64_t* cidx, int tid, int nthreads) {
  load_cidx_n(S, cidx, S.n_struct < CI ? S.n_struct : CI, tid, nthreads);
}

// Packed FP32x2 helpers (FFMA2 / FADD2 on sm_100a): r^2 = sum_f (x_f - o_f)^2 two features at a time.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 f2_unpack(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// r^2 between packed candidate features xp[DMAX/2] and an observed row o (DP floats, 16-byte aligned)
__device__ __forceinline__ float r2_packed(const unsigned long long* xp, const float* o, int DP) {
  unsigned long long acc0 = 0ull, acc1 = 0ull;
  const ulonglong2* o2 = reinterpret_cast<const ulonglong2*>(o);
#pragma unroll
  for (int f4 = 0; f4 < DMAX / 4; ++f4) {
    if (4 * f4 < DP) {
      const ulonglong2 ov = o2[f4];
      const unsigned long long d0 = f2_sub(xp[2 * f4], ov.x);
      const unsigned long long d1 = f2_sub(xp[2 * f4 + 1], ov.y);
      acc0 = f2_fma(d0, d0, acc0);
      acc1 = f2_fma(d1, d1, acc1);
    }
  }
  const float2 a = f2_unpack(acc0), b = f2_unpack(acc1);
  return (a.x + b.x) + (a.y + b.y);
}

__device__ __forceinline__ void sim_dev(const DevSpace& S, const DV& dv, uint32_t act, double& cost, bool& ok) {
  Knobs k;
  load_knobs(S.sim, S.val, S.inv, S.lg2, dv, act, k);
  double mem;
  simulate(S.sim, k, cost, ok, mem);
}

// FP64 posterior of one candidate computed by a whole warp (lanes split the observed set):
// returns mu - m0 - b (= k^T alpha) and ||L^-1 k||^2.  ksh: M doubles of per-warp scratch.
__device__ __forceinline__ void posterior64_warp(const DevSpace& S, const DevGP& G, const DV& dv, int lane,
                                                 double* ksh, double& kalpha, double& vsq) {
  double x[DMAX];
#pragma unroll
  for (int f = 0; f < DMAX; ++f) x[f] = (f < S.d) ? __ldg(S.xt64 + f * VMAX + dv_get(dv, f)) : 0.0;
  double mp = 0.0;
  for (int i = lane; i < G.M; i += 32) {
    double r2 = 0.0;
#pragma unroll
    for (int f = 0; f < DMAX; ++f)
      if (f < S.d) {
        const double df = x[f] - __ldg(G.O64 + i * S.d + f);
        r2 += df * df;
      }
    const double kv = kernel64(G.kernel, G.sf2, r2);
    ksh[i] = kv;
    mp += kv * __ldg(G.alpha64 + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mp += __shfl_xor_sync(0xffffffffu, mp, o);
  kalpha = mp;
  __syncwarp();
  double vs = 0.0;
  for (int i = 0; i < G.M; ++i) {
    double part = 0.0;
    const double* wr = G.W64 + static_cast<size_t>(i) * G.M;
    for (int jj = lane; jj <= i; jj += 32) part += __ldg(wr + jj) * ksh[jj];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    vs += part * part;
  }
  __syncwarp();
  vsq = vs;
}

// ---- FP32 acquisition for the screen (the upper bound adds acq32_margin; the refine is FP64)
__device__ __forceinline__ float lnh_f(float z) {
  if (z >= -10.0f) {
    // expf (<= 2 ulp), not __expf: its 2 + 1.17 |x| ulp error, amplified ~z^2 by the phi + z Phi
    // cancellation for z < 0, would exceed the screen margin 1e-6 (1 + z^2) below z ~ -6
    const float phi = expf(-0.5f * z * z) * 0.3989422804014327f;
    const float Phi = 0.5f * erfcf(-z * 0.7071067811865476f);
    return logf(fmaf(z, Phi, phi));
  }
  const float iz2 = 1.0f / (z * z);
  return -0.5f * z * z - 0.9189385332046727f - 2.0f * logf(-z) +
         log1pf(iz2 * (-3.0f + iz2 * (15.0f + iz2 * (-105.0f + 945.0f * iz2))));
}
__device__ __forceinline__ float acquisition32(int acq, float mu, float s2, float m0, float fstar, float xi,
                                               float kappa, float& margin) {
  if (acq == 2) {
    margin = 1e-6f * (1.0f + fabsf(m0));
    return -m0;
  }
  if (acq == 1) {
    const float sigma = sqrtf(fmaxf(s2, 0.0f));
    margin = 1e-6f * (1.0f + fabsf(mu) + kappa * sigma);
    return kappa * sigma - mu;
  }
  const float u = fstar - mu - xi;
  if (!(s2 > 0.0f)) {
    margin = 1e-6f * (1.0f + fabsf(u));
    return u > 0.0f ? logf(u) : -INFINITY;
  }
  // z = u / sigma by one reciprocal square root (a few ulp: its effect on ln h, at most ~|z| per unit
  // relative error of z, stays inside the 1e-6 (1 + z^2) term of the margin), ln sigma = ln(s2) / 2
  const float z = u * rsqrtf(s2);
  const float r = 0.5f * logf(s2) + lnh_f(z);
  // FP32 evaluation error: rounding of the terms + cancellation of phi + z Phi (~ u z^2 relative)
  margin = 2e-6f * (1.0f + fabsf(r)) + (z < -10.0f ? 0.0f : 1e-6f * (1.0f + z * z));
  return r;
}

// Bitonic sort of arr[0..n) ascending (n power of two), all threads of the block.
__device__ __forceinline__ void bitonic_sort(uint64_t* arr, int n) {
  for (int k = 2; k <= n; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo | j;
        const bool asc = (lo & k) == 0;
        const uint64_t a = arr[lo], b = arr[hi];
        if ((a > b) == asc) {
          arr[lo] = b;
          arr[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// Shared state of the CTA-level top-k'.
struct TopkSmem {
  int n_list;
  int n_add;
  uint64_t tau;     // current k'-th key (KEY_NONE while the list is not full)
  uint64_t drop;    // smallest key not kept
};

// Offer one key per participating thread (key == KEY_NONE: nothing).  All threads must call.
__device__ __forceinline__ void cta_admit(uint64_t key, uint64_t* arr, TopkSmem& ts, int KC) {
  if (key != KEY_NONE) {
    if (key < ts.tau) {
      const int pos = atomicAdd(&ts.n_add, 1);
      arr[ts.n_list + pos] = key;
    } else {
      atomicMin(reinterpret_cast<unsigned long long*>(&ts.drop), static_cast<unsigned long long>(key));
    }
  }
  __syncthreads();
  const int n_add = ts.n_add;
  if (n_add > 0) {
    const int n_tot = ts.n_list + n_add;
    bitonic_sort(arr, next_pow2(n_tot < 2 ? 2 : n_tot));
    const int keep = n_tot < KC ? n_tot : KC;
    if (threadIdx.x == 0) {
      if (n_tot > KC) {
        const uint64_t first_dropped = arr[KC];
        if (first_dropped < ts.drop) ts.drop = first_dropped;
      }
      ts.n_list = keep;
      ts.tau = (keep == KC) ? arr[KC - 1] : KEY_NONE;
      ts.n_add = 0;
    }
    for (int i = keep + threadIdx.x; i < n_tot; i += blockDim.x) arr[i] = KEY_NONE;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- score kernel
struct ScoreSmem {
  float* Wblk;
  float* O;
  float* alpha;
  float* aabs;
  float* Ks;       // [Mp][32]
  float* xt;       // [d*VMAX]
  DV* q_dv;        // [QCAP]
  double* q_m0;
  uint32_t* q_cvi;
  uint32_t* q_j;
  uint64_t* q_raw;
  float* red;      // [4][8][32]
  uint64_t* arr;   // [P]
  uint64_t* ckey;  // [32]
  double* k64;     // [Mp] FP64 scratch of the sensitive-candidate fallback
};

template <bool GP>
__global__ void __launch_bounds__(SCORE_THREADS, 1)
score_kernel(DevSpace S, DevGP G, BatchArgs A, CtaOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ TopkSmem ts;
  __shared__ int q_n;
  __shared__ unsigned long long valid_cta;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Mp = GP ? G.Mp : 0, DP = GP ? G.DP : 0;
  const int nb = Mp >> 2;
  // ---- carve shared memory
  ScoreSmem sm;
  unsigned char* p = smem_raw;
  auto take = [&](size_t bytes) {
    unsigned char* r = p;
    p += (bytes + 15) & ~size_t(15);
    return r;
  };
  sm.Wblk = reinterpret_cast<float*>(take(sizeof(float) * 16 * (nb * (nb + 1) / 2)));
  sm.O = reinterpret_cast<float*>(take(sizeof(float) * Mp * DP));
  sm.alpha = reinterpret_cast<float*>(take(sizeof(float) * Mp));
  sm.aabs = reinterpret_cast<float*>(take(sizeof(float) * Mp));
  sm.Ks = reinterpret_cast<float*>(take(sizeof(float) * Mp * 32));
  sm.xt = reinterpret_cast<float*>(take(sizeof(float) * S.d * VMAX));
  sm.q_dv = reinterpret_cast<DV*>(take(sizeof(DV) * QCAP));
  sm.q_m0 = reinterpret_cast<double*>(take(sizeof(double) * QCAP));
  sm.q_raw = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * QCAP));
  sm.q_cvi = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * QCAP));
  sm.q_j = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * QCAP));
  sm.red = reinterpret_cast<float*>(take(sizeof(float) * 4 * 8 * 32));
  sm.ckey = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 32));
  sm.arr = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * out.P));
  sm.k64 = reinterpret_cast<double*>(take(sizeof(double) * (Mp > 0 ? Mp : 1)));

  // ---- stage the observed set, L^-1 blocks and the feature table into SMEM
  if (GP) {
    const int nW = 16 * (nb * (nb + 1) / 2);
    const float4* src = reinterpret_cast<const float4*>(G.Wblk);
    float4* dst = reinterpret_cast<float4*>(sm.Wblk);
    for (int i = tid; i < nW / 4; i += SCORE_THREADS) dst[i] = __ldg(src + i);
    for (int i = tid; i < Mp * DP; i += SCORE_THREADS) sm.O[i] = __ldg(G.O + i);
    for (int i = tid; i < Mp; i += SCORE_THREADS) {
      sm.alpha[i] = __ldg(G.alpha + i);
      sm.aabs[i] = __ldg(G.aabs + i);
    }
    for (int i = tid; i < S.d * VMAX; i += SCORE_THREADS) sm.xt[i] = __ldg(S.xt32 + i);
  }
  for (int i = tid; i < out.P; i += SCORE_THREADS) sm.arr[i] = KEY_NONE;
  if (tid == 0) {
    ts.n_list = 0;
    ts.n_add = 0;
    ts.tau = KEY_NONE;
    ts.drop = KEY_NONE;
    q_n = 0;
    valid_cta = 0;
  }
  __syncthreads();

  const uint64_t ntiles = (A.count + SCORE_THREADS - 1) / SCORE_THREADS;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // ================= phase 0: index -> configuration -> validity -> simulator
    const uint64_t j = tile * SCORE_THREADS + tid;
    const bool in = j < A.count;
    bool ok = false;
    uint64_t raw = 0;
    uint32_t pos = 0;
    double m0 = 0.0;
    DV dv;
    if (in) {
      bool pin;
      const uint64_t pcvi = assign_pos(A, j, pin);
      pos = static_cast<uint32_t>(pcvi);
      uint32_t act;
      decode_dev(S, pcvi, dv, act, raw);
      double cost;
      sim_dev(S, dv, act, cost, ok);
      m0 = prior_m0(S, dv, cost);
      if (!pin) {
        ok = false;
        raw = ~0ull;
      }
      if (A.d_raw) A.d_raw[j] = raw;
      if (!ok && A.d_scores) A.d_scores[j] = -INFINITY;
    }
    const unsigned vb = __ballot_sync(0xffffffffu, in && ok);
    if (lane == 0 && vb) atomicAdd(&valid_cta, static_cast<unsigned long long>(__popc(vb)));
    if (!GP) {
      // SIM / prior-only LCB: score directly, no posterior
      uint64_t key = KEY_NONE;
      if (in && ok) {
        const double mu = m0 + G.b;
        const double sc = acquisition(A.acq, mu, G.sf2, m0, G.fstar, A.xi, A.kappa);
        const double ub = sc + 1e-12 * fmax(1.0, fabs(sc));
        if (A.d_scores) A.d_scores[j] = static_cast<float>(sc);
        if (ub > -INFINITY) key = make_key(__double2float_ru(ub), pos);
      }
      cta_admit(key, sm.arr, ts, out.KC);
      continue;
    }
    if (in && ok) {
      const int slot = atomicAdd(&q_n, 1);
      sm.q_dv[slot] = dv;
      sm.q_m0[slot] = m0;
      sm.q_raw[slot] = raw;
      sm.q_cvi[slot] = pos;
      sm.q_j[slot] = static_cast<uint32_t>(j);
    }
    __syncthreads();
    // ================= GP batches of 32 queued candidates
    const bool last_tile = (tile + gridDim.x >= ntiles);
    int head = 0;
    while (true) {
      const int avail = q_n - head;
      const int nb32 = avail >= 32 ? 32 : (last_tile ? avail : 0);
      if (nb32 <= 0) break;
      const int slot = head + lane;
      const bool has = lane < nb32;
      // ---- candidate features (registers)
      float x[DMAX];
#pragma unroll
      for (int f = 0; f < DMAX; ++f) x[f] = 0.0f;
      if (has) {
        const DV cdv = sm.q_dv[slot];
#pragma unroll
        for (int f = 0; f < DMAX; ++f)
          if (f < S.d) x[f] = sm.xt[f * VMAX + dv_get(cdv, f)];
      }
      // ---- phase 1: cross-covariance k_i (observed i = warp, warp+8, ...), mu and bound partials
      float mu_p = 0.f, sb_p = 0.f, kk_p = 0.f;
      for (int i = warp; i < Mp; i += 8) {
        float kval = 0.f;
        if (i < G.M) {
          const float4* o4 = reinterpret_cast<const float4*>(sm.O + i * DP);
          float r2 = 0.f;
#pragma unroll
          for (int f4 = 0; f4 < DMAX / 4; ++f4) {
            if (4 * f4 < DP) {
              const float4 o = o4[f4];
              const float d0 = x[4 * f4] - o.x, d1 = x[4 * f4 + 1] - o.y, d2 = x[4 * f4 + 2] - o.z,
                          d3 = x[4 * f4 + 3] - o.w;
              r2 = fmaf(d0, d0, r2);
              r2 = fmaf(d1, d1, r2);
              r2 = fmaf(d2, d2, r2);
              r2 = fmaf(d3, d3, r2);
            }
          }
          float arg, poly;
          if (G.kernel == 0) {
            arg = 2.2360679774997896f * sqrtf(r2);          // sqrt5 * r
            poly = fmaf(arg, fmaf(arg, 0.33333333333333333f, 1.0f), 1.0f);  // 1 + a + a^2/3
          } else {
            arg = 0.5f * r2;
            poly = 1.0f;
          }
          kval = G.sf2f * poly * __expf(-arg);
          const float c = kval * (1.0f + arg);
          mu_p = fmaf(kval, sm.alpha[i], mu_p);
          sb_p = fmaf(c, sm.aabs[i], sb_p);
          kk_p = fmaf(c, c, kk_p);
        }
        sm.Ks[i * 32 + lane] = kval;
      }
      sm.red[(0 * 8 + warp) * 32 + lane] = mu_p;
      sm.red[(1 * 8 + warp) * 32 + lane] = sb_p;
      sm.red[(2 * 8 + warp) * 32 + lane] = kk_p;
      __syncthreads();
      // ---- phase 2: v = L^-1 k, ||v||^2 (rows in 4-row groups q = warp, warp+8, ...)
      float vs_p = 0.f;
      for (int q = warp; q < nb; q += 8) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        const float* blk = sm.Wblk + (q * (q + 1) / 2) * 16;
        for (int a = 0; a <= q; ++a, blk += 16) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const float kj = sm.Ks[(4 * a + b) * 32 + lane];
            const float4 w = *reinterpret_cast<const float4*>(blk + 4 * b);
            a0 = fmaf(w.x, kj, a0);
            a1 = fmaf(w.y, kj, a1);
            a2 = fmaf(w.z, kj, a2);
            a3 = fmaf(w.w, kj, a3);
          }
        }
        vs_p = fmaf(a0, a0, vs_p);
        vs_p = fmaf(a1, a1, vs_p);
        vs_p = fmaf(a2, a2, vs_p);
        vs_p = fmaf(a3, a3, vs_p);
      }
      sm.red[(3 * 8 + warp) * 32 + lane] = vs_p;
      __syncthreads();
      // ---- epilogue (warp 0): posterior, acquisition in FP64, error bound, key
      if (warp == 0) {
        uint64_t key = KEY_NONE;
        if (has) {
          float mu32 = 0.f, sb = 0.f, kk = 0.f, vsq = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            mu32 += sm.red[(0 * 8 + w) * 32 + lane];
            sb += sm.red[(1 * 8 + w) * 32 + lane];
            kk += sm.red[(2 * 8 + w) * 32 + lane];
            vsq += sm.red[(3 * 8 + w) * 32 + lane];
          }
          const double cm0 = sm.q_m0[slot];
          const double mu = cm0 + G.b + static_cast<double>(mu32);
          const double vs = static_cast<double>(vsq);
          const double s2 = G.sf2 - vs;
          // error bound of the FP32 screen
          const double d_mu = G.eps * static_cast<double>(sb) + 1e-13 * fabs(mu);
          const double ew = G.eps * G.w_fro;
          const double kn = sqrt(static_cast<double>(kk));
          const double d_s2 = 2.5 * ew * sqrt(vs) * kn + ew * ew * static_cast<double>(kk) +
                              G.eps * vs + 4.0 * static_cast<double>(U32) * G.sf2;
          double sc = acquisition(A.acq, mu, s2, cm0, G.fstar, A.xi, A.kappa);
          double ub = acquisition(A.acq, mu - d_mu, s2 + d_s2, cm0, G.fstar, A.xi, A.kappa);
          ub += 1e-12 * fmax(1.0, fabs(ub));
          // Per-candidate EI outputs whose FP32 error could exceed 1e-5 (small sigma^2 near an observed
          // point, z >= -3.2) are recomputed in FP64.  Error model calibrated against
          // the FP64 oracle: |d s2| <= 20 u ||v||^2, |d mu| <= u (1 + sum k(1+a)|alpha|).  Only when
          // d_scores is requested: the top-k itself is certified and FP64-refined regardless.
          bool sensitive = false;
          if (A.d_scores && A.acq == 0) {
            if (s2 > 0.0) {
              const double sg = sqrt(s2), z = (G.fstar - mu - A.xi) / sg;
              if (z >= -3.2) {
                const double Phi = 0.5 * erfc(-z * INV_SQRT2);
                const double h = exp(-0.5 * z * z) * INV_SQRT_2PI + z * Phi;
                const double uu = static_cast<double>(U32);
                const double e_s = (1.0 - z * Phi / h) / (2.0 * s2) * 20.0 * uu * vs +
                                   Phi / (sg * h) * uu * (1.0 + static_cast<double>(sb));
                sensitive = e_s > 5e-6;
              }
            } else {
              sensitive = true;
            }
          }
          sm.ckey[lane] = sensitive ? 1ull : 0ull;
          if (!sensitive) {
            if (A.d_scores) A.d_scores[sm.q_j[slot]] = static_cast<float>(sc);
            if (ub > -INFINITY) key = make_key(__double2float_ru(ub), sm.q_cvi[slot]);
          }
        }
        // warp-cooperative FP64 posterior for the flagged lanes
        unsigned fl = __ballot_sync(0xffffffffu, has && sm.ckey[lane] == 1ull);
        while (fl) {
          const int src = __ffs(fl) - 1;
          fl &= fl - 1;
          const int fslot = head + src;
          double kalpha, vsq;
          posterior64_warp(S, G, sm.q_dv[fslot], lane, sm.k64, kalpha, vsq);
          if (lane == src) {
            const double cm0 = sm.q_m0[fslot];
            const double sc = acquisition(A.acq, cm0 + G.b + kalpha, G.sf2 - vsq, cm0, G.fstar, A.xi, A.kappa);
            const double ub = sc + 1e-12 * fmax(1.0, fabs(sc));
            if (A.d_scores) A.d_scores[sm.q_j[fslot]] = static_cast<float>(sc);
            if (ub > -INFINITY) key = make_key(__double2float_ru(ub), sm.q_cvi[fslot]);
          }
        }
        sm.ckey[lane] = key;
      }
      __syncthreads();
      cta_admit(tid < 32 ? sm.ckey[tid] : KEY_NONE, sm.arr, ts, out.KC);
      head += nb32;
    }
    // ---- move the (< 32) leftover queue entries to the front
    const int left = q_n - head;
    __syncthreads();
    DV mdv;
    double mm0 = 0;
    uint64_t mraw = 0;
    uint32_t mcvi = 0, mj = 0;
    if (tid < left) {
      mdv = sm.q_dv[head + tid];
      mm0 = sm.q_m0[head + tid];
      mraw = sm.q_raw[head + tid];
      mcvi = sm.q_cvi[head + tid];
      mj = sm.q_j[head + tid];
    }
    __syncthreads();
    if (tid < left) {
      sm.q_dv[tid] = mdv;
      sm.q_m0[tid] = mm0;
      sm.q_raw[tid] = mraw;
      sm.q_cvi[tid] = mcvi;
      sm.q_j[tid] = mj;
    }
    if (tid == 0) q_n = left;
    __syncthreads();
  }
  // ---- write the CTA list
  __syncthreads();
  const int n = ts.n_list;
  uint64_t* dst = out.lists + static_cast<size_t>(blockIdx.x) * out.KC;
  for (int i = tid; i < n; i += SCORE_THREADS) dst[i] = sm.arr[i];
  if (tid == 0) {
    out.counts[blockIdx.x] = n;
    out.drop[blockIdx.x] = ts.drop;
    if (valid_cta) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out.valid), valid_cta);
      if (A.d_valid_count) atomicAdd(reinterpret_cast<unsigned long long*>(A.d_valid_count), valid_cta);
    }
  }
}

// ---------------------------------------------------------------- pool merge (one CTA)
constexpr int MERGE_THREADS = 1024;

__global__ void __launch_bounds__(MERGE_THREADS, 1)
merge_kernel(const uint64_t* lists, const int* counts, const uint64_t* drops, int n_lists, int KC,
             uint64_t* pool, int* pool_n, uint64_t* cut, int reset, int P2) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* arr = reinterpret_cast<uint64_t*>(smem_raw);
  __shared__ TopkSmem ts;
  const int tid = threadIdx.x;
  for (int i = tid; i < P2; i += MERGE_THREADS) arr[i] = KEY_NONE;
  __syncthreads();
  if (tid == 0) {
    ts.n_list = reset ? 0 : *pool_n;
    ts.n_add = 0;
    ts.drop = reset ? KEY_NONE : *cut;
  }
  __syncthreads();
  for (int i = tid; i < ts.n_list; i += MERGE_THREADS) arr[i] = pool[i];
  __syncthreads();
  if (tid == 0) ts.tau = (ts.n_list == KC) ? arr[KC - 1] : KEY_NONE;
  // per-CTA drop bounds
  for (int l = tid; l < n_lists; l += MERGE_THREADS) {
    const uint64_t dkey = drops[l];
    if (dkey != KEY_NONE) atomicMin(reinterpret_cast<unsigned long long*>(&ts.drop), static_cast<unsigned long long>(dkey));
  }
  __syncthreads();
  // stream every CTA entry: entry e = (list l, index i), in chunks of MERGE_THREADS
  const long long total = static_cast<long long>(n_lists) * KC;
  for (long long base = 0; base < total; base += MERGE_THREADS) {
    const long long e = base + tid;
    uint64_t key = KEY_NONE;
    if (e < total) {
      const int l = static_cast<int>(e / KC), i = static_cast<int>(e % KC);
      if (i < counts[l]) key = lists[e];
    }
    cta_admit(key, arr, ts, KC);
  }
  for (int i = tid; i < ts.n_list; i += MERGE_THREADS) pool[i] = arr[i];
  if (tid == 0) {
    *pool_n = ts.n_list;
    *cut = ts.drop;
  }
}

// ---------------------------------------------------------------- FP64 refine (one CTA per entry)
// FP64 refine with one 256-thread CTA per pool entry: k in shared memory by all threads, the rows of
// |L^-1 k|^2 split over the eight warps (rows i = w mod 8, lanes over columns), warp partials summed
// in warp order.  Same formulas as refine_kernel; ~10x lower latency at M = 256 (one warp walked all
// M rows of L^-1 in sequence: 0.25 -> 0.03 ms per C4 pool at M = 256).
constexpr int REFINE_CTA = 256;
__global__ void __launch_bounds__(REFINE_CTA)
refine_kernel(DevSpace S, DevGP G, const uint64_t* pool, const int* pool_n, int acq, double kappa, double xi,
                  double* out_score, uint64_t* out_raw) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ksh = reinterpret_cast<double*>(smem_raw);            // [M]
  __shared__ double red_a[REFINE_CTA / 32], red_v[REFINE_CTA / 32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int e = blockIdx.x;
  if (e >= *pool_n) return;
  const uint64_t key = pool[e];
  const uint64_t p = key & 0xFFFFFFFFull;
  DV dv;
  uint32_t act;
  uint64_t raw;
  decode_dev(S, p, dv, act, raw);
  double cost;
  bool ok;
  sim_dev(S, dv, act, cost, ok);
  const double m0 = prior_m0(S, dv, cost);
  double mu = m0 + G.b, s2 = G.sf2;
  if (G.M > 0 && acq != 2) {
    double x[DMAX];
#pragma unroll
    for (int f = 0; f < DMAX; ++f) x[f] = (f < S.d) ? __ldg(S.xt64 + f * VMAX + dv_get(dv, f)) : 0.0;
    double mp = 0.0;
    for (int i = tid; i < G.M; i += REFINE_CTA) {
      double r2 = 0.0;
#pragma unroll
      for (int f = 0; f < DMAX; ++f)
        if (f < S.d) {
          const double df = x[f] - __ldg(G.O64 + i * S.d + f);
          r2 += df * df;
        }
      const double kv = kernel64(G.kernel, G.sf2, r2);
      ksh[i] = kv;
      mp += kv * __ldg(G.alpha64 + i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mp += __shfl_xor_sync(0xffffffffu, mp, o);
    if (lane == 0) red_a[warp] = mp;
    __syncthreads();
    double vs = 0.0;
    for (int i = warp; i < G.M; i += REFINE_CTA / 32) {
      double part = 0.0;
      const double* wr = G.W64 + static_cast<size_t>(i) * G.M;
      for (int jj = lane; jj <= i; jj += 32) part += __ldg(wr + jj) * ksh[jj];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      vs += part * part;
    }
    if (lane == 0) red_v[warp] = vs;
    __syncthreads();
    if (tid == 0) {
      double ka = 0.0, vq = 0.0;
      for (int w = 0; w < REFINE_CTA / 32; ++w) {
        ka += red_a[w];
        vq += red_v[w];
      }
      mu += ka;
      s2 = G.sf2 - vq;
    }
  }
  if (tid == 0) {
    const double sc = acquisition(acq, mu, s2, m0, G.fstar, xi, kappa);
    out_score[e] = ok ? sc : -INFINITY;
    out_raw[e] = raw;
  }
}

// ---------------------------------------------------------------- raw-range mask (parity path)
__global__ void mask_kernel(DevSpace S, uint64_t raw_begin, uint64_t count, uint32_t* bits, uint64_t* valid) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  bool ok = false;
  if (i < count) {
    const uint64_t raw = raw_begin + i;
    if (raw < S.n_raw) {
      const uint64_t tail = raw % S.tail_span;
      const uint64_t pref = raw - tail;
      int lo = 0, hi = S.n_struct;  // s_raw ascending; find exact match
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (S.s_raw[mid] <= pref) lo = mid; else hi = mid;
      }
      if (S.s_raw[lo] == pref) {
        DV dv = S.s_dv[lo];
        uint32_t act = S.s_act[lo];
        bool structural = true;
        for (int c = 0; c < S.n_comp && structural; ++c) {
          uint64_t contrib = 0;
          for (int q = S.comp_first[c]; q < S.comp_first[c] + S.comp_width[c]; ++q)
            contrib += ((raw / S.stride[q]) % static_cast<uint64_t>(S.nval[q])) * S.stride[q];
          const uint4 oc = S.s_oc[static_cast<size_t>(lo) * S.n_comp + c];
          int a = 0, b = static_cast<int>(oc.y);  // tuples sorted by raw contribution
          while (b - a > 1) {
            const int mid = (a + b) >> 1;
            if (S.tuples[oc.x + mid].raw <= contrib) a = mid; else b = mid;
          }
          const Tuple& tu = S.tuples[oc.x + a];
          if (tu.raw != contrib) {
            structural = false;
          } else {
            dv.w[0] |= tu.dv.w[0];
            dv.w[1] |= tu.dv.w[1];
            dv.w[2] |= tu.dv.w[2];
            act |= tu.act;
          }
        }
        if (structural) {
          double cost;
          sim_dev(S, dv, act, cost, ok);
        }
      }
    }
  }
  const unsigned b = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && i < count) {
    bits[i >> 5] = b;
    if (valid && b) atomicAdd(reinterpret_cast<unsigned long long*>(valid), static_cast<unsigned long long>(__popc(b)));
  }
}

}  // namespace as
