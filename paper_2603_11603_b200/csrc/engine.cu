// extern "C" boundary of libautoscout.so (include/autoscout.h): host orchestration of the
// sm_100a kernels in kernels.cuh.  No torch types; plain pointers and sizes.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/autoscout.h"
#include "kernels.cuh"
#include "kernels_tc.cuh"
#include "kernels_tc2.cuh"
#include "host_pool.hpp"
#include "kernels_lml.cuh"
#include "kernels_pool.cuh"
#include "space.hpp"

using namespace as;

namespace {
thread_local std::string g_err;

as_status fail(as_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      if (e_ == cudaErrorMemoryAllocation) return fail(AS_ERR_OOM, cudaGetErrorString(e_)); \
      return fail(AS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
    }                                                                                 \
  } while (0)

constexpr int KC_CAP = 4096;  // largest pool the merge kernel handles (P2 = 8192 keys = 64 KB)

inline int next_pow2_h(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

size_t score_smem_bytes(int Mp, int DP, int d, int P) {
  auto r16 = [](size_t b) { return (b + 15) & ~size_t(15); };
  const int nb = Mp / 4;
  size_t s = 0;
  s += r16(sizeof(float) * 16 * (nb * (nb + 1) / 2));
  s += r16(sizeof(float) * Mp * DP);
  s += r16(sizeof(float) * Mp);
  s += r16(sizeof(float) * Mp);
  s += r16(sizeof(float) * Mp * 32);
  s += r16(sizeof(float) * d * VMAX);
  s += r16(sizeof(DV) * QCAP);
  s += r16(sizeof(double) * QCAP);
  s += r16(sizeof(uint64_t) * QCAP);
  s += r16(sizeof(uint32_t) * QCAP);
  s += r16(sizeof(uint32_t) * QCAP);
  s += r16(sizeof(float) * 4 * 8 * 32);
  s += r16(sizeof(uint64_t) * 32);
  s += r16(sizeof(uint64_t) * P);
  s += r16(sizeof(double) * (Mp > 0 ? Mp : 1));
  return s;
}

size_t tc_smem_bytes(int Mp16, int DP, int d, int P) {
  auto r128 = [](size_t b) { return (b + 127) & ~size_t(127); };
  size_t s = 0;
  s += r128(static_cast<size_t>(TC_NB) * 2ull * Mp16 * TC_KCH * 4);
  s += r128(sizeof(float) * Mp16 * DP);
  s += r128(sizeof(float) * 2 * Mp16);
  s += r128(0);
  s += r128(sizeof(float) * d * VMAX);
  s += r128(sizeof(DV) * TC_QCAP);
  s += r128(sizeof(double) * TC_QCAP);
  s += 2 * r128(sizeof(uint32_t) * TC_QCAP);
  s += 2 * r128(sizeof(uint32_t) * TC_TI * TC_ROWS);
  s += r128(sizeof(double) * TC_TI * TC_ROWS);
  s += r128(sizeof(float) * TC_TI * 3 * TC_ROWS);
  s += r128(sizeof(float) * 4 * TC_ROWS);
  s += r128(sizeof(uint64_t) * P);
  s += r128(sizeof(uint64_t) * 32);
  s += r128(sizeof(uint64_t) * CI);
  return s;
}

// one-hot R2 kernel (kernels_tc2.cuh): fixed arrays + B ring + T ring + E (2) + top-k' keys
size_t tc2_smem_bytes(int Mp16, int Kp, int P, bool big) { return tc2_smem_total(Mp16, Kp, P, big); }
using Tc2KernelFn = void (*)(DevSpace, DevGP, BatchArgs, CtaOut, TcB, Tc2B, CandList);
template <int KT, int NCH>
Tc2KernelFn tc2_kernel_kt(int nh) {
  return nh == 0 ? score_tc2_kernel<16, KT, 0, NCH>
                 : (nh == 2 ? score_tc2_kernel<16, KT, 2, NCH> : score_tc2_kernel<16, KT, 4, NCH>);
}
// compile-time chunk counts for the Matern kernel at M in (240, 256] (C4) and (112, 128] (C5)
Tc2KernelFn tc2_kernel_for(int kernel, int nh, int nch) {
  if (kernel == 0) return nch == 16 ? tc2_kernel_kt<0, 16>(nh) : (nch == 8 ? tc2_kernel_kt<0, 8>(nh) : tc2_kernel_kt<0, 0>(nh));
  return tc2_kernel_kt<1, 0>(nh);
}

using TcKernelFn = void (*)(DevSpace, DevGP, BatchArgs, CtaOut, TcB);
template <int KT>
TcKernelFn tc_kernel_kt(int DP) {
  switch (DP / 4) {
    case 1: return score_tc_kernel<1, 16, KT>;
    case 2: return score_tc_kernel<2, 16, KT>;
    case 3: return score_tc_kernel<3, 16, KT>;
    case 4: return score_tc_kernel<4, 16, KT>;
    case 5: return score_tc_kernel<5, 16, KT>;
    default: return score_tc_kernel<6, 16, KT>;
  }
}
constexpr int TC_WARPS = 16;   // producer warps of the tensor-core kernel (A/B-tested against 8)
TcKernelFn tc_kernel_for(int DP, int kernel) { return kernel == 0 ? tc_kernel_kt<0>(DP) : tc_kernel_kt<1>(DP); }

// TF32 round-to-nearest (ties away), as cvt.rna.tf32.f32
float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

template <typename T>
as_status dalloc(T** p, size_t n, std::vector<void*>& owned) {
  *p = nullptr;
  if (n == 0) n = 1;
  CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T)));
  owned.push_back(*p);
  return AS_OK;
}

template <typename T>
as_status upload(T** p, const std::vector<T>& v, std::vector<void*>& owned) {
  as_status st = dalloc(p, v.size(), owned);
  if (st != AS_OK) return st;
  if (!v.empty()) CUDA_TRY(cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return AS_OK;
}

float key_score(uint64_t key) {
  const uint32_t ord = ~static_cast<uint32_t>(key >> 32);
  const uint32_t u = (ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

struct Entry {
  double score;
  uint64_t raw;
};
static_assert(sizeof(Entry) == 16, "pool entry layout");

bool entry_less(const Entry& a, const Entry& b) {  // score desc, raw asc
  if (a.score != b.score) return a.score > b.score;
  return a.raw < b.raw;
}
}  // namespace

struct as_space {
  HostSpace H;
  int device = -1;
  int n_sm = 0;
  int smem_optin = 0;
  std::vector<void*> owned;
  DevSpace D{};
  // observed set + fit
  std::vector<uint64_t> obs_raw;
  std::vector<double> obs_cost, obs_sim;
  std::vector<DV> obs_dv;
  std::vector<uint32_t> obs_act;
  GPFit fit;
  EnsembleFit ens;                 // NEXT-1 regression-simulator ensemble (gp.prior = "ensemble")
  double* d_ens_tab = nullptr;     // [DMAX * VMAX] its per-(feature, digit) table on the device
  DevGP G{};
  float *d_O = nullptr, *d_alpha = nullptr, *d_aabs = nullptr, *d_Wblk = nullptr;
  double *d_O64 = nullptr, *d_alpha64 = nullptr, *d_W64 = nullptr;
  std::vector<float> h_O, h_alpha, h_aabs, h_Wblk, h_Bch;
  float* d_Bch = nullptr;          // L^-1^T hi/lo chunks for the tensor-core path
  std::vector<uint16_t> h_Tch;     // one-hot R2 operand T (FP16 hi/lo groups, kernels_tc2.cuh)
  std::vector<float> h_xh, h_oh;   // SIMT features of the one-hot kernel (scaled)
  std::vector<uint16_t> h_Wch;     // L^-1^T FP16 hi/lo chunks of the one-hot kernel (scaled by 2^ew)
  uint16_t* d_Tch = nullptr;
  uint16_t* d_ezero = nullptr;
  unsigned char* h_stage = nullptr;   // pinned host staging of the refined pool (one DMA per copy, no pageable bounce)   // zeros for the one-hot E buffers (bulk-copied by the loader warp)
  uint16_t* d_Wch = nullptr;
  float *d_xh = nullptr, *d_oh = nullptr;
  Tc2B t2{};
  CandList list{};                 // compact valid-candidate list of one slice (kernels_gen.cuh)
  size_t list_cap = 0;
  std::vector<cudaEvent_t> sev;    // per-slice events: [gen start, gen end / score start, score end]
  int sev_used = 0;
  bool tc2_auto = true;            // auto path prefers the one-hot kernel when its shared memory fits
  double* d_scratch = nullptr;     // FP64 scratch of the sensitive-output fallback (TC path)
  size_t scratch_cap = 0;
  TcB tb{};
  int path = 0;                    // 0 auto, 1 SIMT, 2 tensor cores (SIMT r^2), 3 tensor cores (one-hot r^2)
  uint64_t slice = 1ull << 27;     // candidates per generate + score slice of the one-hot path (GEN_SLICE)
  std::vector<double> h_O64, h_alpha64, h_W64;
  // pool state
  int KC = 0;
  int KC_max = 0;
  uint64_t* d_lists = nullptr;
  size_t lists_cap = 0;
  int* d_counts = nullptr;
  uint64_t* d_drops = nullptr;
  int counts_cap = 0;
  uint64_t *d_pool = nullptr, *d_cut = nullptr, *d_valid = nullptr;
  int* d_pool_n = nullptr;
  double* d_ref_score = nullptr;
  PoolEntry* d_merge_scratch = nullptr;   // device merge of large gathered pools (> 96 KB)
  size_t merge_scratch_n = 0;
  uint64_t* d_ref_raw = nullptr;
  std::vector<as_score_args> batches;
  bool scored = false;
  uint64_t n_launches = 0;
  uint64_t fit_upload_bytes = 0;   // H2D bytes of the last GP upload (bench e2e accounting)
  // asynchronous observe (autoscout_set_async_observe, prior "sim" only): the host GP fit and the
  // operand tables run on a worker thread; every call that reads the fit joins it first, and
  // score_batch launches the fit-independent candidate generation of its first slice before joining
  bool async_observe = false;
  std::thread fit_thr;
  bool fit_pending = false;
  as_status fit_status = AS_OK;
  std::string fit_msg;
  int pending_M = 0;
  bool gen0_launched = false;      // slice 0 of the next one-hot launch was generated before the join
  // timing
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool ev_recorded = false;
};

namespace {

// host half of the GP upload: device-layout operands staged in host vectors (no CUDA calls; runs
// on the async-observe worker thread)
as_status build_gp_host(as_space* s) {
  const HostSpace& H = s->H;
  const GPFit& F = s->fit;
  const int M = F.M, d = H.d;
  const int Mp = M > 0 ? ((M + 3) / 4) * 4 : 0;
  const int DP = ((d + 3) / 4) * 4;
  const int nb = Mp / 4;
  s->h_O.assign(static_cast<size_t>(Mp) * DP, 0.f);
  s->h_alpha.assign(Mp, 0.f);
  s->h_aabs.assign(Mp, 0.f);
  s->h_Wblk.assign(static_cast<size_t>(16) * (nb * (nb + 1) / 2), 0.f);
  s->h_O64.assign(static_cast<size_t>(M) * d, 0.0);
  s->h_alpha64 = F.alpha;
  s->h_W64 = F.Wl;
  for (int i = 0; i < M; ++i) {
    for (int j = 0; j < d; ++j) {
      s->h_O[i * DP + j] = H.xt32[j * VMAX + dv_get(s->obs_dv[i], j)];
      s->h_O64[i * d + j] = F.X[i * d + j];
    }
    s->h_alpha[i] = static_cast<float>(F.alpha[i]);
    s->h_aabs[i] = static_cast<float>(std::fabs(F.alpha[i]));
  }
  for (int q = 0; q < nb; ++q)
    for (int a = 0; a <= q; ++a)
      for (int b = 0; b < 4; ++b)
        for (int r = 0; r < 4; ++r) {
          const int row = 4 * q + r, col = 4 * a + b;
          float w = 0.f;
          if (row < M && col < M && col <= row) w = static_cast<float>(F.Wl[static_cast<size_t>(row) * M + col]);
          s->h_Wblk[(static_cast<size_t>(q) * (q + 1) / 2 + a) * 16 + b * 4 + r] = w;
        }
  // B operand of the tensor-core path: chunk c = rows i in [16c, Mp16) x columns j in [16c, 16c+16)
  // of L^-1 (i.e. L^-1^T in K-major form), split hi/lo TF32, core-matrix layout (kmajor_off).
  const int Mp16 = M > 0 ? ((M + 15) / 16) * 16 : 0;
  const int nch = Mp16 / TC_KCH;
  s->h_Bch.clear();
  s->tb = TcB{};
  s->tb.Mp16 = Mp16;
  s->tb.nch = nch;
  s->tb.ndb = (2 * Mp16 + 32 * TC_NA <= 512) ? 2 : 1;
  {
    uint32_t need = static_cast<uint32_t>(s->tb.ndb * Mp16 + 32 * TC_NA), cols = 32;
    while (cols < need) cols <<= 1;
    s->tb.tmem_cols = cols;
  }
  // chunk offsets first, then the chunks in parallel on the host pool (each writes its own range)
  HostPool& pool = HostPool::get();
  const bool par = M >= 128;  // small fits: inline (the pool wake-ups would dominate)
  {
    size_t tot = 0;
    for (int c = 0; c < nch; ++c) {
      s->tb.off[c] = static_cast<uint32_t>(tot);
      tot += 2ull * (Mp16 - c * TC_KCH) * TC_KCH;
    }
    s->h_Bch.assign(tot, 0.f);
  }
  pool.run(nch, [&](int c) {
    const int N = Mp16 - c * TC_KCH;
    const size_t base = s->tb.off[c];
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < TC_KCH; ++k) {
        const int i = c * TC_KCH + n, j = c * TC_KCH + k;
        float w = 0.f;
        if (i < M && j < M && j <= i) w = static_cast<float>(F.Wl[static_cast<size_t>(i) * M + j]);
        const float hi = tf32_rna(w), lo = tf32_rna(w - hi);
        const uint32_t off = tc::kmajor_off(n, k, TC_KCH / 4) / 4;
        s->h_Bch[base + off] = hi;
        s->h_Bch[base + static_cast<size_t>(N) * TC_KCH + off] = lo;
      }
  }, par);
  // T operand of the one-hot R2 contraction (kernels_tc2.cuh): group g = observed points
  // [64g, 64g+64) x one-hot columns (f, v); T = 2^s (xt_f[v] - o_jf)^2 in FP64, split hi + lo FP16.
  // SIMT features: 2^(s/2) xt and 2^(s/2) o in FP32.
  {
    Tc2B& t2 = s->t2;
    const int Kp = t2.Kp, nh = t2.nh, GR = TC2_RG * TC_KCH;
    const int ngr = (nch + TC2_RG - 1) / TC2_RG;
    s->h_Tch.assign(static_cast<size_t>(ngr) * 2 * GR * Kp, 0);
    double tmax = 0.0;
    for (int f = 0; f < d; ++f) {
      if (t2.eoff[f] < 0) continue;
      for (int v = 0; v < H.feat[f].n; ++v)
        for (int w = 0; w < H.feat[f].n; ++w) {
          const double q = H.xt64[f * VMAX + v] - H.xt64[f * VMAX + w];
          tmax = std::max(tmax, q * q);
        }
    }
    int sc = 0;   // even, largest one-hot entry in (2^13, 2^15]
    if (tmax > 0.0) {
      while (tmax * std::ldexp(1.0, sc) > 32768.0) sc -= 2;
      while (tmax * std::ldexp(1.0, sc + 2) <= 32768.0) sc += 2;
    }
    t2.r2_scale = static_cast<float>(std::ldexp(1.0, -sc));
    t2.r_scale = static_cast<float>(std::ldexp(1.0, -sc / 2));
    auto h16 = [](double x) {
      const __half h = __double2half(x);
      uint16_t u;
      std::memcpy(&u, &h, 2);
      return u;
    };
    auto v16 = [](uint16_t u) {
      __half h;
      std::memcpy(&h, &u, 2);
      return static_cast<double>(__half2float(h));
    };
    pool.run(ngr * GR, [&](int task) {     // one observed point per task
      const int gi = task / GR, n = task % GR;
      uint16_t* base = s->h_Tch.data() + static_cast<size_t>(gi) * 2 * GR * Kp;
      {
        const int j = gi * GR + n;
        if (j >= M) return;
        for (int f = 0; f < d; ++f) {
          if (t2.eoff[f] < 0) continue;
          for (int v = 0; v < H.feat[f].n; ++v) {
            const double q = H.xt64[f * VMAX + v] - F.X[static_cast<size_t>(j) * d + f];
            const double x = std::ldexp(q * q, sc);
            const uint16_t hi = h16(x);
            // row order inside the group: producer thread jq reads its 4 points of each of the 4
            // chunks as 16 contiguous accumulator columns (kernels_tc2.cuh)
            const int np = 16 * ((n % 16) / 4) + 4 * (n / 16) + (n % 4);
            const uint32_t o = tc::kmajor_off16(np, t2.eoff[f] + v, Kp / 8) / 2;
            base[o] = hi;
            base[static_cast<size_t>(GR) * Kp + o] = h16(x - v16(hi));
          }
        }
      }
    }, par);
    // L^-1^T chunks for the FP16 contraction: chunk c = rows i in [16c, Mp16) x columns j in
    // [16c, 16c+16), 2^ew L^-1[i][j] split hi + lo FP16 (kmajor_off16); k is scaled by 2^ek in-kernel
    {
      double wmax = 0.0;
      for (double w : F.Wl) wmax = std::max(wmax, std::fabs(w));
      int ew = 0;
      if (wmax > 0.0) {
        while (wmax * std::ldexp(1.0, ew) > 32768.0) --ew;
        while (wmax * std::ldexp(1.0, ew + 1) <= 32768.0) ++ew;
      }
      int ek = 0;
      while (H.sf2 * std::ldexp(1.0, ek) > 32768.0) --ek;
      while (H.sf2 * std::ldexp(1.0, ek + 1) <= 32768.0) ++ek;
      t2.ek = ek;
      t2.k_unscale = static_cast<float>(std::ldexp(1.0, -ek));
      t2.vsq_unscale = static_cast<float>(std::ldexp(1.0, -2 * (ek + ew)));
      {
        size_t tot = 0;
        for (int c = 0; c < nch; ++c) {
          t2.woff[c] = static_cast<uint32_t>(tot);
          tot += 2ull * (Mp16 - c * TC_KCH) * TC_KCH;
        }
        s->h_Wch.assign(tot, 0);
      }
      pool.run(nch, [&](int c) {
        const int N = Mp16 - c * TC_KCH;
        const size_t base = t2.woff[c];
        for (int n = 0; n < N; ++n)
          for (int k = 0; k < TC_KCH; ++k) {
            const int i = c * TC_KCH + n, j = c * TC_KCH + k;
            double w = 0.0;
            if (i < M && j < M && j <= i) w = std::ldexp(F.Wl[static_cast<size_t>(i) * M + j], ew);
            const uint16_t hi = h16(w);
            const uint32_t o = tc::kmajor_off16(n, k, TC_KCH / 8) / 2;
            s->h_Wch[base + o] = hi;
            s->h_Wch[base + static_cast<size_t>(N) * TC_KCH + o] = h16(w - v16(hi));
          }
      }, par);
    }
    const double hs = std::ldexp(1.0, sc / 2);
    s->h_xh.assign(static_cast<size_t>(4) * VMAX, 0.f);
    s->h_oh.assign(static_cast<size_t>(std::max(Mp16, 1)) * 4, 0.f);
    for (int h = 0; h < nh; ++h) {
      const int f = t2.hf[h];
      if (f < 0) continue;
      for (int v = 0; v < H.feat[f].n; ++v) s->h_xh[h * VMAX + v] = static_cast<float>(H.xt64[f * VMAX + v] * hs);
      for (int j = 0; j < M; ++j) s->h_oh[j * nh + h] = static_cast<float>(F.X[static_cast<size_t>(j) * d + f] * hs);
    }
  }
  DevGP& G = s->G;
  G.M = M;
  G.Mp = Mp;
  G.DP = DP;
  G.kernel = H.kernel;
  G.sf2 = H.sf2;
  G.sf2f = static_cast<float>(H.sf2);
  G.b = F.b;
  G.fstar = M > 0 ? F.fstar : INFINITY;
  G.eps = 2.0 * (d + 8 + M) * std::ldexp(1.0, -24);
  G.w_fro = F.w_fro;
  return AS_OK;
}

// device half of the GP upload: H2D of the staged operands on stream st
as_status upload_gp_device(as_space* s, cudaStream_t st) {
  if (s->device < 0) return AS_OK;
  DevGP& G = s->G;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> as_status {
    if (bytes) CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    s->fit_upload_bytes += bytes;
    return AS_OK;
  };
  as_status r;
  s->fit_upload_bytes = 0;
  if ((r = cp(s->d_O, s->h_O.data(), s->h_O.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_alpha, s->h_alpha.data(), s->h_alpha.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_aabs, s->h_aabs.data(), s->h_aabs.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_Wblk, s->h_Wblk.data(), s->h_Wblk.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_O64, s->h_O64.data(), s->h_O64.size() * 8)) != AS_OK) return r;
  if ((r = cp(s->d_alpha64, s->h_alpha64.data(), s->h_alpha64.size() * 8)) != AS_OK) return r;
  if ((r = cp(s->d_W64, s->h_W64.data(), s->h_W64.size() * 8)) != AS_OK) return r;
  if ((r = cp(s->d_Bch, s->h_Bch.data(), s->h_Bch.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_Tch, s->h_Tch.data(), s->h_Tch.size() * 2)) != AS_OK) return r;
  if ((r = cp(s->d_Wch, s->h_Wch.data(), s->h_Wch.size() * 2)) != AS_OK) return r;
  s->t2.wch = s->d_Wch;
  if ((r = cp(s->d_xh, s->h_xh.data(), s->h_xh.size() * 4)) != AS_OK) return r;
  if ((r = cp(s->d_oh, s->h_oh.data(), s->h_oh.size() * 4)) != AS_OK) return r;
  s->t2.tch = s->d_Tch;
  s->t2.xh = s->d_xh;
  s->t2.oh = s->d_oh;
  s->tb.chunks = s->d_Bch;
  CUDA_TRY(cudaStreamSynchronize(st));  // staging vectors may be reused by the next observe()
  G.O = s->d_O;
  G.alpha = s->d_alpha;
  G.aabs = s->d_aabs;
  G.Wblk = s->d_Wblk;
  G.O64 = s->d_O64;
  G.alpha64 = s->d_alpha64;
  G.W64 = s->d_W64;
  return AS_OK;
}

as_status upload_gp(as_space* s, cudaStream_t st) {
  as_status r = build_gp_host(s);
  return r == AS_OK ? upload_gp_device(s, st) : r;
}

// wait for an asynchronous observe(): commit its fit (or report its deferred error) and upload it
as_status join_fit(const as_space* cs, cudaStream_t st) {
  as_space* s = const_cast<as_space*>(cs);
  if (!s->fit_pending) return AS_OK;
  s->fit_thr.join();
  s->fit_pending = false;
  if (s->fit_status != AS_OK) {
    const as_status r = s->fit_status;
    s->fit_status = AS_OK;
    return fail(r, "deferred observe(): " + s->fit_msg);
  }
  return upload_gp_device(s, st);
}

as_status ensure_lists(as_space* s, int grid) {
  const size_t need = static_cast<size_t>(grid) * s->KC;
  if (need > s->lists_cap) {
    if (s->d_lists) cudaFree(s->d_lists);
    CUDA_TRY(cudaMalloc(&s->d_lists, need * sizeof(uint64_t)));
    s->lists_cap = need;
  }
  if (grid > s->counts_cap) {
    if (s->d_counts) cudaFree(s->d_counts);
    if (s->d_drops) cudaFree(s->d_drops);
    CUDA_TRY(cudaMalloc(&s->d_counts, grid * sizeof(int)));
    CUDA_TRY(cudaMalloc(&s->d_drops, grid * sizeof(uint64_t)));
    s->counts_cap = grid;
  }
  return AS_OK;
}

// One-hot tensor-core path: the batch is processed in slices (default 2^27 candidates, a 5.4 GB worst-
// case list; autoscout_set_slice lowers it); per slice
// the generate kernel writes the compact list of valid candidates and the score kernel consumes
// it (one CTA per SM), then the pool merge.
constexpr uint64_t GEN_SLICE = 1ull << 27;   // default slice (one slice for the 10^8 bench batch)
constexpr int SEV_MAX = 3 * 64;

as_status ensure_cand_list(as_space* s, size_t cap) {
  if (cap <= s->list_cap) return AS_OK;
  CandList& L = s->list;
  void* ptrs[] = {L.cvi, L.j, L.m0, L.dv0, L.dv1, L.dv2, L.count};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  L = CandList{};
  const size_t n = cap + TC_ROWS;   // padding: the last tile's staging copy is rounded up
  CUDA_TRY(cudaMalloc(&L.cvi, n * 4));
  CUDA_TRY(cudaMalloc(&L.j, n * 4));
  CUDA_TRY(cudaMalloc(&L.m0, n * 8));
  CUDA_TRY(cudaMalloc(&L.dv0, n * 8));
  CUDA_TRY(cudaMalloc(&L.dv1, n * 8));
  CUDA_TRY(cudaMalloc(&L.dv2, n * 8));
  CUDA_TRY(cudaMalloc(&L.count, sizeof(unsigned long long)));
  s->list_cap = cap;
  return AS_OK;
}

// Per-structure partial evaluation of the derived simulator for the generation kernel (common.cuh
// SimRec): false (generic path) unless every base-term knob is a structural-prefix feature (or
// absent) and the resource check reads at most 64 combinations of tail digits.  Self-checked on
// the host against simulate() before it is used.
bool build_simrec(const HostSpace& H, std::vector<SimRec>& rec, SimFast& F) {
  F = SimFast{};
  rec.clear();
  const SimParams& P = H.sim;
  if (P.mode != 1 || H.n_struct <= 0) return false;
  auto tail = [&](int kb) { return P.kf[kb] >= H.n_prefix; };
  for (int kb : {K_PP, K_VPP, K_TP, K_DP, K_CP, K_EP, K_MBS, K_AR, K_ARL})
    if (tail(kb)) return false;
  // tail features the resource check reads (dopt, sp), with their tail gate ancestors so that the
  // combination fixes their activity
  std::vector<int> cf;
  std::vector<int> stack;
  for (int kb : {K_DOPT, K_SP})
    if (tail(kb)) stack.push_back(P.kf[kb]);
  while (!stack.empty()) {
    const int f = stack.back();
    stack.pop_back();
    if (f < H.n_prefix || std::find(cf.begin(), cf.end(), f) != cf.end()) continue;
    cf.push_back(f);
    for (const Atom& a : H.feat[f].req) stack.push_back(a.ref);
  }
  std::sort(cf.begin(), cf.end());
  uint64_t ncomb = 1;
  for (int f : cf) ncomb *= static_cast<uint64_t>(H.feat[f].n);
  if (cf.size() > static_cast<size_t>(SR_MAXCF) || ncomb > 64) return false;
  F.n_cf = static_cast<int>(cf.size());
  uint32_t mul = 1;
  for (int i = F.n_cf - 1; i >= 0; --i) {
    F.cf_w[i] = cf[i] >> 3;
    F.cf_s[i] = (cf[i] & 7) * 8;
    F.cf_mul[i] = mul;
    mul *= static_cast<uint32_t>(H.feat[cf[i]].n);
  }
  rec.resize(H.n_struct);
  for (int st = 0; st < H.n_struct; ++st) {
    Knobs k;
    load_knobs(P, H.val.data(), H.inv.data(), H.lg2.data(), H.s_dv[st], H.s_act[st], k);
    SimRec& r = rec[st];
    simrec_base(P, k, r);
    r.memok = 0;
    r.pad2 = 0;
    for (uint64_t c = 0; c < ncomb; ++c) {
      // the structure with combination c in the listed tail features and every other tail feature
      // at its default digit
      uint64_t raw = H.s_raw[st];
      for (int f = H.n_prefix; f < H.d; ++f) raw += static_cast<uint64_t>(H.feat[f].dflt) * H.stride[f];
      for (int i = 0; i < F.n_cf; ++i) {
        const uint64_t dig = (c / F.cf_mul[i]) % static_cast<uint64_t>(H.feat[cf[i]].n);
        raw += (dig - static_cast<uint64_t>(H.feat[cf[i]].dflt)) * H.stride[cf[i]];
      }
      int dg[DMAX];
      DV dv;
      uint32_t act;
      bool structural;
      if (!raw_decode(H, raw, dg, dv, act, structural) || !structural) continue;   // never occurs
      double cost, mem;
      bool ok;
      simulate_host(H, dv, act, cost, ok, mem);
      if (ok) r.memok |= 1ull << c;
    }
  }
  F.on = 1;
  // self-check on a sample of valid-structure configurations: the same resource bit, the cost to
  // FP64 re-association
  const uint64_t n_check = std::min<uint64_t>(H.n_cvi, 20000);
  for (uint64_t i = 0; i < n_check; ++i) {
    const uint64_t p = (H.n_cvi <= n_check) ? i : (splitmix64(0xC4EC ^ i) % H.n_cvi);
    DV dv;
    uint32_t act;
    uint64_t raw;
    if (!cvi_decode(H, p, dv, act, raw)) continue;
    int st = static_cast<int>(std::upper_bound(H.prefix.begin(), H.prefix.begin() + H.n_struct + 1, p) - H.prefix.begin()) - 1;
    double c1, m1, c2;
    bool ok1, ok2;
    simulate_host(H, dv, act, c1, ok1, m1);
    sim_fast(P, F, H.val.data(), H.lg2.data(), rec[st], dv, act, c2, ok2);
    if (ok1 != ok2 || !(std::fabs(c1 - c2) <= 1e-12 * std::fabs(c1))) {
      F = SimFast{};
      rec.clear();
      return false;
    }
  }
  return true;
}

struct GenCfg {
  void (*k)(DevSpace, BatchArgs, uint64_t, uint64_t, CandList, int, unsigned long long*);
  int ci_n;
  size_t smem;
  int grid;
};

// generation kernel configuration (independent of the GP fit)
GenCfg gen_config(as_space* s) {
  GenCfg g{};
  // whole prefix table + bucket index in SMEM when they fit, else a coarse index of GEN_CI_MAX entries
  const bool by_bucket = s->H.n_struct + 1 <= GEN_CI_MAX;
  const int ci_n = by_bucket ? -1 : std::min(s->H.n_struct, GEN_CI_MAX);
  const size_t gen_smem = by_bucket ? (static_cast<size_t>(s->H.n_struct) + 1) * 8 + (s->D.n_bucket + 1) * 4
                                    : static_cast<size_t>(ci_n) * 8;
  // tail-group count 5 (C2, C4, C5) as a compile-time constant: all group records loaded up front
  const bool nc5 = s->D.n_comp == 5;
  auto gen_k = s->D.ens_on ? (nc5 ? gen_kernel<true, 5> : gen_kernel<true, 0>)
                           : (nc5 ? gen_kernel<false, 5> : gen_kernel<false, 0>);
  int occ = 1;
  if (cudaFuncSetAttribute(gen_k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gen_smem)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gen_k, GEN_THREADS, gen_smem) != cudaSuccess)
    occ = 1;
  g.k = gen_k;
  g.ci_n = ci_n;
  g.smem = gen_smem;
  g.grid = s->n_sm * std::max(occ, 1);
  return g;
}

// candidates [j0, j0 + nj) of the batch into the compact list (count reset first)
as_status gen_launch(as_space* s, const GenCfg& g, const BatchArgs& A, uint64_t j0, uint64_t nj, cudaStream_t st) {
  CUDA_TRY(cudaMemsetAsync(s->list.count, 0, sizeof(unsigned long long), st));
  g.k<<<g.grid, GEN_THREADS, g.smem, st>>>(s->D, A, j0, nj, s->list, g.ci_n, reinterpret_cast<unsigned long long*>(s->d_valid));
  CUDA_TRY(cudaGetLastError());
  ++s->n_launches;
  return AS_OK;
}

BatchArgs batch_args(const as_space* s, const as_score_args& a) {
  BatchArgs A{};
  A.mode = a.mode;
  A.acq = a.acq;
  A.begin = a.begin;
  A.count = a.count;
  A.fk = feistel_make(s->H.n_cvi, a.seed);
  A.list = a.mode == AS_MODE_LIST ? a.d_positions : nullptr;
  A.n_cvi = s->H.n_cvi;
  A.kappa = a.kappa;
  A.xi = a.xi;
  A.d_scores = a.d_scores;
  A.d_screen = a.d_screen;
  A.d_raw = a.d_raw;
  A.d_valid_count = a.d_valid_count;
  return A;
}

as_status launch_tc2(as_space* s, const BatchArgs& A, CtaOut out, size_t smem, bool reset, cudaStream_t st) {
  s->sev_used = 0;
  if (s->timing) CUDA_TRY(cudaEventRecord(s->ev[0], st));
  const uint64_t count = A.count;
  const int grid = s->n_sm;
  as_status r = ensure_lists(s, grid);
  if (r != AS_OK) return r;
  out.lists = s->d_lists;            // ensure_lists may have reallocated them
  out.counts = s->d_counts;
  out.drop = s->d_drops;
  if (count > 0) {
    r = ensure_cand_list(s, static_cast<size_t>(std::min<uint64_t>(count, s->slice)));
    if (r != AS_OK) return r;
  }
  const GenCfg gc = gen_config(s);
  auto k2 = tc2_kernel_for(s->G.kernel, s->t2.nh, s->tb.nch);
  CUDA_TRY(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  TcB tb = s->tb;
  tb.scratch = s->d_scratch;
  const int P2 = next_pow2_h(s->KC + MERGE_THREADS);
  CUDA_TRY(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P2 * 8));
  const uint64_t SL = s->slice;
  const uint64_t n_slices = count == 0 ? 1 : (count + SL - 1) / SL;
  for (uint64_t sl = 0; sl < n_slices; ++sl) {
    const uint64_t j0 = sl * SL, nj = std::min<uint64_t>(SL, count - j0);
    const bool ev = s->timing && s->sev_used + 3 <= static_cast<int>(s->sev.size());
    if (nj > 0) {
      if (ev) CUDA_TRY(cudaEventRecord(s->sev[s->sev_used], st));
      if (sl == 0 && s->gen0_launched) {
        s->gen0_launched = false;              // generated before the observe() join (score_batch)
      } else {
        r = gen_launch(s, gc, A, j0, nj, st);
        if (r != AS_OK) return r;
      }
      if (ev) CUDA_TRY(cudaEventRecord(s->sev[s->sev_used + 1], st));
      static unsigned long long* tr_buf = nullptr;
      const char* tr_path = std::getenv("AS_TC2_TRACE");   // development aid: CTA-0 phase timeline
      const size_t tr_n = static_cast<size_t>(TC2_TR_TILES) * TC2_TR_EV * TC2_TR_W;
      if (tr_path != nullptr && tr_buf == nullptr) {
        CUDA_TRY(cudaMalloc(&tr_buf, tr_n * 8));
        CUDA_TRY(cudaMemcpyToSymbol(g_tc2_trace, &tr_buf, sizeof(tr_buf)));
      }
      if (tr_buf != nullptr) CUDA_TRY(cudaMemsetAsync(tr_buf, 0, tr_n * 8, st));
      k2<<<grid, TC2_THREADS, smem, st>>>(s->D, s->G, A, out, tb, s->t2, s->list);
      CUDA_TRY(cudaGetLastError());
      ++s->n_launches;
      if (tr_buf != nullptr) {
        std::vector<unsigned long long> h(tr_n);
        CUDA_TRY(cudaMemcpyAsync(h.data(), tr_buf, tr_n * 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (FILE* f = std::fopen(tr_path, "ab")) {
          std::fwrite(h.data(), 8, tr_n, f);
          std::fclose(f);
        }
      }
      if (ev) {
        CUDA_TRY(cudaEventRecord(s->sev[s->sev_used + 2], st));
        s->sev_used += 3;
      }
    }
    if (sl + 1 == n_slices && s->timing) CUDA_TRY(cudaEventRecord(s->ev[1], st));
    merge_kernel<<<1, MERGE_THREADS, P2 * 8, st>>>(s->d_lists, s->d_counts, s->d_drops, nj > 0 ? grid : 0, s->KC,
                                                   s->d_pool, s->d_pool_n, s->d_cut, (reset && sl == 0) ? 1 : 0, P2);
    CUDA_TRY(cudaGetLastError());
    ++s->n_launches;
  }
  if (s->timing) {
    CUDA_TRY(cudaEventRecord(s->ev[2], st));
    s->ev_recorded = true;
  }
  return AS_OK;
}

as_status launch_batch(as_space* s, const as_score_args& a, bool reset, cudaStream_t st) {
  const bool gp = (a.acq != AS_ACQ_SIM) && s->G.M > 0;
  int P = next_pow2_h(s->KC + SCORE_THREADS);
  const int P_tc2 = next_pow2_h(s->KC + 4 * TC_ROWS);   // lazy admission: room for >= 3 tiles before a prune
  const bool tc2_fits = tc2_smem_bytes(s->tb.Mp16, s->t2.Kp, P_tc2, s->G.kernel == 0 && s->tb.nch == 16) <= static_cast<size_t>(s->smem_optin);
  // auto: the one-hot tensor-core kernel for M >= 64, and below that for large batches too (its
  // generation split beats the fused SIMT kernel there: C4, M = 48, 10^8 candidates 38.5 -> 15.3 ms;
  // small batches keep the single-launch SIMT kernel for latency)
  const bool big = a.count >= (1ull << 20);
  const bool use_tc2 = gp && (s->path == 3 || (s->path == 0 && (s->G.M >= 64 || big) && tc2_fits && s->tc2_auto));
  const bool use_tc = !use_tc2 && gp && (s->path == 2 || (s->path == 0 && s->G.M >= 64));
  size_t smem = 0;
  if (use_tc2) {
    P = P_tc2;
    smem = tc2_smem_bytes(s->tb.Mp16, s->t2.Kp, P, s->G.kernel == 0 && s->tb.nch == 16);
  } else if (use_tc) {
    smem = tc_smem_bytes(s->tb.Mp16, s->G.DP, s->H.d, P);
  } else {
    smem = score_smem_bytes(gp ? s->G.Mp : 0, gp ? s->G.DP : 0, s->H.d, P);
  }
  if (smem > static_cast<size_t>(s->smem_optin))
    return fail(AS_ERR_CAPACITY, "score kernel shared memory exceeds the per-CTA limit (M or k too large)");
  const uint64_t ntiles = (a.count + SCORE_THREADS - 1) / SCORE_THREADS;
  int grid = 0;
  if (a.count > 0) {
    int occ = 1;
    if (use_tc2) {
      CUDA_TRY(cudaFuncSetAttribute(tc2_kernel_for(s->G.kernel, s->t2.nh, s->tb.nch), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      occ = 1;
    } else if (use_tc) {
      CUDA_TRY(cudaFuncSetAttribute(tc_kernel_for(s->G.DP, s->G.kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      occ = 1;
    } else if (gp) {
      CUDA_TRY(cudaFuncSetAttribute(score_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score_kernel<true>, SCORE_THREADS, smem));
    } else {
      CUDA_TRY(cudaFuncSetAttribute(score_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score_kernel<false>, SCORE_THREADS, smem));
    }
    if (occ < 1) occ = 1;
    const uint64_t g = std::min<uint64_t>(static_cast<uint64_t>(s->n_sm) * occ, ntiles);
    grid = static_cast<int>(g);
  }
  if (use_tc2) grid = s->n_sm;        // persistent: one CTA per SM over the candidate lists
  as_status r = ensure_lists(s, std::max(grid, 1));
  if (r != AS_OK) return r;
  if ((use_tc || use_tc2) && a.d_scores && a.acq == AS_ACQ_EI) {
    const size_t need = static_cast<size_t>(std::max(grid, 1)) * TC_EPI_WARPS * std::max(s->tb.Mp16, 1);
    if (need > s->scratch_cap) {
      if (s->d_scratch) cudaFree(s->d_scratch);
      CUDA_TRY(cudaMalloc(&s->d_scratch, need * sizeof(double)));
      s->scratch_cap = need;
    }
  }
  const BatchArgs A = batch_args(s, a);
  if (!use_tc2) s->gen0_launched = false;   // an early slice-0 generation is simply unused
  CtaOut out{s->d_lists, s->d_counts, s->d_drops, s->d_valid, s->KC, P};
  DevGP G = s->G;
  if (use_tc2) return launch_tc2(s, A, out, smem, reset, st);
  s->sev_used = 0;
  if (s->timing) CUDA_TRY(cudaEventRecord(s->ev[0], st));
  if (grid > 0) {
    if (use_tc) {
      TcB tb = s->tb;
      tb.scratch = s->d_scratch;
      tc_kernel_for(s->G.DP, s->G.kernel)<<<grid, TC_WARPS * 32 + 32, smem, st>>>(s->D, G, A, out, tb);
    } else if (gp) {
      score_kernel<true><<<grid, SCORE_THREADS, smem, st>>>(s->D, G, A, out);
    } else {
      score_kernel<false><<<grid, SCORE_THREADS, smem, st>>>(s->D, G, A, out);
    }
    CUDA_TRY(cudaGetLastError());
    ++s->n_launches;
  }
  if (s->timing) CUDA_TRY(cudaEventRecord(s->ev[1], st));
  const int P2 = next_pow2_h(s->KC + MERGE_THREADS);
  CUDA_TRY(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P2 * 8));
  merge_kernel<<<1, MERGE_THREADS, P2 * 8, st>>>(s->d_lists, s->d_counts, s->d_drops, grid, s->KC, s->d_pool,
                                                 s->d_pool_n, s->d_cut, reset ? 1 : 0, P2);
  CUDA_TRY(cudaGetLastError());
  ++s->n_launches;
  if (s->timing) {
    CUDA_TRY(cudaEventRecord(s->ev[2], st));
    s->ev_recorded = true;
  }
  return AS_OK;
}

// Refine the running pool in FP64 and bring it to the host, sorted (score desc, raw asc).
as_status refine_pool(as_space* s, int acq, double kappa, double xi, cudaStream_t st, std::vector<Entry>& ent,
                      uint64_t& cut, int& n_pool) {
  const size_t smem = static_cast<size_t>(std::max(s->G.M, 1)) * sizeof(double);
  refine_kernel<<<s->KC, REFINE_CTA, smem, st>>>(s->D, s->G, s->d_pool, s->d_pool_n, acq, kappa, xi,
                                                         s->d_ref_score, s->d_ref_raw);
  CUDA_TRY(cudaGetLastError());
  ++s->n_launches;
  // into pinned staging: [cut u64][n_pool i32 (+pad)][KC scores][KC raws]
  unsigned char* hs = s->h_stage;
  double* sc = reinterpret_cast<double*>(hs + 16);
  uint64_t* rw = reinterpret_cast<uint64_t*>(hs + 16 + static_cast<size_t>(s->KC) * 8);
  CUDA_TRY(cudaMemcpyAsync(hs, s->d_cut, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(hs + 8, s->d_pool_n, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(sc, s->d_ref_score, s->KC * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(rw, s->d_ref_raw, s->KC * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  std::memcpy(&cut, hs, sizeof(uint64_t));
  std::memcpy(&n_pool, hs + 8, sizeof(int));
  ent.clear();
  for (int e = 0; e < n_pool; ++e)
    if (std::isfinite(sc[e])) ent.push_back({sc[e], rw[e]});
  std::sort(ent.begin(), ent.end(), entry_less);
  // a configuration scored more than once (repeated LIST positions, overlapping accumulated
  // batches) has one FP64 score: equal raws are adjacent after the sort, keep one
  ent.erase(std::unique(ent.begin(), ent.end(), [](const Entry& x, const Entry& y) { return x.raw == y.raw; }),
            ent.end());
  return AS_OK;
}

// A refit (observe, observe_clear, set_gp_hyper) changes every score: the running pool and the
// recorded batches belong to the previous fit, so topk needs a new score_batch first.
void invalidate_pool(as_space* s) {
  s->scored = false;
  s->batches.clear();
}

as_status rescore_all(as_space* s, cudaStream_t st) {
  for (size_t i = 0; i < s->batches.size(); ++i) {
    as_score_args a = s->batches[i];
    as_status r = launch_batch(s, a, i == 0, st);
    if (r != AS_OK) return r;
  }
  return AS_OK;
}

// Certified refine: grow k' and re-score the recorded batches until the k-th refined score beats
// the upper bound of every dropped candidate.
as_status certified_pool(as_space* s, int k, cudaStream_t st, std::vector<Entry>& ent, Entry& cut_e,
                         bool& certified) {
  const as_score_args& a0 = s->batches.front();
  for (;;) {
    uint64_t cut;
    int n_pool;
    as_status r = refine_pool(s, a0.acq, a0.kappa, a0.xi, st, ent, cut, n_pool);
    if (r != AS_OK) return r;
    if (cut == KEY_NONE) {
      cut_e = Entry{-INFINITY, ~0ull};
    } else {
      DV dv;
      uint32_t act;
      uint64_t raw = 0;
      cvi_decode(s->H, cut & 0xFFFFFFFFull, dv, act, raw);
      cut_e = Entry{static_cast<double>(key_score(cut)), raw};
    }
    certified = (cut == KEY_NONE) || (static_cast<int>(ent.size()) >= k && entry_less(ent[k - 1], cut_e));
    if (certified || s->KC * 2 > s->KC_max) return AS_OK;
    s->KC *= 2;
    r = rescore_all(s, st);
    if (r != AS_OK) return r;
  }
}

}  // namespace

extern "C" {

const char* autoscout_last_error(void) { return g_err.c_str(); }

as_status autoscout_space_create(const char* space_json, int32_t cuda_device, as_space** out) {
  if (!space_json || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  as_space* s = new as_space();
  Status st = build_space(space_json, s->H);
  if (!st.ok()) {
    delete s;
    return fail(static_cast<as_status>(st.code), st.msg);
  }
  s->device = cuda_device;
  {
    // one-hot layout of the R2 contraction (kernels_tc2.cuh): column of (f, v) = eoff[f] + v.
    // The widest features move to the SIMT side (at most 4) while the one-hot width exceeds
    // gp.onehot_max_width (default TC2_KPMAX = 64); their count is padded to 0 / 2 / 4 with a zero feature (hf = -1).
    Tc2B& t2 = s->t2;
    const int d = s->H.d;
    std::vector<bool> simt(d, false);
    int K = 0;
    for (int f = 0; f < d; ++f) K += s->H.feat[f].n;
    int nh = 0;
    for (int f = 0; f < 4; ++f) t2.hf[f] = -1;
    while (K > s->H.onehot_max && nh < 4) {
      int best = -1;
      for (int f = 0; f < d; ++f)
        if (!simt[f] && (best < 0 || s->H.feat[f].n > s->H.feat[best].n)) best = f;
      if (best < 0) break;
      simt[best] = true;
      t2.hf[nh++] = best;
      K -= s->H.feat[best].n;
    }
    t2.nh = nh == 0 ? 0 : (nh <= 2 ? 2 : 4);
#ifdef AS_EXP_NH0
    t2.nh = 0;   // timing experiment only: SIMT features dropped (wrong scores)
#endif
    K = 0;
    for (int f = 0; f < DMAX; ++f) {
      t2.eoff[f] = (f < d && simt[f]) ? -1 : K;
      if (f < d && !simt[f]) K += s->H.feat[f].n;
    }
    t2.Kp = std::max(16, ((K + 15) / 16) * 16);
  }
  // GP fit with no observations (prior only)
  gp_fit(s->H, {}, {}, {}, {}, s->fit);
  s->G = DevGP{};
  s->G.kernel = s->H.kernel;
  s->G.sf2 = s->H.sf2;
  s->G.sf2f = static_cast<float>(s->H.sf2);
  s->G.fstar = INFINITY;
  if (cuda_device >= 0) {
    auto cleanup = [&](as_status r) {
      autoscout_space_destroy(s);
      return r;
    };
    cudaError_t e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return cleanup(fail(AS_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
    if (cudaDeviceGetAttribute(&s->n_sm, cudaDevAttrMultiProcessorCount, cuda_device) != cudaSuccess ||
        cudaDeviceGetAttribute(&s->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, cuda_device) != cudaSuccess)
      return cleanup(fail(AS_ERR_CUDA, "device attribute query failed"));
    s->smem_optin -= 256;  // static shared memory of the score kernel
    const HostSpace& H = s->H;
    DevSpace& D = s->D;
    D.d = H.d;
    D.n_prefix = H.n_prefix;
    D.n_comp = static_cast<int>(H.comp_first.size());
    D.n_struct = H.n_struct;
    D.n_cvi = H.n_cvi;
    D.n_raw = H.n_raw;
    D.tail_span = H.tail_span;
    for (int j = 0; j < DMAX; ++j) {
      D.stride[j] = j < H.d ? H.stride[j] : 0;
      D.nval[j] = j < H.d ? H.feat[j].n : 1;
      D.comp_first[j] = j < D.n_comp ? H.comp_first[j] : 0;
      D.comp_width[j] = j < D.n_comp ? H.comp_width[j] : 0;
    }
    D.sim = H.sim;
    // (offset, count, magic, shifts): t / count as (hi + ((t - hi) >> sh1)) >> sh2 with
    // hi = umulhi(magic, t) (Granlund-Montgomery round-up method; exact for every 32-bit t)
    std::vector<uint4> oc(H.s_off.size());
    for (size_t i = 0; i < oc.size(); ++i) {
      const uint32_t c = H.s_cnt[i] > 0 ? H.s_cnt[i] : 1;
      int l = 0;
      while ((1ull << l) < c) ++l;
      const uint32_t magic = static_cast<uint32_t>((((1ull << 32) * ((1ull << l) - c)) / c) + 1);
      const uint32_t sh1 = l > 0 ? 1u : 0u, sh2 = l > 0 ? static_cast<uint32_t>(l - 1) : 0u;
      oc[i] = make_uint4(H.s_off[i], H.s_cnt[i], magic, sh1 | (sh2 << 8));
    }
    as_status r;
    uint64_t *p_prefix, *p_sraw;
    uint32_t* p_sact;
    DV* p_sdv;
    uint4* p_oc;
    Tuple* p_tu;
    double *p_val, *p_inv, *p_lg2, *p_xt64;
    float* p_xt32;
    if ((r = upload(&p_prefix, H.prefix, s->owned)) != AS_OK) return cleanup(r);
    {
      // bucket index: bucket[b] = structure holding position b << bshift (positions beyond n_cvi
      // map to the last structure); at most 4096 buckets
      int bshift = 0;
      while (((H.n_cvi + (1ull << bshift) - 1) >> bshift) > 4096) ++bshift;
      const int nb = static_cast<int>((H.n_cvi + (1ull << bshift) - 1) >> bshift);
      std::vector<uint32_t> bk(static_cast<size_t>(nb) + 1);
      int st = 0;
      for (int b = 0; b <= nb; ++b) {
        const uint64_t pos = std::min<uint64_t>(static_cast<uint64_t>(b) << bshift, H.n_cvi - 1);
        while (st + 1 < H.n_struct && H.prefix[st + 1] <= pos) ++st;
        bk[b] = static_cast<uint32_t>(st);
      }
      uint32_t* p_bk;
      if ((r = upload(&p_bk, bk, s->owned)) != AS_OK) return cleanup(r);
      D.bucket = p_bk;
      D.n_bucket = nb;
      D.bshift = bshift;
    }
    if ((r = upload(&p_sraw, H.s_raw, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_sact, H.s_act, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_sdv, H.s_dv, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_oc, oc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_tu, H.tuples, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_val, H.val, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_inv, H.inv, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_lg2, H.lg2, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_xt64, H.xt64, s->owned)) != AS_OK) return cleanup(r);
    if ((r = upload(&p_xt32, H.xt32, s->owned)) != AS_OK) return cleanup(r);
    D.prefix = p_prefix;
    D.s_raw = p_sraw;
    D.s_act = p_sact;
    D.s_dv = p_sdv;
    D.s_oc = p_oc;
    D.tuples = p_tu;
    D.val = p_val;
    D.inv = p_inv;
    D.lg2 = p_lg2;
    D.xt64 = p_xt64;
    D.xt32 = p_xt32;
    {
      std::vector<SimRec> srec;
      SimFast sf;
      D.srec = nullptr;
      D.sf = SimFast{};
      if (build_simrec(H, srec, sf)) {
        SimRec* p_srec;
        if ((r = upload(&p_srec, srec, s->owned)) != AS_OK) return cleanup(r);
        D.srec = p_srec;
        D.sf = sf;
      }
    }
    if ((r = dalloc(&s->d_ens_tab, static_cast<size_t>(DMAX) * VMAX, s->owned)) != AS_OK) return cleanup(r);
    D.ens_tab = s->d_ens_tab;
    D.ens_on = 0;
    // GP buffers at capacity
    const int Mc = MMAX, DPc = ((H.d + 3) / 4) * 4, nbc = Mc / 4;
    if ((r = dalloc(&s->d_O, static_cast<size_t>(Mc) * DPc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_alpha, Mc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_aabs, Mc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_Wblk, static_cast<size_t>(16) * nbc * (nbc + 1) / 2, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_O64, static_cast<size_t>(Mc) * H.d, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_alpha64, Mc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_W64, static_cast<size_t>(Mc) * Mc, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_Bch, static_cast<size_t>(2) * TC_KCH * (Mc / TC_KCH) * (Mc / TC_KCH + 1) / 2 * TC_KCH,
                    s->owned)) != AS_OK)
      return cleanup(r);
    if ((r = dalloc(&s->d_Tch, static_cast<size_t>(Mc) * 2 * s->t2.Kp, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_xh, static_cast<size_t>(4) * VMAX, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_Wch, static_cast<size_t>(2) * TC_KCH * (Mc / TC_KCH) * (Mc / TC_KCH + 1) / 2 * TC_KCH,
                    s->owned)) != AS_OK)
      return cleanup(r);
    if ((r = dalloc(&s->d_oh, static_cast<size_t>(Mc) * 4, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_ezero, static_cast<size_t>(TC_ROWS) * s->t2.Kp, s->owned)) != AS_OK) return cleanup(r);
    CUDA_TRY(cudaMemset(s->d_ezero, 0, static_cast<size_t>(TC_ROWS) * s->t2.Kp * sizeof(uint16_t)));
    s->t2.ezero = s->d_ezero;
    // pool buffers at capacity
    s->KC_max = KC_CAP;
    if ((r = dalloc(&s->d_pool, KC_CAP, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_pool_n, 1, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_cut, 1, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_valid, 2, s->owned)) != AS_OK) return cleanup(r);   // [0] valid count, [1] pool flag
    if ((r = dalloc(&s->d_ref_score, KC_CAP, s->owned)) != AS_OK) return cleanup(r);
    if ((r = dalloc(&s->d_ref_raw, KC_CAP, s->owned)) != AS_OK) return cleanup(r);
    if (cudaMallocHost(reinterpret_cast<void**>(&s->h_stage), 16 + static_cast<size_t>(KC_CAP) * 16) != cudaSuccess)
      return cleanup(fail(AS_ERR_OOM, "pinned host staging allocation failed"));
    e = cudaMemset(s->d_pool_n, 0, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(s->d_valid, 0, sizeof(uint64_t));
    if (e != cudaSuccess) return cleanup(fail(AS_ERR_CUDA, cudaGetErrorString(e)));
    for (int i = 0; i < 4; ++i)
      if (cudaEventCreate(&s->ev[i]) != cudaSuccess) return cleanup(fail(AS_ERR_CUDA, "cudaEventCreate"));
    s->sev.assign(SEV_MAX, nullptr);
    for (auto& e : s->sev)
      if (cudaEventCreate(&e) != cudaSuccess) return cleanup(fail(AS_ERR_CUDA, "cudaEventCreate"));
  }
  *out = s;
  return AS_OK;
}

void autoscout_space_destroy(as_space* s) {
  if (!s) return;
  if (s->fit_pending) {   // a pending asynchronous fit finishes before the handle goes away
    s->fit_thr.join();
    s->fit_pending = false;
  }
  if (s->device >= 0) {
    cudaSetDevice(s->device);
    for (void* p : s->owned) cudaFree(p);
    if (s->h_stage) cudaFreeHost(s->h_stage);
    if (s->d_merge_scratch) cudaFree(s->d_merge_scratch);
    if (s->d_lists) cudaFree(s->d_lists);
    if (s->d_counts) cudaFree(s->d_counts);
    if (s->d_drops) cudaFree(s->d_drops);
    if (s->d_scratch) cudaFree(s->d_scratch);
    for (auto& e : s->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : s->sev)
      if (e) cudaEventDestroy(e);
    {
      CandList& L = s->list;
      void* ptrs[] = {L.cvi, L.j, L.m0, L.dv0, L.dv1, L.dv2, L.count};
      for (void* q : ptrs)
        if (q) cudaFree(q);
    }
  }
  delete s;
}

as_status autoscout_space_info(const as_space* s, as_space_info* out) {
  if (!s || !out) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  out->n_raw = s->H.n_raw;
  out->n_cvi = s->H.n_cvi;
  out->n_features = s->H.d;
  out->n_structures = s->H.n_struct;
  out->n_prefix = s->H.n_prefix;
  out->n_components = static_cast<int32_t>(s->H.comp_first.size());
  out->n_observed = s->fit.M;
  out->max_observed = MMAX;
  out->n_launches = s->n_launches;
  out->fit_upload_bytes = s->fit_upload_bytes;
  return AS_OK;
}

as_status autoscout_observe(as_space* s, const uint64_t* raw_idx, const double* cost, int64_t n, void* cuda_stream) {
  if (!s || n < 0 || (n > 0 && (!raw_idx || !cost))) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  {
    const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream));
    if (jr != AS_OK) return jr;
  }
  if (static_cast<int64_t>(s->obs_raw.size()) + n > MMAX)
    return fail(AS_ERR_CAPACITY, "more than " + std::to_string(MMAX) + " observed configurations");
  std::vector<DV> ndv;
  std::vector<uint32_t> nact;
  std::vector<double> nsim;
  for (int64_t i = 0; i < n; ++i) {
    if (!(cost[i] > 0.0) || !std::isfinite(cost[i])) return fail(AS_ERR_INVALID_ARG, "observed cost must be finite and > 0");
    int dig[DMAX];
    DV dv;
    uint32_t act;
    bool structural;
    if (!raw_decode(s->H, raw_idx[i], dig, dv, act, structural))
      return fail(AS_ERR_INDEX_RANGE, "observed raw index >= n_raw");
    double cs, mem;
    bool ok;
    simulate_host(s->H, dv, act, cs, ok, mem);
    if (!structural || !ok) return fail(AS_ERR_INVALID_CONFIG, "observed configuration is not valid (raw " + std::to_string(raw_idx[i]) + ")");
    ndv.push_back(dv);
    nact.push_back(act);
    nsim.push_back(cs);
  }
  std::vector<DV> all_dv = s->obs_dv;
  std::vector<uint32_t> all_act = s->obs_act;
  std::vector<double> all_cost = s->obs_cost, all_sim = s->obs_sim;
  all_dv.insert(all_dv.end(), ndv.begin(), ndv.end());
  all_act.insert(all_act.end(), nact.begin(), nact.end());
  all_cost.insert(all_cost.end(), cost, cost + n);
  all_sim.insert(all_sim.end(), nsim.begin(), nsim.end());
  // the numeric fit (+ the device-layout operand tables): inline, or on a worker thread
  auto fit_work = [s, all_dv = std::move(all_dv), all_act = std::move(all_act), all_cost = std::move(all_cost),
                   all_sim = std::move(all_sim), raws = std::vector<uint64_t>(raw_idx, raw_idx + n)]() mutable
      -> std::pair<as_status, std::string> {
    GPFit fit;
    EnsembleFit ens;
    std::vector<double> m0_ens;
    if (s->H.prior == 1) {
      ensemble_fit(s->H, all_dv, all_cost, ens);
      if (ens.on)
        for (const DV& dv : all_dv) m0_ens.push_back(ensemble_m0(s->H, ens, dv));
    }
    Status st = gp_fit(s->H, all_dv, all_act, all_cost, all_sim, fit, ens.on ? &m0_ens : nullptr);
    if (!st.ok()) return {static_cast<as_status>(st.code), st.msg};
    s->ens = std::move(ens);
    s->obs_raw.insert(s->obs_raw.end(), raws.begin(), raws.end());
    s->obs_dv = std::move(all_dv);
    s->obs_act = std::move(all_act);
    s->obs_cost = std::move(all_cost);
    s->obs_sim = std::move(all_sim);
    s->fit = std::move(fit);
    return {build_gp_host(s), std::string()};
  };
  // asynchronous only where the fit is worth a thread (M >= 128: ~1 ms of host work at M = 256)
  if (s->async_observe && s->H.prior != 1 && s->device >= 0 && s->obs_dv.size() + ndv.size() >= 128) {
    invalidate_pool(s);   // the running pool was screened under the previous fit
    s->pending_M = static_cast<int>(s->obs_dv.size() + ndv.size());
    s->fit_pending = true;
    s->fit_thr = std::thread([s, w = std::move(fit_work)]() mutable {
      const auto r = w();
      s->fit_status = r.first;
      s->fit_msg = r.second;
    });
    return AS_OK;
  }
  const auto r = fit_work();
  if (r.first != AS_OK) return fail(r.first, r.second);
  invalidate_pool(s);     // the running pool was screened under the previous fit
  if (s->device >= 0) {
    if (s->ens.on) {
      CUDA_TRY(cudaMemcpy(s->d_ens_tab, s->ens.tab.data(), s->ens.tab.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    s->D.ens_on = s->ens.on ? 1 : 0;
    s->D.ens_c0 = s->ens.c0;
  }
  const as_status ur = upload_gp_device(s, static_cast<cudaStream_t>(cuda_stream));
  if (ur == AS_OK && s->ens.on) s->fit_upload_bytes += s->ens.tab.size() * sizeof(double);
  return ur;
}

as_status autoscout_observe_clear(as_space* s) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  join_fit(s, nullptr);   // a pending fit is superseded (a deferred error no longer matters)
  s->obs_raw.clear();
  s->obs_dv.clear();
  s->obs_act.clear();
  s->obs_cost.clear();
  s->obs_sim.clear();
  gp_fit(s->H, {}, {}, {}, {}, s->fit);
  s->ens = EnsembleFit{};
  s->D.ens_on = 0;
  invalidate_pool(s);
  return upload_gp(s, nullptr);
}

as_status autoscout_observe_info(const as_space* s, int32_t* m_out, double* b_out, double* fstar_out) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  if (m_out) *m_out = s->fit.M;
  if (b_out) *b_out = s->fit.b;
  if (fstar_out) *fstar_out = s->fit.M > 0 ? s->fit.fstar : INFINITY;
  return AS_OK;
}

as_status autoscout_score_batch(as_space* s, const as_score_args* a, void* cuda_stream) {
  if (!s || !a) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (s->device < 0) return fail(AS_ERR_STATE, "host-only handle cannot score (no CUDA device)");
  if (a->mode != AS_MODE_RANGE && a->mode != AS_MODE_SAMPLE && a->mode != AS_MODE_LIST)
    return fail(AS_ERR_INVALID_ARG, "bad mode");
  if (a->mode == AS_MODE_LIST && a->count > 0 && !a->d_positions)
    return fail(AS_ERR_INVALID_ARG, "LIST mode needs d_positions");
  if (a->mode == AS_MODE_LIST && a->count > 0 && s->H.n_cvi == 0)
    return fail(AS_ERR_INDEX_RANGE, "LIST mode on a space without valid configurations");
  if (a->acq < AS_ACQ_EI || a->acq > AS_ACQ_SIM) return fail(AS_ERR_INVALID_ARG, "bad acquisition");
  if (a->k < 1 || a->k > 1024) return fail(AS_ERR_INVALID_ARG, "k must be in [1, 1024]");
  // the screen's upper bound evaluates LCB at s2 + d_s2 and EI at mu - d_mu: monotone only for
  // kappa >= 0; non-finite kappa / xi would void the certificate
  if (!std::isfinite(a->kappa) || !std::isfinite(a->xi) || a->kappa < 0.0f)
    return fail(AS_ERR_INVALID_ARG, "kappa must be finite and >= 0, xi finite");
  if (a->mode != AS_MODE_LIST && (a->begin > s->H.n_cvi || a->count > s->H.n_cvi - a->begin))
    return fail(AS_ERR_INDEX_RANGE, "batch exceeds [0, n_cvi)");
  if (a->acq == AS_ACQ_EI && (s->fit_pending ? s->pending_M : s->G.M) == 0)
    return fail(AS_ERR_NO_OBSERVATIONS, "EI needs at least one observation");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CUDA_TRY(cudaSetDevice(s->device));
  const bool reset = !a->accumulate || !s->scored;
  if (!reset) {
    const as_score_args& b0 = s->batches.front();
    if (a->acq != b0.acq || a->kappa != b0.kappa || a->xi != b0.xi)
      return fail(AS_ERR_INVALID_ARG, "accumulate = 1 needs the acquisition, kappa and xi of the pool's first batch");
  }
  if (reset) CUDA_TRY(cudaMemsetAsync(s->d_valid, 0, sizeof(uint64_t), st));
  if (s->fit_pending) {
    // asynchronous observe(): the candidate generation of the first slice does not depend on the
    // fit, so it runs on the GPU while the host thread finishes the fit (one-hot path only)
    if (reset && a->acq != AS_ACQ_SIM && a->count > 0 && (s->path == 0 || s->path == 3)) {
      const uint64_t nj = std::min<uint64_t>(a->count, s->slice);
      as_status r = ensure_cand_list(s, static_cast<size_t>(nj));
      if (r == AS_OK) r = gen_launch(s, gen_config(s), batch_args(s, *a), 0, nj, st);
      if (r != AS_OK) return r;
      s->gen0_launched = true;
    }
    const as_status jr = join_fit(s, st);
    if (jr != AS_OK) {
      s->gen0_launched = false;
      return jr;
    }
  }
  if (reset) {
    s->batches.clear();
    s->KC = std::min(a->k + std::max(a->k, 64), s->KC_max);
  }
  as_score_args rec = *a;
  rec.d_scores = nullptr;
  rec.d_raw = nullptr;
  rec.d_valid_count = nullptr;
  rec.d_screen = nullptr;
  s->batches.push_back(rec);
  as_status r = launch_batch(s, *a, reset, st);
  if (r != AS_OK) return r;
  s->scored = true;
  return AS_OK;
}

as_status autoscout_topk(as_space* s, int32_t k, uint64_t* raw_out, double* score_out, int32_t* n_out,
                         void* cuda_stream) {
  if (!s || !raw_out || !score_out || !n_out || k < 1) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream))) return jr;
  if (!s->scored || s->batches.empty()) return fail(AS_ERR_STATE, "nothing scored");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CUDA_TRY(cudaSetDevice(s->device));
  std::vector<Entry> ent;
  Entry cut_e;
  bool certified;
  as_status r = certified_pool(s, k, st, ent, cut_e, certified);
  if (r != AS_OK) return r;
  const int n = std::min<int>(k, static_cast<int>(ent.size()));
  for (int i = 0; i < n; ++i) {
    raw_out[i] = ent[i].raw;
    score_out[i] = ent[i].score;
  }
  *n_out = n;
  if (!certified) return fail(AS_ERR_UNCERTIFIED, "top-k could not be certified at the maximum pool size");
  return AS_OK;
}

as_status autoscout_topk_pool(as_space* s, int32_t k, void* pool_out, int32_t cap, int32_t* n_out, void* cut_out,
                              void* cuda_stream) {
  if (!s || !pool_out || !n_out || !cut_out || cap < 1 || k < 1) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream))) return jr;
  if (!s->scored || s->batches.empty()) return fail(AS_ERR_STATE, "nothing scored");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CUDA_TRY(cudaSetDevice(s->device));
  std::vector<Entry> ent;
  Entry cut_e;
  bool certified;
  // a locally certified pool keeps the global certificate cheap; it is re-checked in topk_merge
  as_status r = certified_pool(s, k, st, ent, cut_e, certified);
  if (r != AS_OK) return r;
  const int n = std::min<int>(cap, static_cast<int>(ent.size()));
  // entries beyond `cap` are dropped here: the best of them bounds the rest
  if (static_cast<int>(ent.size()) > cap && entry_less(ent[cap], cut_e)) cut_e = ent[cap];
  std::memcpy(pool_out, ent.data(), static_cast<size_t>(n) * sizeof(Entry));
  std::memcpy(cut_out, &cut_e, sizeof(Entry));
  *n_out = n;
  return AS_OK;
}

as_status autoscout_topk_merge(const as_space* s, const void* pools, const int32_t* counts, const void* cuts,
                               int32_t n_pools, int32_t cap, int32_t k, uint64_t* raw_out, double* score_out,
                               int32_t* n_out, int32_t* certified_out) {
  (void)s;
  if (!pools || !counts || !cuts || n_pools < 1 || cap < 1 || k < 1 || !raw_out || !score_out || !n_out)
    return fail(AS_ERR_INVALID_ARG, "bad arguments");
  const Entry* P = static_cast<const Entry*>(pools);
  const Entry* C = static_cast<const Entry*>(cuts);
  std::vector<Entry> all;
  Entry cut{-INFINITY, ~0ull};
  bool any_cut = false;
  for (int p = 0; p < n_pools; ++p) {
    if (counts[p] < 0 || counts[p] > cap) return fail(AS_ERR_INVALID_ARG, "pool count out of range");
    for (int i = 0; i < counts[p]; ++i) all.push_back(P[static_cast<size_t>(p) * cap + i]);
    if (C[p].score != -INFINITY) {
      if (!any_cut || entry_less(C[p], cut)) cut = C[p];
      any_cut = true;
    }
  }
  std::sort(all.begin(), all.end(), entry_less);
  all.erase(std::unique(all.begin(), all.end(), [](const Entry& a, const Entry& b) { return a.raw == b.raw; }),
            all.end());
  const int n = std::min<int>(k, static_cast<int>(all.size()));
  for (int i = 0; i < n; ++i) {
    raw_out[i] = all[i].raw;
    score_out[i] = all[i].score;
  }
  *n_out = n;
  const bool cert = !any_cut || (static_cast<int>(all.size()) >= k && entry_less(all[k - 1], cut));
  if (certified_out) *certified_out = cert ? 1 : 0;
  return cert ? AS_OK : fail(AS_ERR_UNCERTIFIED, "merged top-k could not be certified");
}

as_status autoscout_topk_pool_device(as_space* s, int32_t k, void* d_pool_out, int32_t cap, void* cuda_stream) {
  if (!s || !d_pool_out || cap < 1 || k < 1) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream))) return jr;
  if (s->device < 0) return fail(AS_ERR_STATE, "host-only handle");
  if (!s->scored || s->batches.empty()) return fail(AS_ERR_STATE, "nothing scored");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CUDA_TRY(cudaSetDevice(s->device));
  const as_score_args& a0 = s->batches.front();
  int* h_flag = reinterpret_cast<int*>(s->h_stage);   // pinned; refine_pool is not running concurrently
  for (;;) {
    const size_t rsm = static_cast<size_t>(std::max(s->G.M, 1)) * sizeof(double);
    refine_kernel<<<s->KC, REFINE_CTA, rsm, st>>>(s->D, s->G, s->d_pool, s->d_pool_n, a0.acq, a0.kappa,
                                                          a0.xi, s->d_ref_score, s->d_ref_raw);
    CUDA_TRY(cudaGetLastError());
    ++s->n_launches;
    const int n2 = next_pow2_h(std::max(s->KC, 2));
    CUDA_TRY(cudaFuncSetAttribute(pool_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, n2 * 16));
    pool_pack_kernel<<<1, POOL_THREADS, static_cast<size_t>(n2) * 16, st>>>(
        s->D, s->d_ref_score, s->d_ref_raw, s->d_pool_n, s->d_cut, n2, k, cap, static_cast<PoolEntry*>(d_pool_out),
        reinterpret_cast<int*>(s->d_valid) + 2);
    CUDA_TRY(cudaGetLastError());
    ++s->n_launches;
    // 4 bytes back (the local certificate), not the pool: grow k' and re-score if it failed
    CUDA_TRY(cudaMemcpyAsync(h_flag, reinterpret_cast<int*>(s->d_valid) + 2, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (*h_flag || s->KC * 2 > s->KC_max) return AS_OK;
    s->KC *= 2;
    as_status r = rescore_all(s, st);
    if (r != AS_OK) return r;
  }
}

as_status autoscout_topk_merge_device(as_space* s, const void* d_pools, int32_t n_pools, int32_t cap, int32_t k,
                                      void* d_out, void* cuda_stream) {
  if (!s || !d_pools || !d_out || n_pools < 1 || cap < 1 || k < 1) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (s->device < 0) return fail(AS_ERR_STATE, "host-only handle");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  CUDA_TRY(cudaSetDevice(s->device));
  const int n2 = next_pow2_h(std::max(n_pools * cap, 2));
  const size_t bytes = static_cast<size_t>(n2) * sizeof(PoolEntry);
  PoolEntry* gbuf = nullptr;
  size_t smem = 0;
  if (bytes <= 96 * 1024) {
    smem = bytes;
    CUDA_TRY(cudaFuncSetAttribute(pool_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  } else {
    if (s->merge_scratch_n < static_cast<size_t>(n2)) {
      if (s->d_merge_scratch) cudaFree(s->d_merge_scratch);
      s->d_merge_scratch = nullptr;
      CUDA_TRY(cudaMalloc(&s->d_merge_scratch, bytes));
      s->merge_scratch_n = n2;
    }
    gbuf = s->d_merge_scratch;
  }
  pool_merge_kernel<<<1, POOL_THREADS, smem, st>>>(static_cast<const PoolEntry*>(d_pools), n_pools, cap, k, n2, gbuf,
                                                   static_cast<PoolEntry*>(d_out));
  CUDA_TRY(cudaGetLastError());
  ++s->n_launches;
  return AS_OK;
}

as_status autoscout_decode(const as_space* s, uint64_t raw, int32_t* digits_out, int32_t* valid_out) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  int dig[DMAX];
  DV dv;
  uint32_t act;
  bool structural;
  if (!raw_decode(s->H, raw, dig, dv, act, structural)) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  if (digits_out)
    for (int j = 0; j < s->H.d; ++j) digits_out[j] = dig[j];
  if (valid_out) {
    double c, m;
    bool ok = false;
    if (structural) simulate_host(s->H, dv, act, c, ok, m);
    *valid_out = (structural && ok) ? 1 : 0;
  }
  return AS_OK;
}

as_status autoscout_activity(const as_space* s, uint64_t raw, uint32_t* active_mask_out) {
  if (!s || !active_mask_out) return fail(AS_ERR_INVALID_ARG, "null argument");
  int dig[DMAX];
  DV dv;
  uint32_t act;
  bool structural;
  if (!raw_decode(s->H, raw, dig, dv, act, structural)) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  *active_mask_out = act;
  return AS_OK;
}

as_status autoscout_cvi_to_raw(const as_space* s, uint64_t cvi, uint64_t* raw_out) {
  if (!s || !raw_out) return fail(AS_ERR_INVALID_ARG, "null argument");
  DV dv;
  uint32_t act;
  if (!cvi_decode(s->H, cvi, dv, act, *raw_out)) return fail(AS_ERR_INDEX_RANGE, "cvi >= n_cvi");
  return AS_OK;
}

// ---------------------------------------------------------------- NEXT-4: ML-II evidence on the device
as_status autoscout_gp_lml(as_space* s, const double* hyp, int32_t n_set, double* lml_out, void* cuda_stream) {
  if (!s || (n_set > 0 && (!hyp || !lml_out)) || n_set < 0) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream))) return jr;
  if (s->device < 0) return fail(AS_ERR_STATE, "host-only handle cannot launch (no CUDA device)");
  const int M = s->fit.M, d = s->H.d;
  if (M == 0) return fail(AS_ERR_NO_OBSERVATIONS, "the evidence needs observations");
  for (int64_t i = 0; i < static_cast<int64_t>(n_set) * (d + 2); ++i)
    if (!(hyp[i] > 0.0) || !std::isfinite(hyp[i])) return fail(AS_ERR_INVALID_ARG, "hyper-parameters must be finite and > 0");
  if (n_set == 0) return AS_OK;
  CUDA_TRY(cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  std::vector<double> phi(static_cast<size_t>(M) * d);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < d; ++j) {
      const int n = s->H.feat[j].n;
      phi[static_cast<size_t>(i) * d + j] = n > 1 ? double(dv_get(s->obs_dv[i], j)) / double(n - 1) : 0.0;
    }
  const int grid = std::min<int>(n_set, s->n_sm * 2);
  const size_t work = static_cast<size_t>(grid) * M * M;
  double *d_phi = nullptr, *d_r = nullptr, *d_hyp = nullptr, *d_out = nullptr, *d_work = nullptr;
  auto release = [&]() {
    cudaFree(d_phi);
    cudaFree(d_r);
    cudaFree(d_hyp);
    cudaFree(d_out);
    cudaFree(d_work);
  };
  cudaError_t e = cudaMalloc(&d_phi, phi.size() * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_r, static_cast<size_t>(M) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_hyp, static_cast<size_t>(n_set) * (d + 2) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_out, static_cast<size_t>(n_set) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&d_work, work * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_phi, phi.data(), phi.size() * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_r, s->fit.r.data(), static_cast<size_t>(M) * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_hyp, hyp, static_cast<size_t>(n_set) * (d + 2) * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    lml_kernel<<<grid, LML_THREADS, (2 * static_cast<size_t>(M) + d) * sizeof(double), st>>>(
        d_phi, d_r, M, d, s->H.kernel, d_hyp, n_set, d_work, d_out);
    e = cudaGetLastError();
    ++s->n_launches;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(lml_out, d_out, static_cast<size_t>(n_set) * 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  release();
  if (e != cudaSuccess) return fail(AS_ERR_CUDA, std::string("gp_lml: ") + cudaGetErrorString(e));
  return AS_OK;
}

namespace {
// hyper-parameters -> host feature tables and their device copies
as_status apply_gp_hyper(as_space* s, const double* lengthscale, double sf2, double sn2) {
  s->H.ls.assign(lengthscale, lengthscale + s->H.d);
  s->H.sf2 = sf2;
  s->H.sn2 = sn2;
  feature_tables(s->H);
  if (s->device >= 0) {
    CUDA_TRY(cudaSetDevice(s->device));
    CUDA_TRY(cudaMemcpy(const_cast<double*>(s->D.xt64), s->H.xt64.data(), s->H.xt64.size() * sizeof(double), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(const_cast<float*>(s->D.xt32), s->H.xt32.data(), s->H.xt32.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  return AS_OK;
}
}  // namespace

as_status autoscout_set_gp_hyper(as_space* s, const double* lengthscale, double sf2, double sn2) {
  if (!s || !lengthscale) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  for (int j = 0; j < s->H.d; ++j)
    if (!(lengthscale[j] > 0.0) || !std::isfinite(lengthscale[j])) return fail(AS_ERR_INVALID_ARG, "lengthscale must be > 0");
  if (!(sf2 > 0.0) || !(sn2 > 0.0) || !std::isfinite(sf2) || !std::isfinite(sn2))
    return fail(AS_ERR_INVALID_ARG, "sf2 and sn2 must be finite and > 0");
  const std::vector<double> old_ls = s->H.ls;
  const double old_sf2 = s->H.sf2, old_sn2 = s->H.sn2;
  const std::vector<uint64_t> raws = s->obs_raw;
  const std::vector<double> costs = s->obs_cost;
  const bool async0 = s->async_observe;   // the refit below must report its error here (synchronous)
  s->async_observe = false;
  as_status r = apply_gp_hyper(s, lengthscale, sf2, sn2);
  // refit the current observed set under the new hyper-parameters (observe_clear + observe)
  if (r == AS_OK) r = autoscout_observe_clear(s);
  if (r == AS_OK && !raws.empty())
    r = autoscout_observe(s, raws.data(), costs.data(), static_cast<int64_t>(raws.size()), nullptr);
  if (r != AS_OK) {
    // e.g. AS_ERR_NUMERIC from the Cholesky: restore the previous hyper-parameters and the
    // previous fit of the same observations (which succeeded before), keep the error
    const std::string why = g_err;
    apply_gp_hyper(s, old_ls.data(), old_sf2, old_sn2);
    autoscout_observe_clear(s);
    if (!raws.empty()) autoscout_observe(s, raws.data(), costs.data(), static_cast<int64_t>(raws.size()), nullptr);
    g_err = why;
  }
  s->async_observe = async0;
  return r;
}

namespace {
// ML-II candidate h (R21): h = 0 is the current setting; h > 0 draws every coordinate
// log-uniformly from counter-based uniforms u = (splitmix64(seed ^ 0x3111 ^ (64 h + k)) >> 11) 2^-53:
// l_j in [0.1, 10], sf2 in [1e-3, 10], sn2 / sf2 in [1e-6, 1e-1].
void ml2_candidate(const HostSpace& H, uint64_t seed, int h, double* out) {
  const int d = H.d;
  if (h == 0) {
    for (int j = 0; j < d; ++j) out[j] = H.ls[j];
    out[d] = H.sf2;
    out[d + 1] = H.sn2;
    return;
  }
  auto u = [&](int k) {
    return static_cast<double>(splitmix64(seed ^ 0x3111ull ^ (64ull * static_cast<uint64_t>(h) + static_cast<uint64_t>(k))) >> 11) *
           0x1.0p-53;
  };
  for (int j = 0; j < d; ++j) out[j] = std::exp(std::log(0.1) + u(j) * std::log(100.0));
  out[d] = std::exp(std::log(1e-3) + u(d) * std::log(1e4));
  out[d + 1] = out[d] * std::exp(std::log(1e-6) + u(d + 1) * std::log(1e5));
}
}  // namespace

as_status autoscout_ml2(as_space* s, int32_t n_set, uint64_t seed, int32_t apply, double* best_hyp_out,
                        double* best_lml_out, int32_t* best_index_out, void* cuda_stream) {
  if (!s || n_set < 1) return fail(AS_ERR_INVALID_ARG, "n_set must be >= 1");
  if (const as_status jr = join_fit(s, static_cast<cudaStream_t>(cuda_stream))) return jr;
  const int d = s->H.d;
  std::vector<double> hyp(static_cast<size_t>(n_set) * (d + 2)), lml(n_set);
  for (int h = 0; h < n_set; ++h) ml2_candidate(s->H, seed, h, hyp.data() + static_cast<size_t>(h) * (d + 2));
  as_status r = autoscout_gp_lml(s, hyp.data(), n_set, lml.data(), cuda_stream);
  if (r != AS_OK) return r;
  int best = 0;
  for (int h = 1; h < n_set; ++h)
    if (lml[h] > lml[best]) best = h;          // ties / NaN: the lowest index stays
  if (best_hyp_out) std::copy(hyp.begin() + static_cast<size_t>(best) * (d + 2), hyp.begin() + static_cast<size_t>(best + 1) * (d + 2), best_hyp_out);
  if (best_lml_out) *best_lml_out = lml[best];
  if (best_index_out) *best_index_out = best;
  if (apply && best != 0) {
    const double* b = hyp.data() + static_cast<size_t>(best) * (d + 2);
    return autoscout_set_gp_hyper(s, b, b[d], b[d + 1]);
  }
  return AS_OK;
}

as_status autoscout_prior(const as_space* s, uint64_t raw, double* m0_out, int32_t* source_out) {
  if (!s || !m0_out) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  int dig[DMAX];
  DV dv;
  uint32_t act;
  bool structural;
  if (!raw_decode(s->H, raw, dig, dv, act, structural)) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  if (s->ens.on) {
    *m0_out = ensemble_m0(s->H, s->ens, dv);
  } else {
    double c, mem;
    bool ok;
    simulate_host(s->H, dv, act, c, ok, mem);
    *m0_out = std::log(c);
  }
  if (source_out) *source_out = s->ens.on ? 1 : 0;
  return AS_OK;
}

as_status autoscout_ensemble_info(const as_space* s, double* r2_out, double* w_out, int32_t* available_out) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  for (int m = 0; m < 4; ++m) {
    if (r2_out) r2_out[m] = s->ens.r2[m];
    if (w_out) w_out[m] = s->ens.w[m];
  }
  if (available_out) *available_out = s->ens.on ? 1 : 0;
  return AS_OK;
}

as_status autoscout_raw_to_cvi(const as_space* s, uint64_t raw, uint64_t* cvi_out, int32_t* member_out) {
  if (!s || !cvi_out) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (raw >= s->H.n_raw) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  bool m = false;
  *cvi_out = cvi_rank(s->H, raw, &m);
  if (member_out) *member_out = m ? 1 : 0;
  return AS_OK;
}

as_status autoscout_subtree_range(const as_space* s, const int32_t* digits, int32_t n_assigned,
                                  uint64_t* begin_out, uint64_t* count_out) {
  if (!s || !begin_out || !count_out || (n_assigned > 0 && !digits)) return fail(AS_ERR_INVALID_ARG, "null argument");
  const HostSpace& H = s->H;
  if (n_assigned < 0 || n_assigned > H.d) return fail(AS_ERR_INVALID_ARG, "n_assigned outside [0, d]");
  uint64_t lo = 0;
  for (int f = 0; f < n_assigned; ++f) {
    if (digits[f] < 0 || digits[f] >= H.feat[f].n) return fail(AS_ERR_INVALID_ARG, "digit outside its domain");
    lo += static_cast<uint64_t>(digits[f]) * H.stride[f];
  }
  const uint64_t hi = lo + (n_assigned > 0 ? H.stride[n_assigned - 1] : H.n_raw);
  const uint64_t b = cvi_rank(H, lo, nullptr), e = cvi_rank(H, hi, nullptr);
  *begin_out = b;
  *count_out = e - b;
  return AS_OK;
}

as_status autoscout_neighbors(const as_space* s, uint64_t raw, uint64_t* cvi_out, int32_t cap, int32_t* n_out) {
  if (!s || !n_out || (cap > 0 && !cvi_out) || cap < 0) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  const HostSpace& H = s->H;
  if (raw >= H.n_raw) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  int dig[DMAX];
  bool act[DMAX];
  for (int f = 0; f < H.d; ++f) dig[f] = static_cast<int>((raw / H.stride[f]) % H.feat[f].n);
  activity(H, dig, act);
  int n = 0;
  for (int f = 0; f < H.d; ++f) {
    if (!H.feat[f].dense || !act[f]) continue;
    for (int step = 1; step < H.feat[f].n; step *= 2)
      for (int dir = 1; dir >= -1; dir -= 2) {
        const int nd = dig[f] + dir * step;
        if (nd < 0 || nd >= H.feat[f].n) continue;
        const uint64_t r2 = raw - static_cast<uint64_t>(dig[f]) * H.stride[f] + static_cast<uint64_t>(nd) * H.stride[f];
        bool m = false;
        const uint64_t pos = cvi_rank(H, r2, &m);
        if (!m) continue;
        if (n < cap) cvi_out[n] = pos;
        ++n;
      }
  }
  *n_out = n;
  if (n > cap) return fail(AS_ERR_CAPACITY, "more neighbours than cap");
  return AS_OK;
}

as_status autoscout_sample_to_cvi(const as_space* s, uint64_t seed, uint64_t ordinal, uint64_t* cvi_out) {
  if (!s || !cvi_out) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (ordinal >= s->H.n_cvi) return fail(AS_ERR_INDEX_RANGE, "ordinal >= n_cvi");
  *cvi_out = feistel_pi(feistel_make(s->H.n_cvi, seed), ordinal);
  return AS_OK;
}

as_status autoscout_simulate(const as_space* s, uint64_t raw, double* cost_out, double* mem_out, int32_t* ok_out) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  int dig[DMAX];
  DV dv;
  uint32_t act;
  bool structural;
  if (!raw_decode(s->H, raw, dig, dv, act, structural)) return fail(AS_ERR_INDEX_RANGE, "raw >= n_raw");
  double c, m;
  bool ok;
  simulate_host(s->H, dv, act, c, ok, m);
  if (cost_out) *cost_out = c;
  if (mem_out) *mem_out = m;
  if (ok_out) *ok_out = (ok && structural) ? 1 : 0;
  return AS_OK;
}

as_status autoscout_mask_range(as_space* s, uint64_t raw_begin, uint64_t count, uint32_t* d_bits,
                               uint64_t* d_valid_count, void* cuda_stream) {
  if (!s || (count > 0 && !d_bits)) return fail(AS_ERR_INVALID_ARG, "bad arguments");
  if (s->device < 0) return fail(AS_ERR_STATE, "host-only handle");
  if (raw_begin > s->H.n_raw || count > s->H.n_raw - raw_begin) return fail(AS_ERR_INDEX_RANGE, "range exceeds n_raw");
  if (count == 0) return AS_OK;
  CUDA_TRY(cudaSetDevice(s->device));
  const int threads = 256;
  const uint64_t blocks = (count + threads - 1) / threads;
  if (blocks > 0x7FFFFFFFull) return fail(AS_ERR_INVALID_ARG, "range too large for one launch");
  mask_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
      s->D, raw_begin, count, d_bits, d_valid_count);
  CUDA_TRY(cudaGetLastError());
  ++s->n_launches;
  return AS_OK;
}

as_status autoscout_set_path(as_space* s, int32_t path) {
  if (!s || path < 0 || path > 3)
    return fail(AS_ERR_INVALID_ARG, "path must be 0 (auto), 1 (SIMT), 2 (tensor cores) or 3 (tensor cores, one-hot r^2)");
  s->path = path;
  return AS_OK;
}

as_status autoscout_set_slice(as_space* s, uint64_t max_candidates) {
  if (!s || max_candidates < TC_ROWS || max_candidates > (1ull << 31))
    return fail(AS_ERR_INVALID_ARG, "slice must be in [128, 2^31] candidates");
  s->slice = max_candidates;
  return AS_OK;
}

as_status autoscout_set_async_observe(as_space* s, int32_t enable) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  if (const as_status jr = join_fit(s, nullptr)) return jr;
  s->async_observe = enable != 0;
  return AS_OK;
}

as_status autoscout_set_timing(as_space* s, int32_t enable) {
  if (!s) return fail(AS_ERR_INVALID_ARG, "null argument");
  s->timing = enable != 0 && s->device >= 0;
  s->ev_recorded = false;
  return AS_OK;
}

as_status autoscout_last_phase_ms(as_space* s, double* gen_ms, double* score_ms) {
  if (!s || !s->ev_recorded) return fail(AS_ERR_STATE, "no timed launch recorded");
  double g = 0, k = 0;
  for (int i = 0; i + 3 <= s->sev_used; i += 3) {
    float a = 0, b = 0;
    CUDA_TRY(cudaEventSynchronize(s->sev[i + 2]));
    CUDA_TRY(cudaEventElapsedTime(&a, s->sev[i], s->sev[i + 1]));
    CUDA_TRY(cudaEventElapsedTime(&b, s->sev[i + 1], s->sev[i + 2]));
    g += a;
    k += b;
  }
  if (gen_ms) *gen_ms = g;
  if (score_ms) *score_ms = k;
  return AS_OK;
}

as_status autoscout_last_kernel_ms(as_space* s, double* score_ms, double* merge_ms) {
  if (!s || !s->ev_recorded) return fail(AS_ERR_STATE, "no timed launch recorded");
  float a = 0, b = 0;
  CUDA_TRY(cudaEventSynchronize(s->ev[2]));
  CUDA_TRY(cudaEventElapsedTime(&a, s->ev[0], s->ev[1]));
  CUDA_TRY(cudaEventElapsedTime(&b, s->ev[1], s->ev[2]));
  if (score_ms) *score_ms = a;
  if (merge_ms) *merge_ms = b;
  return AS_OK;
}

}  // extern "C"
