// Tensor-core score kernel: the posterior contraction v = L^-1 k of 128-candidate
// tiles on tcgen05 (kind::tf32, 3xTF32 split, FP32 accumulators in TMEM), fed by SIMT producer
// warps that generate candidates from indices and compute the cross-covariance tile.
//
// Warp roles (544 threads, 1 CTA per SM):
//   warps 0-15  producers: decode + mask + simulator -> queue of valid candidates -> per tile of
//               128: k(x_c, o_j) in K-chunks of 16 observed points (4 per thread), split into
//               TF32 hi/lo and stored with tcgen05.st straight into a 4-stage A ring in TMEM (each
//               warp writes its own lane quadrant = its 32 candidates); then the epilogue of a
//               finished tile: tcgen05.ld of their TMEM lane quadrant (warp % 4) and column
//               quarter (warp / 4) -> ||v||^2 -> mu, FP32 acquisition + bound -> CTA top-k'.
//               TMEM = D accumulator(s) [NDB x Mp16 columns] + A ring [4 x 32 columns]; D is
//               double-buffered when it fits (M <= 192: epilogue of tile t-1 after producing t),
//               else single (epilogue of tile t right after producing it).
//   warp 16     MMA issuer + B loader (one thread): per K-chunk c, 3 MMAs x 2 k-steps into
//               D[:, 16c : Mp16) (triangular skipping: L^-1 has no entries above the diagonal);
//               bulk async copies of the host-pre-laid-out L^-1^T hi/lo chunks, 2 chunks ahead.
// No warp is idle by design: idle-waiting warps were measured to steal issue slots from the
// producers (profiles/r1_tc_*.md).
#pragma once
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace as {

constexpr int TC_ROWS = 128;                 // candidates per tile = TMEM lanes
constexpr int TC_KCH = 16;                   // observed points per K-chunk
constexpr int TC_NA = 4;                     // A ring stages
constexpr int TC_NB = 3;                     // B ring stages
constexpr int TC_TI = 2;                     // tile-info / meta slots
constexpr int TC_PW_MAX = 16;                // producer warps (template parameter PW in {8, 16})
constexpr int TC_QCAP = TC_ROWS - 1 + TC_PW_MAX * 32;
constexpr int TC_MAXCH = MMAX / TC_KCH;
constexpr int TC_EPI_WARPS = 4;              // warps that finalise rows (rows 0..127)

struct TcB {
  const float* chunks;          // all chunks back to back: [hi (N_c x 16)][lo (N_c x 16)] per chunk
  uint32_t off[TC_MAXCH];       // float offset of chunk c
  int nch;                      // Mp16 / 16
  int Mp16;                     // M padded to 16
  int ndb;                      // TMEM accumulator buffers (2 if 2*Mp16 + 32*NA <= 512, else 1)
  uint32_t tmem_cols;           // allocation (power of two >= ndb*Mp16 + 32*NA)
  double* scratch;              // [grid][4][Mp16] FP64 scratch of the sensitive-output fallback
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Top-k' admission among the `nt` threads synchronised by named barrier `id`.
__device__ __forceinline__ void group_bitonic(uint64_t* arr, int n_el, int t, int nt, int id) {
  for (int k = 2; k <= n_el; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < (n_el >> 1); i += nt) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo | j;
        const bool asc = (lo & k) == 0;
        const uint64_t a = arr[lo], b = arr[hi];
        if ((a > b) == asc) {
          arr[lo] = b;
          arr[hi] = a;
        }
      }
      named_sync(id, nt);
    }
}

__device__ __forceinline__ void group_admit(uint64_t key, uint64_t* arr, TopkSmem& ts, int KC, int t, int nt, int id) {
  if (key != KEY_NONE) {
    if (key < ts.tau) {
      const int pos = atomicAdd(&ts.n_add, 1);
      arr[ts.n_list + pos] = key;
    } else {
      atomicMin(reinterpret_cast<unsigned long long*>(&ts.drop), static_cast<unsigned long long>(key));
    }
  }
  named_sync(id, nt);
  const int n_add = ts.n_add;
  if (n_add > 0) {
    const int n_tot = ts.n_list + n_add;
    group_bitonic(arr, next_pow2(n_tot < 2 ? 2 : n_tot), t, nt, id);
    const int keep = n_tot < KC ? n_tot : KC;
    if (t == 0) {
      if (n_tot > KC && arr[KC] < ts.drop) ts.drop = arr[KC];
      ts.n_list = keep;
      ts.tau = (keep == KC) ? arr[KC - 1] : KEY_NONE;
      ts.n_add = 0;
    }
    for (int i = keep + t; i < n_tot; i += nt) arr[i] = KEY_NONE;
    named_sync(id, nt);
  }
}

struct TcSmem {
  float* B0;                // B ring: stage s at B0 + s b_stage (hi then lo)
  float* O;                 // [Mp16][DP]
  float* alpha;
  float* aabs;
  float* xt;
  DV* q_dv;
  double* q_m0;
  uint32_t* q_cvi;
  uint32_t* q_j;
  uint32_t* m_cvi;          // [TI][128]
  uint32_t* m_j;
  double* m_m0;
  float* m_part;            // [TI][3][128]  mu, sb, kk sums (atomically reduced over the JQ groups)
  float* vpart;             // [JQ][128] ||v||^2 partials of the column groups
  uint64_t* arr;            // top-k' [P]
  uint64_t* bars;           // mbarriers
  uint64_t* cidx;           // coarse structure index [CI]
};

// NF4 = feature width in float4 units (d padded to 4); compile-time so the r^2 loop has no guards.
// PW = producer warps (8 or 16): PW*32/128 threads share a candidate, each computes TC_KCH*128/(PW*32)
// observed points per K-chunk.
template <int NF4, int PW, int KT>
__global__ void __launch_bounds__(PW * 32 + 32, 1)
score_tc_kernel(DevSpace S, DevGP G, BatchArgs A, CtaOut out, TcB TB) {
  constexpr int TC_PROD_WARPS = PW;
  constexpr int TC_PROD_THREADS = PW * 32;
  constexpr int TC_THREADS = TC_PROD_THREADS + 32;
  constexpr int TC_MMA_WARP = PW;
  constexpr int TC_JQ = TC_PROD_THREADS / TC_ROWS;   // producer threads per candidate
  constexpr int TC_JPT = TC_KCH / TC_JQ;             // observed points per thread per chunk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ TopkSmem ts;
  __shared__ int q_n;
  __shared__ int tinfo[TC_TI];
  __shared__ uint32_t tmem_base;
  __shared__ unsigned long long valid_cta;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Mp16 = TB.Mp16, DP = G.DP, nch = TB.nch;
  const int NDB = TB.ndb;
  const uint32_t A0col = static_cast<uint32_t>(NDB * Mp16);      // TMEM column of A stage 0
  const uint32_t b_stage_bytes = 2u * Mp16 * TC_KCH * 4;         // hi + lo at the widest chunk
  TcSmem sm;
  unsigned char* p = smem_raw;
  auto take = [&](size_t bytes) {
    unsigned char* r = p;
    p += (bytes + 127) & ~size_t(127);
    return r;
  };
  sm.B0 = reinterpret_cast<float*>(take(static_cast<size_t>(TC_NB) * b_stage_bytes));
  const uint32_t sB0 = tc::smem_u32(sm.B0);
  sm.O = reinterpret_cast<float*>(take(sizeof(float) * Mp16 * DP));
  sm.alpha = reinterpret_cast<float*>(take(sizeof(float) * 2 * Mp16));   // (alpha_j, |alpha_j|) pairs
  sm.aabs = nullptr;
  sm.xt = reinterpret_cast<float*>(take(sizeof(float) * S.d * VMAX));
  sm.q_dv = reinterpret_cast<DV*>(take(sizeof(DV) * TC_QCAP));
  sm.q_m0 = reinterpret_cast<double*>(take(sizeof(double) * TC_QCAP));
  sm.q_cvi = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * TC_QCAP));
  sm.q_j = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * TC_QCAP));
  sm.m_cvi = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * TC_TI * TC_ROWS));
  sm.m_j = reinterpret_cast<uint32_t*>(take(sizeof(uint32_t) * TC_TI * TC_ROWS));
  sm.m_m0 = reinterpret_cast<double*>(take(sizeof(double) * TC_TI * TC_ROWS));
  sm.m_part = reinterpret_cast<float*>(take(sizeof(float) * TC_TI * 3 * TC_ROWS));
  sm.vpart = reinterpret_cast<float*>(take(sizeof(float) * 4 * TC_ROWS));   // sized for TC_JQ <= 4
  sm.arr = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * out.P));
  sm.bars = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * 32));
  sm.cidx = reinterpret_cast<uint64_t*>(take(sizeof(uint64_t) * CI));
  uint64_t* a_full = sm.bars;                 // [NA] count 16 (producer warps)
  uint64_t* a_empty = a_full + TC_NA;         // [NA] count 1 (commit)
  uint64_t* b_full = a_empty + TC_NA;         // [NB] count 1 + tx
  uint64_t* b_empty = b_full + TC_NB;         // [NB] count 1 (commit)
  uint64_t* d_full = b_empty + TC_NB;         // [2]  count 1 (commit)
  uint64_t* d_empty = d_full + 2;             // [2]  count 16 (producer warps)
  uint64_t* t_ready = d_empty + 2;            // [TI] count 1 (producer leader)

  // ---- setup: stage observed set + tables, init barriers, allocate TMEM
  for (int i = tid; i < Mp16 * DP; i += TC_THREADS) sm.O[i] = (i < G.Mp * DP) ? __ldg(G.O + i) : 0.f;
  for (int i = tid; i < Mp16; i += TC_THREADS) {
    sm.alpha[2 * i] = i < G.Mp ? __ldg(G.alpha + i) : 0.f;
    sm.alpha[2 * i + 1] = i < G.Mp ? __ldg(G.aabs + i) : 0.f;
  }
  for (int i = tid; i < S.d * VMAX; i += TC_THREADS) sm.xt[i] = __ldg(S.xt32 + i);
  for (int i = tid; i < out.P; i += TC_THREADS) sm.arr[i] = KEY_NONE;
  load_cidx(S, sm.cidx, tid, TC_THREADS);
  if (tid == 0) {
    for (int s = 0; s < TC_NA; ++s) {
      tc::mbar_init(a_full + s, TC_PROD_WARPS);
      tc::mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < TC_NB; ++s) {
      tc::mbar_init(b_full + s, 1);
      tc::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(d_full + s, 1);
      tc::mbar_init(d_empty + s, TC_PROD_WARPS);
    }
    for (int s = 0; s < TC_TI; ++s) tc::mbar_init(t_ready + s, 1);
    tc::mbar_fence_init();
    ts.n_list = 0;
    ts.n_add = 0;
    ts.tau = KEY_NONE;
    ts.drop = KEY_NONE;
    q_n = 0;
    valid_cta = 0;
  }
  const uint32_t tmem_cols = TB.tmem_cols;
  if (warp == 0) tc::tmem_alloc(&tmem_base, tmem_cols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;

  if (warp < TC_PROD_WARPS) {
    // =========================================================== producers (+ epilogue)
    const int pt = tid;                              // 0..511
    const int cand = pt & (TC_ROWS - 1);             // candidate row of the tile
    const int jq = pt >> 7;                          // observed-point group of a chunk (warp-uniform)
    const int quad = warp & 3;                       // TMEM lane quadrant of this warp
    const uint32_t sO = tc::smem_u32(sm.O), sAl = tc::smem_u32(sm.alpha);
    // k = sf2 poly(a) exp(-a):  exp2 argument folds ln(sf2):  -a log2(e) + log2(sf2)
    const float ex_c1 = (KT == 0) ? -2.2360679774997896f * 1.4426950408889634f : -0.5f * 1.4426950408889634f;
    const float ex_c0 = log2f(G.sf2f);
    const uint32_t a_off = tc::kmajor_off(cand, jq * TC_JPT, TC_KCH / 4);   // + 128 B per further 4 points
    double* scratch = TB.scratch + (static_cast<size_t>(blockIdx.x) * TC_EPI_WARPS + (warp & 3)) * Mp16;

    // Epilogue of tile u.  Column block b = [16b, 16b+16) of the accumulator is final once chunk b's
    // MMAs completed (triangular: later chunks only write columns >= 16(b+1)); the producers already
    // read blocks b < nch - NA during the chunk loop (vsq_run), so only the last NA blocks wait for
    // the tile's final commit.
    auto epilogue = [&](int u, float vsq_run) {
      const int us = u % TC_TI, buf = u % NDB;
      tc::mbar_wait(d_full + buf, (u / NDB) & 1);
      tc::fence_after_sync();
      float vsq = vsq_run;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quad * 32) << 16) + buf * Mp16 + TC_JPT * jq;
      for (int b = (nch > TC_NA ? nch - TC_NA : 0); b < nch; ++b) {
#pragma unroll
        for (int h = 0; h < TC_JPT; h += 4) {
          float v[4];
          tc::tmem_ld4(taddr + 16 * b + h, v);
          vsq = fmaf(v[0], v[0], fmaf(v[1], v[1], fmaf(v[2], v[2], fmaf(v[3], v[3], vsq))));
        }
      }
      sm.vpart[jq * TC_ROWS + quad * 32 + lane] = vsq;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(d_empty + buf);
      named_sync(1, TC_PROD_THREADS);
      const int n = tinfo[us];
      uint64_t key = KEY_NONE;
      bool sensitive = false;
      if (pt < TC_ROWS && pt < n) {
        const int row = pt;
        const float* mp = sm.m_part + us * 3 * TC_ROWS;
        const float mu32 = mp[0 * TC_ROWS + row], sb = mp[1 * TC_ROWS + row], kk = mp[2 * TC_ROWS + row];
        float vv = 0.f;
#pragma unroll
        for (int q = 0; q < TC_JQ; ++q) vv += sm.vpart[q * TC_ROWS + row];
        const double cm0 = sm.m_m0[us * TC_ROWS + row];
        const float mu = static_cast<float>(cm0 + G.b) + mu32;
        const float vs = vv;
        const float s2 = static_cast<float>(G.sf2) - vs;
        // FP32 SIMT k + 3xTF32 contraction: error coefficient 8x the SIMT one
        const float eps = 8.0f * static_cast<float>(G.eps);
        const float d_mu = eps * sb + 2e-7f * (1.0f + fabsf(mu));
        const float ew = eps * static_cast<float>(G.w_fro);
        const float d_s2 = 2.5f * ew * sqrtf(vs) * sqrtf(kk) + ew * ew * kk + eps * vs + 8.0f * U32 * G.sf2f;
        const float fstar = static_cast<float>(G.fstar), m0f = static_cast<float>(cm0);
        float m1, m2;
        const float sc = acquisition32(A.acq, mu, s2, m0f, fstar, static_cast<float>(A.xi), static_cast<float>(A.kappa), m1);
        float ub = acquisition32(A.acq, mu - d_mu, s2 + d_s2, m0f, fstar, static_cast<float>(A.xi),
                                 static_cast<float>(A.kappa), m2);
        ub += m2;
        if (A.d_scores) {
          // per-candidate output: FP64 acquisition (and FP64 posterior where FP32 is too sensitive)
          const double mud = cm0 + G.b + static_cast<double>(mu32);
          const double s2d = G.sf2 - static_cast<double>(vv);
          if (A.acq == 0) {
            if (s2d > 0.0) {
              const double sg = sqrt(s2d), z = (G.fstar - mud - A.xi) / sg;
              if (z >= -3.2) {
                const double Phi = 0.5 * erfc(-z * INV_SQRT2);
                const double h = exp(-0.5 * z * z) * INV_SQRT_2PI + z * Phi;
                const double uu = static_cast<double>(U32);
                const double e_s = (1.0 - z * Phi / h) / (2.0 * s2d) * 160.0 * uu * static_cast<double>(vv) +
                                   Phi / (sg * h) * uu * (1.0 + static_cast<double>(sb));
                sensitive = e_s > 5e-6;
              }
            } else {
              sensitive = true;
            }
          }
          if (!sensitive)
            A.d_scores[sm.m_j[us * TC_ROWS + row]] =
                static_cast<float>(acquisition(A.acq, mud, s2d, cm0, G.fstar, A.xi, A.kappa));
        }
        if (!sensitive && ub > -INFINITY) key = make_key(ub, sm.m_cvi[us * TC_ROWS + row]);
        (void)sc;
      }
      if (warp < TC_EPI_WARPS) {
        // warp-cooperative FP64 posterior for the flagged rows of this warp (d_scores mode only)
        unsigned fl = __ballot_sync(0xffffffffu, sensitive);
        while (fl) {
          const int src = __ffs(fl) - 1;
          fl &= fl - 1;
          const int row = warp * 32 + src;
          const uint32_t cvi = sm.m_cvi[us * TC_ROWS + row];
          DV dv;
          uint32_t act;
          uint64_t raw;
          decode_dev(S, cvi, dv, act, raw);
          double kalpha, vq;
          posterior64_warp(S, G, dv, lane, scratch, kalpha, vq);
          if (lane == src) {
            const double cm0 = sm.m_m0[us * TC_ROWS + row];
            const double sc = acquisition(A.acq, cm0 + G.b + kalpha, G.sf2 - vq, cm0, G.fstar, A.xi, A.kappa);
            const double ub = sc + 1e-12 * fmax(1.0, fabs(sc));
            A.d_scores[sm.m_j[us * TC_ROWS + row]] = static_cast<float>(sc);
            if (ub > -INFINITY) key = make_key(__double2float_ru(ub), cvi);
          }
        }
      }
      group_admit(key, sm.arr, ts, out.KC, pt, TC_PROD_THREADS, 1);
    };

    const uint64_t ntiles = (A.count + TC_PROD_THREADS - 1) / TC_PROD_THREADS;
    uint32_t g = 0;                                   // global A-chunk counter
    int t = 0;                                        // tile counter
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      // ---- phase 0: index -> configuration -> validity -> simulator -> queue
      const uint64_t j = tile * TC_PROD_THREADS + pt;
      const bool in = j < A.count;
      bool ok = false;
      if (in) {
        bool pin;
        const uint64_t pcvi = assign_pos(A, j, pin);
        DV dv;
        uint32_t act;
        uint64_t raw;
        decode_dev_idx(S, sm.cidx, pcvi, dv, act, raw);
        double cost;
        sim_dev(S, dv, act, cost, ok);
        if (!pin) {
          ok = false;
          raw = ~0ull;
        }
        if (A.d_raw) A.d_raw[j] = raw;
        if (!ok && A.d_scores) A.d_scores[j] = -INFINITY;
        if (ok) {
          const int slot = atomicAdd(&q_n, 1);
          sm.q_dv[slot] = dv;
          sm.q_m0[slot] = prior_m0(S, dv, cost);
          sm.q_cvi[slot] = static_cast<uint32_t>(pcvi);
          sm.q_j[slot] = static_cast<uint32_t>(j);
        }
      }
      const unsigned vb = __ballot_sync(0xffffffffu, in && ok);
      if (lane == 0 && vb) atomicAdd(&valid_cta, static_cast<unsigned long long>(__popc(vb)));
      named_sync(1, TC_PROD_THREADS);
      const bool last_tile = tile + gridDim.x >= ntiles;
      int head = 0;
      while (true) {
        const int avail = q_n - head;
        const int n = avail >= TC_ROWS ? TC_ROWS : (last_tile ? avail : 0);
        if (n <= 0) break;
        // ---- publish tile t: meta + tile info
        const int ts_ = t % TC_TI;
        if (pt < TC_ROWS) {
          float* mz = sm.m_part + ts_ * 3 * TC_ROWS;
          mz[pt] = 0.f;
          mz[TC_ROWS + pt] = 0.f;
          mz[2 * TC_ROWS + pt] = 0.f;
        }
        if (pt < n) {
          sm.m_cvi[ts_ * TC_ROWS + pt] = sm.q_cvi[head + pt];
          sm.m_j[ts_ * TC_ROWS + pt] = sm.q_j[head + pt];
          sm.m_m0[ts_ * TC_ROWS + pt] = sm.q_m0[head + pt];
        }
        unsigned long long xp[2 * NF4];
        const bool has = cand < n;
        {
          DV cdv;
          cdv.w[0] = cdv.w[1] = cdv.w[2] = 0;
          if (has) cdv = sm.q_dv[head + cand];
#pragma unroll
          for (int f = 0; f < 4 * NF4; f += 2) {
            const float a = (has && f < S.d) ? sm.xt[f * VMAX + dv_get(cdv, f)] : 0.f;
            const float b = (has && f + 1 < S.d) ? sm.xt[(f + 1) * VMAX + dv_get(cdv, f + 1)] : 0.f;
            xp[f / 2] = f2_pack(a, b);
          }
        }
        named_sync(1, TC_PROD_THREADS);
        if (pt == 0) {
          tinfo[ts_] = n;
          tc::mbar_arrive(t_ready + ts_);
        }
        // ---- cross-covariance chunks -> A ring
        float mu_p = 0.f, sb_p = 0.f, kk_p = 0.f, vsq_run = 0.f;
        const uint32_t dq = tmem + (static_cast<uint32_t>(quad * 32) << 16) + (t % NDB) * Mp16 + TC_JPT * jq;
        for (int c = 0; c < nch; ++c, ++g) {
          const int s = g % TC_NA;
          const uint32_t a_par = ((g / TC_NA) & 1u) ^ 1u;
          const bool a_ready = tc::mbar_test(a_empty + s, a_par);   // result consumed after the math
          float kh[TC_JPT], kl[TC_JPT];
#pragma unroll
          for (int q = 0; q < TC_JPT; ++q) {
            // rows >= M of the observed set are zero padded with alpha = 0 and L^-1 columns = 0; rows of
            // an incomplete tile (cand >= n) compute finite values that are never read back
            const int jo = c * TC_KCH + jq * TC_JPT + q;      // warp-uniform
            unsigned long long acc0 = 0ull, acc1 = 0ull;
            const uint32_t orow = sO + static_cast<uint32_t>(jo * NF4 * 16);
#pragma unroll
            for (int f4 = 0; f4 < NF4; ++f4) {
              unsigned long long ox, oy;
              tc::lds_u64x2(orow + 16 * f4, ox, oy);
              const unsigned long long d0 = f2_sub(xp[2 * f4], ox), d1 = f2_sub(xp[2 * f4 + 1], oy);
              acc0 = f2_fma(d0, d0, acc0);
              acc1 = f2_fma(d1, d1, acc1);
            }
            const float2 rs = f2_unpack(f2_add(acc0, acc1));
            const float r2 = rs.x + rs.y;
            float arg, poly, ex;
            if (KT == 0) {
              const float r = tc::sqrt_approx_ftz(r2);
              arg = 2.2360679774997896f * r;
              poly = fmaf(arg, fmaf(arg, 0.33333333333333333f, 1.0f), 1.0f);
              ex = tc::ex2_approx(fmaf(r, ex_c1, ex_c0));
            } else {
              arg = 0.5f * r2;
              poly = 1.0f;
              ex = tc::ex2_approx(fmaf(r2, ex_c1, ex_c0));
            }
            const float kval = poly * ex;
            const float cc = fmaf(kval, arg, kval);           // k (1 + a)
            float al, aa;
            tc::lds_f32x2(sAl + 8 * jo, al, aa);
            mu_p = fmaf(kval, al, mu_p);
            sb_p = fmaf(cc, aa, sb_p);
            kk_p = fmaf(cc, cc, kk_p);
            tc::split_tf32_fast(kval, kh[q], kl[q]);
          }
          if (!a_ready) tc::mbar_wait(a_empty + s, a_par);
          tc::fence_after_sync();
          if (c >= TC_NA) {
            // chunk c - NA of this tile completed (its A stage was released): its column block is final
#pragma unroll
            for (int h = 0; h < TC_JPT; h += 4) {
              float v[4];
              tc::tmem_ld4(dq + 16 * (c - TC_NA) + h, v);
              vsq_run = fmaf(v[0], v[0], fmaf(v[1], v[1], fmaf(v[2], v[2], fmaf(v[3], v[3], vsq_run))));
            }
          }
          const uint32_t acol = tmem + (static_cast<uint32_t>(quad * 32) << 16) + A0col + 32u * s + jq * TC_JPT;
#pragma unroll
          for (int v4 = 0; v4 < TC_JPT / 4; ++v4) {
            tc::tmem_st4(acol + 4 * v4, kh[4 * v4], kh[4 * v4 + 1], kh[4 * v4 + 2], kh[4 * v4 + 3]);
            tc::tmem_st4(acol + 16 + 4 * v4, kl[4 * v4], kl[4 * v4 + 1], kl[4 * v4 + 2], kl[4 * v4 + 3]);
          }
          tc::tmem_st_wait();
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(a_full + s);
        }
        float* mp = sm.m_part + ts_ * 3 * TC_ROWS;
        atomicAdd(mp + cand, mu_p);
        atomicAdd(mp + TC_ROWS + cand, sb_p);
        atomicAdd(mp + 2 * TC_ROWS + cand, kk_p);
        // ---- epilogue of this tile (only the last NA column blocks still wait for the MMAs)
        epilogue(t, vsq_run);
        named_sync(1, TC_PROD_THREADS);
        head += n;
        ++t;
      }
      // ---- compact the queue: leftovers (< 128) to the front
      const int left = q_n - head;
      named_sync(1, TC_PROD_THREADS);
      DV mdv;
      double mm0 = 0;
      uint32_t mcvi = 0, mj = 0;
      if (pt < left) {
        mdv = sm.q_dv[head + pt];
        mm0 = sm.q_m0[head + pt];
        mcvi = sm.q_cvi[head + pt];
        mj = sm.q_j[head + pt];
      }
      named_sync(1, TC_PROD_THREADS);
      if (pt < left) {
        sm.q_dv[pt] = mdv;
        sm.q_m0[pt] = mm0;
        sm.q_cvi[pt] = mcvi;
        sm.q_j[pt] = mj;
      }
      if (pt == 0) q_n = left;
      named_sync(1, TC_PROD_THREADS);
    }
    // ---- end of stream
    if (pt == 0) {
      const int ts_ = t % TC_TI;
      tinfo[ts_] = -1;
      tc::mbar_arrive(t_ready + ts_);
    }
    // ---- CTA list
    named_sync(1, TC_PROD_THREADS);
    const int n = ts.n_list;
    uint64_t* dst = out.lists + static_cast<size_t>(blockIdx.x) * out.KC;
    for (int i = pt; i < n; i += TC_PROD_THREADS) dst[i] = sm.arr[i];
    if (pt == 0) {
      out.counts[blockIdx.x] = n;
      out.drop[blockIdx.x] = ts.drop;
    }
  } else {
    // =========================================================== MMA issuer + B loader
    if (lane == 0) {
      uint32_t g = 0, gl = 0;                        // consumed chunks, loaded chunks (global counters)
      auto load_next = [&]() {
        const int s = gl % TC_NB;
        tc::mbar_wait(b_empty + s, ((gl / TC_NB) & 1u) ^ 1u);
        const int c = gl % nch;
        const uint32_t bytes = 2u * (Mp16 - c * TC_KCH) * TC_KCH * 4;
        tc::mbar_arrive_expect_tx(b_full + s, bytes);
        tc::bulk_g2s(sm.B0 + static_cast<size_t>(s) * (b_stage_bytes / 4), TB.chunks + TB.off[c], bytes, b_full + s);
        ++gl;
      };
      bool primed = false;
      for (int t = 0;; ++t) {
        const int ts_ = t % TC_TI;
        tc::mbar_wait(t_ready + ts_, (t / TC_TI) & 1);
        if (tinfo[ts_] < 0) break;
        if (!primed) {
          for (int i = 0; i < TC_NB - 1; ++i) load_next();
          primed = true;
        }
        const int buf = t % NDB;
        tc::mbar_wait(d_empty + buf, ((t / NDB) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t dcol = tmem + buf * Mp16;
        for (int c = 0; c < nch; ++c, ++g) {
          const int sa = g % TC_NA, sbb = g % TC_NB;
          tc::mbar_wait(a_full + sa, (g / TC_NA) & 1);
          tc::mbar_wait(b_full + sbb, (g / TC_NB) & 1);
          tc::fence_after_sync();
          const int N = Mp16 - c * TC_KCH;
          const uint32_t idesc = tc::idesc_tf32(TC_ROWS, N);
          const uint32_t a_h = tmem + A0col + 32u * sa, a_l = a_h + 16;
          const uint32_t b_h = sB0 + sbb * b_stage_bytes;
          const uint32_t b_l = b_h + N * TC_KCH * 4;
          const uint32_t sbo = (TC_KCH / 4) * 128;
#pragma unroll
          for (int ks = 0; ks < TC_KCH / 8; ++ks) {
            const uint64_t bh = tc::sdesc(b_h + 256 * ks, 128, sbo), bl = tc::sdesc(b_l + 256 * ks, 128, sbo);
            const uint32_t d = dcol + c * TC_KCH;
            tc::mma_tf32_ts(d, a_h + 8 * ks, bh, idesc, (c > 0 || ks > 0) ? 1u : 0u);
            tc::mma_tf32_ts(d, a_h + 8 * ks, bl, idesc, 1u);
            tc::mma_tf32_ts(d, a_l + 8 * ks, bh, idesc, 1u);
          }
          tc::mma_commit(a_empty + sa);
          tc::mma_commit(b_empty + sbb);
          load_next();                               // refill the slot of chunk g-1, 2 chunks ahead
        }
        tc::mma_commit(d_full + buf);
      }
      // drain bulk copies still in flight before the CTA exits
      while (g < gl) {
        tc::mbar_wait(b_full + (g % TC_NB), (g / TC_NB) & 1);
        ++g;
      }
    }
    __syncwarp();
  }
  // ---- teardown
  tc::fence_before_sync();
  __syncthreads();
  if (tid == 0 && valid_cta) {
    atomicAdd(reinterpret_cast<unsigned long long*>(out.valid), valid_cta);
    if (A.d_valid_count) atomicAdd(reinterpret_cast<unsigned long long*>(A.d_valid_count), valid_cta);
  }
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, tmem_cols);
  }
}

}  // namespace as
