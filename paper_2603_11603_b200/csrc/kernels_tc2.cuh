// Tensor-core score kernel, second generation: both contractions of the posterior
// on tcgen05 —
//   (1) squared distances  R2 = E T^T  (kind::f16, FP32 accumulate): E is the one-hot digit encoding
//       of the 128 candidates of a tile (exact in FP16), T[j][(f,v)] = 2^s (xt_f[v] - o_jf)^2 split
//       into two FP16 pieces on the host.  All products are exact and every term is >= 0, so R2 has
//       FP32-accumulation error only (no cancellation); rows of E are built by the producers.
//       Features with many values (NH <= 4 of them, chosen on the host to keep the one-hot width
//       Kp <= 64) are added on the SIMT pipes instead: (x_f - o_jf)^2 in FP32, same 2^s scale.
//       One R2 MMA group covers 4 K-chunks (N = 64): per-instruction cost is flat below N = 64
//       (tools/mma_bench.cu), so wide groups are what keeps the tensor pipe and the issuing warp free.
//   (2) v = L^-1 k  (kind::f16, 3-term FP16 split hi.hi + hi.lo + lo.hi, FP32 accumulate): k is
//       produced scaled by 2^ek and split by mantissa mask (hi) + exact remainder (lo), stored to
//       TMEM as packed f16x2 (A operand from TMEM); L^-1^T chunks are host-split FP16 hi + lo.
// The producers therefore no longer evaluate sum_f (x_f - o_jf)^2 on the FP32 pipe (2 d FP32 ops
// per candidate x observed pair); they read R2 from TMEM and evaluate k(r) only.  Candidates come
// from the compact list of gen_kernel (kernels_gen.cuh): decode, mask and simulator run there.
//
// Warp roles (768 threads, 1 CTA per SM; registers rebalanced by setmaxnreg: producers 96, the
// other two warpgroups 48):
//   warps 0-15  producers: publish tile t+1 (meta + E rows + SIMT-feature values from the staged
//               list records) BEFORE the chunk loop of tile t, so the R2 MMAs of t+1 overlap tile t;
//               chunk loop: R2 group from TMEM -> k -> FP16 hi/lo -> A ring (TMEM); head start on
//               tile t+1; epilogue read (|v|^2 of the last column blocks), then tile t is handed to
//               the finalize warps through an mbarrier (f_ready) -- no CTA barrier.
//   warp 16     L^-1 MMA issuer (warp-converged, one elected lane issues).
//   warp 17     T loader: bulk copies of the T groups and the zero-fill of used one-hot buffers
//               (blocking waits in ring order).
//   warp 18     R2 MMA issuer.        warp 19  L^-1 chunk loader.
//   warps 20-23 finalize (one per SM sub-partition, row = 32 (warp - 20) + lane): FP32 screen +
//               certified bound, lazy CTA top-k' of tile t while the producers run tile t+1; they
//               release the tile's slots (partial sums, |v|^2, meta) through f_free, and lane 0 of
//               warp 20 stages the list records of tile t + 4.  The T loader waits in ring order
//               (blocking) instead of polling with back-off.
// TMEM: D [Mp16] | A ring [8 x 16] | R2 ring [2 groups x 64]  (Mp16 <= 256 -> <= 512 columns).
#pragma once
#include "kernels_gen.cuh"
#include "kernels_tc.cuh"

namespace as {

constexpr int TC2_RG = 4;                    // K-chunks per R2 group (N = 64)
constexpr int TC2_RS = 2;                    // R2 group slots in TMEM
constexpr int TC2_NA = 8;                    // A ring stages (16 TMEM columns each: FP16 hi | lo)
constexpr int TC2_NB = 6;                    // L^-1 chunk ring stages
constexpr int TC2_PF = TC2_NB - 2;           // chunks prefetched ahead of the MMA (L2 latency); a refill
                                             // waits for the MMAs two chunks back, not the previous one
constexpr int TC2_NT = 2;                    // T group ring stages (refilled early by the loader warp)
constexpr int TC2_KPMAX = 64;                // one-hot width the host aims for (features beyond go SIMT)
#ifndef AS_TC2_CB
#define AS_TC2_CB 1
#endif
constexpr int TC2_CB = AS_TC2_CB;                    // chunks whose math is batched ahead of their A-stage waits (ILP)
constexpr int TC2_XW = 8;                    // non-producer warps (MMA, loader, R2, L^-1 loader, 4 finalize)
constexpr int TC2_THREADS = 16 * 32 + TC2_XW * 32;
#ifndef AS_TC2_PREGS
#define AS_TC2_PREGS 96
#define AS_TC2_AREGS 48
#endif
constexpr int TC2_PROD_REGS = AS_TC2_PREGS;            // setmaxnreg: producers 96, the others 48 (80 at launch)
constexpr int TC2_AUX_REGS = AS_TC2_AREGS;

// Shared-memory carve-out: the fixed-size arrays first (compile-time offsets, so the hot loop
// addresses them with immediates), then the rings whose size depends on M and Kp.
constexpr size_t tc2_r128(size_t b) { return (b + 127) & ~size_t(127); }
// Slot counts: the M = 256 instance (BIG, one accumulator) needs 3 meta / 2 partial-sum / 2 staging
// slots with records staged 3 tiles ahead; lag mode (two accumulators, the epilogue one tile later)
// needs one more of each and stages 4 ahead.  The M = 256 layout is the one shared memory is tight for.
constexpr size_t TC2_STG_CVI = 0, TC2_STG_J = 512, TC2_STG_M0 = 1024, TC2_STG_DV0 = 2048, TC2_STG_DV1 = 3072,
                 TC2_STG_DV2 = 4096, TC2_STG_BYTES = 5120;
template <bool BIG>
struct Tc2L {
  static constexpr int TI = BIG ? 3 : 4;       // meta slots (cvi, j, m0): publish -> finalize
  static constexpr int PS = BIG ? 2 : 3;       // partial-sum slots (flush_part -> finalize)
  static constexpr int NS = BIG ? 2 : 3;       // staging slots of list records
  static constexpr int AHEAD = BIG ? 3 : 4;    // records of tile t + AHEAD staged after hand-off t
  static constexpr size_t BARS = 0;
  static constexpr size_t ALPHA = BARS + 64 * 8;
  static constexpr size_t OH = ALPHA + 2 * MMAX * 4;
  static constexpr size_t MXH = OH + 4 * MMAX * 4;
  static constexpr size_t MPART = MXH + 4 * TC_TI * TC_ROWS * 4;
  static constexpr size_t VPART = MPART + PS * 4 * 3 * TC_ROWS * 4;   // [PS][jq][3][128]: one slot per thread
  static constexpr size_t MCVI = VPART + 2 * 4 * TC_ROWS * 4;         // vpart: [2 slots][jq][128]
  static constexpr size_t MJ = MCVI + TI * TC_ROWS * 4;
  static constexpr size_t MM0 = MJ + TI * TC_ROWS * 4;
  static constexpr size_t XH = MM0 + TI * TC_ROWS * 8;
  static constexpr size_t STG = XH + 4 * VMAX * 4;                    // staged records: cvi | j | m0 | dv0-2
  static constexpr size_t VAR = tc2_r128(STG + NS * TC2_STG_BYTES);
};
// + NB L^-1 stages (2 Mp16 16 4 B) + NT T stages (2 64 Kp 2 B) + 2 E buffers (128 Kp 2 B) + P keys
__host__ __device__ constexpr size_t tc2_smem_total(int Mp16, int Kp, int P, bool big) {
  return (big ? Tc2L<true>::VAR : Tc2L<false>::VAR) + static_cast<size_t>(TC2_NB) * 2 * Mp16 * 16 * 2 +
         static_cast<size_t>(TC2_NT) * 2 * 64 * Kp * 2 + 2ull * 128 * Kp * 2 + static_cast<size_t>(P) * 8;
}

// Phase timeline of CTA 0 (development aid, off unless the host sets AS_TC2_TRACE): clock64 per
// (tile < TC2_TR_TILES, event, warp); written by lane 0 of each warp.
constexpr int TC2_TR_TILES = 64, TC2_TR_EV = 16, TC2_TR_W = 24;
__device__ unsigned long long* g_tc2_trace = nullptr;

struct Tc2B {
  const uint16_t* tch;          // T groups: [ng][2 pieces][64 x Kp] FP16, kmajor_off16 layout
  const float* xh;              // [NH][VMAX] 2^(s/2) xt of the SIMT features
  const float* oh;              // [Mp16][NH] 2^(s/2) o of the SIMT features (0 beyond M)
  int Kp;                       // one-hot width (sum of n_f over one-hot features) padded to 16
  int nh;                       // SIMT features (0, 2 or 4 after padding with a zero feature)
  int hf[4];                    // their feature indices (-1 = padding)
  float r2_scale;               // 2^-s    (R2 in TMEM is 2^s r^2)
  float r_scale;                // 2^-s/2
  int eoff[DMAX];               // one-hot column of digit 0 of feature f (-1: SIMT feature)
  // v = L^-1 k in kind::f16: k scaled by 2^ek and L^-1 by 2^ew, each split into FP16 hi + lo
  const uint16_t* ezero;        // >= 128 x Kp FP16 zeros: bulk-copied over a used E buffer by the loader
  const uint16_t* wch;          // L^-1^T chunks: chunk c = [hi (N_c x 16)][lo (N_c x 16)], kmajor_off16
  uint32_t woff[TC_MAXCH];      // element offset of chunk c
  int ek;                       // k scale exponent (kernel values leave the exp2 already scaled)
  float k_unscale;              // 2^-ek
  float vsq_unscale;            // 2^-2(ek + ew)
};

// Lazy top-k' admission (finalize() below): keys below the (possibly stale) threshold tau are
// appended to the unsorted tail of arr; the sort-and-prune to KC entries runs only when the next
// tile could overflow arr (P - 128 entries), and once at the end.  tau only ever tightens, so a
// stale tau admits more keys, never fewer; rejected keys lower drop exactly as in group_admit.
__device__ __forceinline__ void tc2_prune(uint64_t* arr, TopkSmem& ts, int KC, int t, int nt, int id) {
  const int n_tot = ts.n_list + ts.n_add;
  // every thread has read n_tot before thread 0 rewrites ts (bitonic's barriers, or this one when
  // there is nothing to sort -- compute-sanitizer racecheck)
  if (n_tot > 0) group_bitonic(arr, next_pow2(n_tot < 2 ? 2 : n_tot), t, nt, id);
  else named_sync(id, nt);
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
// NCH > 0: the number of K-chunks (Mp16 / 16) as a compile-time constant (16: M = 256, 8: M = 128):
// ring stages, parities and TMEM offsets reduce to cheap functions of the group index (the group
// and chunk loops themselves stay rolled for the instruction cache).  NCH = 0: any M <= 256.
template <int PW, int KT, int NH, int NCH>
__global__ void __launch_bounds__(PW * 32 + TC2_XW * 32, 1)
score_tc2_kernel(DevSpace S, DevGP G, BatchArgs A, CtaOut out, TcB TB, Tc2B T2, CandList L) {
  constexpr int TC_PROD_WARPS = PW;
  constexpr int TC_PROD_THREADS = PW * 32;
  constexpr int TC_THREADS = TC_PROD_THREADS + TC2_XW * 32;  // + MMA, loader, R2, L^-1 loader, 4 finalize warps
  constexpr int FW0 = PW + 4;                                // first finalize warp
  using LY = Tc2L<NCH == 16>;
  constexpr int TC_JQ = TC_PROD_THREADS / TC_ROWS;   // producer threads per candidate
  constexpr int TC_JPT = TC_KCH / TC_JQ;             // observed points per thread per chunk
  static_assert(TC_JQ == 4 && TC_JPT == 4, "R2 group columns are laid out for 16 producer warps");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ TopkSmem ts;
  __shared__ uint32_t tmem_base;
  __shared__ int eoff_s[DMAX];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Mp16 = NCH > 0 ? NCH * TC_KCH : TB.Mp16, nch = NCH > 0 ? NCH : TB.nch, Kp = T2.Kp;
  unsigned long long* const trace = blockIdx.x == 0 ? g_tc2_trace : nullptr;
  auto TR = [&](int u, int ev) {
    if (trace != nullptr && lane == 0 && u < TC2_TR_TILES)
      trace[(static_cast<size_t>(u) * TC2_TR_EV + ev) * TC2_TR_W + warp] = clock64();
  };
  const int ng = (nch + TC2_RG - 1) / TC2_RG;                         // R2 groups per tile
  // accumulators: one D (M > 128: 256 columns, the next tile's MMAs wait for the epilogue read) or two
  // (Mp16 <= 128: tile t's accumulator is read while the MMAs of tile t + 1 run -- "lag" mode)
  // (Mp16 <= 64, a single R2 group per tile: the head-start scheme measured better -- C4 stress
  // M = 48 8.72 -> 8.36 ms -- and C2 is neutral)
  const int ND = NCH > 0 ? (NCH * TC_KCH <= 128 ? 2 : 1) : ((Mp16 <= 128 && Mp16 > 64) ? 2 : 1);
  auto dcol = [&](int u) -> uint32_t { return static_cast<uint32_t>((ND == 2 ? (u & 1) : 0) * Mp16); };
  const uint32_t A0col = static_cast<uint32_t>(ND * Mp16);            // TMEM column of A stage 0
  const uint32_t R0col = A0col + 16u * TC2_NA;                        // TMEM column of R2 stage 0
  const uint32_t b_stage_bytes = 2u * Mp16 * TC_KCH * 2;              // L^-1 FP16 hi + lo at the widest chunk
  const uint32_t t_stage_bytes = 2u * (TC2_RG * TC_KCH) * Kp * 2;     // T: 2 FP16 pieces x 64 points
  const uint32_t e_bytes = static_cast<uint32_t>(TC_ROWS) * Kp * 2;   // E: 128 rows x Kp FP16
  unsigned char* const sm0 = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm0 + LY::BARS);
  float* alpha_s = reinterpret_cast<float*>(sm0 + LY::ALPHA);   // (alpha_j, |alpha_j|) pairs
  float* oh_s = reinterpret_cast<float*>(sm0 + LY::OH);         // [Mp16][NH]
  float* m_xh = reinterpret_cast<float*>(sm0 + LY::MXH);        // [TI][128][NH]
  float* m_part = reinterpret_cast<float*>(sm0 + LY::MPART);
  float* vpart = reinterpret_cast<float*>(sm0 + LY::VPART);
  uint32_t* m_cvi = reinterpret_cast<uint32_t*>(sm0 + LY::MCVI);
  uint32_t* m_j = reinterpret_cast<uint32_t*>(sm0 + LY::MJ);
  double* m_m0 = reinterpret_cast<double*>(sm0 + LY::MM0);
  float* xh_s = reinterpret_cast<float*>(sm0 + LY::XH);         // [NH][VMAX]
  unsigned char* stg = sm0 + LY::STG;                           // [2][TC2_STG_BYTES]
  // this CTA's tiles of the candidate list: blockIdx.x, blockIdx.x + gridDim.x, ...
  const uint64_t n_list = *L.count;
  const uint64_t n_tiles = (n_list + TC_ROWS - 1) / TC_ROWS;
  const int my_tiles = blockIdx.x < n_tiles ? static_cast<int>((n_tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
  unsigned char* B0 = sm0 + LY::VAR;
  unsigned char* T0 = B0 + static_cast<size_t>(TC2_NB) * b_stage_bytes;
  unsigned char* E0 = T0 + static_cast<size_t>(TC2_NT) * t_stage_bytes;
  uint64_t* arr = reinterpret_cast<uint64_t*>(E0 + 2ull * e_bytes);
  const uint32_t sB0 = tc::smem_u32(B0), sT0 = tc::smem_u32(T0), sE0 = tc::smem_u32(E0);
  uint64_t* a_full = bars;                     // [NA] count PW
  uint64_t* a_empty = a_full + TC2_NA;          // [NA] commit
  uint64_t* b_full = a_empty + TC2_NA;          // [NB] 1 + tx
  uint64_t* b_empty = b_full + TC2_NB;         // [NB] commit
  uint64_t* d_full = b_empty + TC2_NB;         // [ND] commit
  uint64_t* d_empty = d_full + 2;              // [ND] count PW
  uint64_t* t_ready = d_empty + 2;             // [TI] count 1 (tile meta + E rows published)
  uint64_t* r_full = t_ready + TC_TI;          // [RS] commit
  uint64_t* r_empty = r_full + TC2_RS;         // [RS] count PW
  uint64_t* x_full = r_empty + TC2_RS;         // [NT] 1 + tx  (T group loaded)
  uint64_t* x_empty = x_full + TC2_NT;         // [NT] commit
  uint64_t* s_full = x_empty + TC2_NT;         // [NS] 1 + tx  (tile records staged)
  uint64_t* s_empty = s_full + LY::NS;         // [NS] count PW
  uint64_t* ez_full = s_empty + LY::NS;        // [2]  1 + tx  (E buffer zeroed again by a bulk copy)
  uint64_t* f_free = ez_full + 2;              // [2]  count 4   (finalize done with the tile's slots)
  // hand-off of tile t to the finalize warps.  (A pair of named barriers -- producers bar.arrive,
  // finalize bar.sync -- deadlocked the NEXT launch in lag mode: stray barrier state outlived the
  // CTA.  mbarriers carry no state across launches.)
  uint64_t* f_ready = f_free + 2;              // [2]  count PW  (tile partial sums + |v|^2 written)

  // ---- setup
  // point-pair layout: [al_2p, al_2p+1, |al_2p|, |al_2p+1|] so one LDS.128 feeds packed f32x2 math
  for (int i = tid; i < Mp16; i += TC_THREADS) {
    alpha_s[4 * (i >> 1) + (i & 1)] = i < G.Mp ? __ldg(G.alpha + i) : 0.f;
    alpha_s[4 * (i >> 1) + 2 + (i & 1)] = i < G.Mp ? __ldg(G.aabs + i) : 0.f;
  }
  for (int i = tid; i < out.P; i += TC_THREADS) arr[i] = KEY_NONE;
  if (tid < DMAX) eoff_s[tid] = T2.eoff[tid];
  // SIMT features, point-pair layout: [pair][h][2 points]
  for (int i = tid; i < NH * Mp16; i += TC_THREADS) {
    const int j = i / (NH > 0 ? NH : 1), h = i - j * NH;
    oh_s[(j >> 1) * 2 * NH + 2 * h + (j & 1)] = __ldg(T2.oh + i);
  }
  for (int i = tid; i < NH * VMAX; i += TC_THREADS) xh_s[i] = __ldg(T2.xh + i);
  {
    // both one-hot buffers start zeroed; afterwards the loader re-zeroes a buffer with a bulk copy
    // as soon as the last R2 MMAs of its tile have completed (no zeroing pass, no barrier in publish)
    unsigned char* E0z = sm0 + LY::VAR + static_cast<size_t>(TC2_NB) * 2u * TB.Mp16 * TC_KCH * 2 +
                         static_cast<size_t>(TC2_NT) * 2u * (TC2_RG * TC_KCH) * T2.Kp * 2;
    for (uint32_t i = tid; i < 2u * TC_ROWS * T2.Kp * 2 / 16; i += TC_THREADS)
      *reinterpret_cast<uint4*>(E0z + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
    tc::fence_proxy_async();
  }
  if (tid == 0) {
    for (int s = 0; s < TC2_NA; ++s) {
      tc::mbar_init(a_full + s, TC_PROD_WARPS);
      tc::mbar_init(a_empty + s, 1);
    }
    for (int s = 0; s < TC2_NB; ++s) {
      tc::mbar_init(b_full + s, 1);
      tc::mbar_init(b_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(d_full + s, 1);
      tc::mbar_init(d_empty + s, TC_PROD_WARPS);
    }
    for (int s = 0; s < TC_TI; ++s) tc::mbar_init(t_ready + s, 1);
    for (int s = 0; s < TC2_RS; ++s) {
      tc::mbar_init(r_full + s, 1);
      tc::mbar_init(r_empty + s, TC_PROD_WARPS);
    }
    for (int s = 0; s < TC2_NT; ++s) {
      tc::mbar_init(x_full + s, 1);
      tc::mbar_init(x_empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(ez_full + s, 1);
      tc::mbar_init(f_free + s, TC_EPI_WARPS);
      tc::mbar_init(f_ready + s, TC_PROD_WARPS);
    }
    for (int s = 0; s < LY::NS; ++s) {
      tc::mbar_init(s_full + s, 1);
      tc::mbar_init(s_empty + s, TC_PROD_WARPS);
    }
    tc::mbar_fence_init();
    ts.n_list = 0;
    ts.n_add = 0;
    ts.tau = KEY_NONE;
    ts.drop = KEY_NONE;
  }
  const uint32_t tmem_cols = 512;
  if (warp == 0) tc::tmem_alloc(&tmem_base, tmem_cols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;

  if (warp < TC_PROD_WARPS) {
    // =========================================================== producers (+ epilogue read)
    tc::setmaxnreg_inc<TC2_PROD_REGS>();
    const int pt = tid;
    const int cand = pt & (TC_ROWS - 1);
    const int jq = pt >> 7;
    const int quad = warp & 3;
    const uint32_t sAl = tc::smem_u32(alpha_s);
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16);
    // k = sf2 poly(a) exp(-a) from R2 = 2^s r^2:  a = sqrt5 r = (sqrt5 2^-s/2) sqrt(R2)  (Matern 5/2),
    // a = r^2 / 2 = (2^-s / 2) R2 (RBF); exp2 argument folds ln(sf2).
    const float c_arg = (KT == 0) ? 2.2360679774997896f * T2.r_scale : 0.5f * T2.r2_scale;
    const float ex_c1 = -c_arg * 1.4426950408889634f;
    const float ex_c0 = log2f(G.sf2f) + static_cast<float>(T2.ek);   // k leaves the exp2 scaled by 2^ek

    // ---- epilogue of tile u (column blocks < nch - NA were accumulated during the chunk loop)
    // ---- epilogue, part 1 (all producer warps): the last NA column blocks of D -> |v|^2 partial,
    // release D.
    auto epilogue_read = [&](int u, float vsq_run) {
      tc::mbar_wait(d_full + (ND == 2 ? (u & 1) : 0), (ND == 2 ? (u >> 1) : u) & 1);
      TR(u, 4);
      tc::fence_after_sync();
      float vsq = vsq_run;
      const uint32_t taddr = lane_base + TC_JPT * jq + dcol(u);
      const int bfirst = nch > TC2_NA ? nch - TC2_NA : 0;
      for (int b0 = bfirst; b0 < nch; b0 += 4) {
        float v[16];
        uint32_t ad[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) ad[i] = taddr + 16u * static_cast<uint32_t>(b0 + i < nch ? b0 + i : b0);
        tc::tmem_ld4x4(ad[0], ad[1], ad[2], ad[3], v);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (b0 + i < nch)
            vsq = fmaf(v[4 * i], v[4 * i],
                       fmaf(v[4 * i + 1], v[4 * i + 1], fmaf(v[4 * i + 2], v[4 * i + 2], fmaf(v[4 * i + 3], v[4 * i + 3], vsq))));
      }
      vpart[((u & 1) * TC_JQ + jq) * TC_ROWS + quad * 32 + lane] = vsq * T2.vsq_unscale;
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(d_empty + (ND == 2 ? (u & 1) : 0));
      if (lane == 0) tc::mbar_arrive(f_ready + (u & 1));   // partial sums + |v|^2 of tile u -> finalize
      TR(u, 5);
    };

    // publish tile u: meta rows, zeroed partial sums, one-hot rows E[u & 1] and the SIMT-feature
    // values, from the staged list records; returns n (0 = end of this CTA's tiles)
    auto publish = [&](int u) -> int {
      int n = 0;
      const int us = u % TC_TI;
      if (u < my_tiles) {
        const uint64_t r0 = (blockIdx.x + static_cast<uint64_t>(u) * gridDim.x) * TC_ROWS;
        n = static_cast<int>(n_list - r0 < TC_ROWS ? n_list - r0 : TC_ROWS);
        const int ss = u % LY::NS;
        const unsigned char* sg = stg + ss * TC2_STG_BYTES;
        tc::mbar_wait(s_full + ss, (u / LY::NS) & 1);
        if (pt < n) {
          const int ms = u % LY::TI;
          m_cvi[ms * TC_ROWS + pt] = reinterpret_cast<const uint32_t*>(sg + TC2_STG_CVI)[pt];
          m_j[ms * TC_ROWS + pt] = reinterpret_cast<const uint32_t*>(sg + TC2_STG_J)[pt];
          m_m0[ms * TC_ROWS + pt] = reinterpret_cast<const double*>(sg + TC2_STG_M0)[pt];
        }
        unsigned char* E = E0 + (u & 1) * e_bytes;
        if (cand < n) {
          DV cdv;
          cdv.w[0] = reinterpret_cast<const uint64_t*>(sg + TC2_STG_DV0)[cand];
          cdv.w[1] = reinterpret_cast<const uint64_t*>(sg + TC2_STG_DV1)[cand];
          cdv.w[2] = reinterpret_cast<const uint64_t*>(sg + TC2_STG_DV2)[cand];
          int eo[DMAX / TC_JQ];                                  // this thread's features, loads hoisted
#pragma unroll
          for (int q = 0; q < DMAX / TC_JQ; ++q) eo[q] = (jq + TC_JQ * q < S.d) ? eoff_s[jq + TC_JQ * q] : -1;
          if (u >= 2) tc::mbar_wait(ez_full + (u & 1), ((u >> 1) + 1) & 1);   // buffer re-zeroed
#pragma unroll
          for (int q = 0; q < DMAX / TC_JQ; ++q) {
            if (eo[q] < 0) continue;
            const uint32_t col = static_cast<uint32_t>(eo[q]) + dv_get(cdv, jq + TC_JQ * q);
            *reinterpret_cast<uint16_t*>(E + tc::kmajor_off16(cand, col, Kp / 8)) = 0x3C00;   // FP16 1.0
          }
          if (jq < NH) {
            const int f = T2.hf[jq];
            m_xh[(us * TC_ROWS + cand) * (NH > 0 ? NH : 1) + jq] = f >= 0 ? xh_s[jq * VMAX + dv_get(cdv, f)] : 0.f;
          }
        }
        tc::fence_proxy_async();   // generic-proxy stores -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_empty + ss);   // staged records consumed
      }
      named_sync(1, TC_PROD_THREADS);
      if (pt == 0 && n > 0) tc::mbar_arrive(t_ready + us);   // E rows of tile u published (R2 warp)
      return n;
    };

    int n_cur = publish(0);
    const uint32_t sOH = tc::smem_u32(oh_s);
    // Chunks [cb, ce) of tile u (cb a multiple of the R2 group size; ce == nch or a multiple of it):
    // R2 (+ SIMT features) -> k -> A ring; partial sums accumulate into the caller's registers.
    // A-ring position of chunk c of tile u is u * nch + c and R2-group position u * ng + c / RG:
    // derived, not counted, so that with a compile-time nch (multiple of NA and of 2 RG) every
    // stage / slot / parity folds to a constant
    auto produce = [&](int u, int cb, int ce, unsigned long long& mu2, unsigned long long& sb2,
                       unsigned long long& kk2, float& vsq_run) {
      const uint32_t dq = lane_base + TC_JPT * jq + dcol(u);
      const uint32_t gbase = static_cast<uint32_t>(u) * static_cast<uint32_t>(nch);
      const uint32_t grbase = static_cast<uint32_t>(u) * static_cast<uint32_t>(ng);
      unsigned long long xb[NH > 0 ? NH : 1];                 // (x_h, x_h): broadcast over a point pair
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const float xv = m_xh[((u % TC_TI) * TC_ROWS + cand) * (NH > 0 ? NH : 1) + h];
        xb[h] = f2_pack(xv, xv);
      }
      const unsigned long long carg2 = f2_pack(c_arg, c_arg), c1_2 = f2_pack(ex_c1, ex_c1),
                               c0_2 = f2_pack(ex_c0, ex_c0), one2 = f2_pack(1.0f, 1.0f),
                               third2 = f2_pack(0.33333333333333333f, 0.33333333333333333f);
        // R2 groups are NOT unrolled: one group body (~360 instructions) keeps the producers' hot
        // loop inside the instruction cache (the fully unrolled 16-chunk loop was 26-43 KB of code and
        // stalled every warp on instruction fetch, ncu no_inst 19 % of samples)
#pragma unroll 1
        for (int c0 = cb; c0 < ce; c0 += TC2_RG) {
          // ---- one R2 group: the thread's 4 points of each of the 4 chunks are 16 contiguous
          // columns (T rows are permuted on the host), read with one load
          const uint32_t gr = grbase + static_cast<uint32_t>(c0 / TC2_RG);
          const int rs = gr % TC2_RS;
          float rv[TC2_RG * TC_JPT];
          tc::mbar_wait(r_full + rs, (gr / TC2_RS) & 1u);
          tc::fence_after_sync();
          tc::tmem_ld16(lane_base + R0col + 64u * rs + 16u * jq, rv);
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(r_empty + rs);
          const uint32_t g = gbase + static_cast<uint32_t>(c0);
          // The whole group's math first (4 chunks x 2 packed point pairs: eight independent chains
          // the scheduler can interleave), then the A-stage waits and stores: the waits are asm
          // volatile and would otherwise fence every chunk's two chains off from the next chunk's.
          const int ncg = nch - c0 < TC2_RG ? nch - c0 : TC2_RG;
#pragma unroll
          for (int hb = 0; hb < TC2_RG; hb += TC2_CB) {
            if (hb >= ncg) break;
            uint32_t hw[TC2_CB][2], lw[TC2_CB][2];
#pragma unroll
            for (int cb = 0; cb < TC2_CB; ++cb) {
              const int cg = hb + cb;
              const int c = c0 + cg;
              if (cg >= ncg) break;
#pragma unroll
              for (int qp = 0; qp < TC_JPT / 2; ++qp) {
                const int jo = c * TC_KCH + jq * TC_JPT + 2 * qp;      // even
                // R2 >= 0 by construction (non-negative products, FP32 accumulation; squares)
                unsigned long long r2p = f2_pack(rv[cg * TC_JPT + 2 * qp], rv[cg * TC_JPT + 2 * qp + 1]);
                if (NH > 0) {
#pragma unroll
                  for (int h = 0; h < NH; h += 2) {
                    unsigned long long o0, o1;
                    tc::lds_u64x2_nv(sOH + 4u * ((jo >> 1) * 2 * NH + 2 * h), o0, o1);
                    const unsigned long long d0 = f2_sub(xb[h], o0), d1 = f2_sub(xb[h + 1], o1);
                    r2p = f2_fma(d0, d0, r2p);
                    r2p = f2_fma(d1, d1, r2p);
                  }
                }
                unsigned long long argp, expp, polyp;
                if (KT == 0) {
                  const float2 r2 = f2_unpack(r2p);
                  const unsigned long long rp = f2_pack(tc::sqrt_approx_ftz(r2.x), tc::sqrt_approx_ftz(r2.y));
                  argp = f2_mul(rp, carg2);
                  const float2 ea = f2_unpack(f2_fma(rp, c1_2, c0_2));
                  expp = f2_pack(tc::ex2_approx(ea.x), tc::ex2_approx(ea.y));
                  polyp = f2_fma(argp, f2_fma(argp, third2, one2), one2);
                } else {
                  argp = f2_mul(r2p, carg2);
                  const float2 ea = f2_unpack(f2_fma(r2p, c1_2, c0_2));
                  expp = f2_pack(tc::ex2_approx(ea.x), tc::ex2_approx(ea.y));
                  polyp = one2;
                }
                const unsigned long long kvalp = f2_mul(polyp, expp);
                const unsigned long long ccp = f2_fma(kvalp, argp, kvalp);
                unsigned long long alp, aap;
                tc::lds_u64x2_nv(sAl + 16u * (jo >> 1), alp, aap);
                mu2 = f2_fma(kvalp, alp, mu2);
                sb2 = f2_fma(ccp, aap, sb2);
                kk2 = f2_fma(ccp, ccp, kk2);
                // FP16 hi / lo split of the (2^ek-scaled) cross-covariances, packed two per column:
                // hi = k with the low 13 mantissa bits cleared (an FP16 value: 11 significant bits,
                // exponent inside the FP16 range by the 2^ek scale), lo = k - hi exactly in FP32, then
                // both converted (hi exactly, lo rounded: |k - hi - lo16| <= 2^-22 |k|); the mask runs
                // on the ALU pipe instead of two FP16->FP32 conversions on the FMA pipe
                const float2 kk = f2_unpack(kvalp);
                const float h0 = __uint_as_float(__float_as_uint(kk.x) & 0xFFFFE000u);
                const float h1 = __uint_as_float(__float_as_uint(kk.y) & 0xFFFFE000u);
                const float2 lo = f2_unpack(f2_sub(kvalp, f2_pack(h0, h1)));
                hw[cb][qp] = tc::pack_f16x2(h0, h1);
                lw[cb][qp] = tc::pack_f16x2(lo.x, lo.y);
              }
            }
#pragma unroll
            for (int cb = 0; cb < TC2_CB; ++cb) {
              const int cg = hb + cb;
              if (cg >= ncg) break;
              const int s = (g + cg) % TC2_NA;
              tc::mbar_wait(a_empty + s, (((g + cg) / TC2_NA) & 1u) ^ 1u);
              tc::fence_after_sync();
              const uint32_t acol = lane_base + A0col + 16u * s + 2 * jq;
              tc::tmem_st2(acol, hw[cb][0], hw[cb][1]);
              tc::tmem_st2(acol + 8, lw[cb][0], lw[cb][1]);
            }
          }
          tc::tmem_st_wait();
          tc::fence_before_sync();
          __syncwarp();
#pragma unroll
          for (int cg = 0; cg < TC2_RG; ++cg) {
            if (c0 + cg >= nch) break;
            if (lane == 0) tc::mbar_arrive(a_full + ((g + cg) % TC2_NA));
          }
          // ---- accumulator column blocks made final by this group's a_empty waits:
          // [c0 - NA, c_last - NA]; one batched read (the last NA blocks are left to the epilogue)
          if (c0 >= TC2_NA && c0 + TC2_RG <= nch) {
            // steady state: blocks c0 - NA .. c0 - NA + 3, all final
            float v[16];
            const uint32_t a0 = dq + 16u * static_cast<uint32_t>(c0 - TC2_NA);
            tc::tmem_ld4x4(a0, a0 + 16u, a0 + 32u, a0 + 48u, v);
            unsigned long long acc = f2_mul(f2_pack(v[0], v[1]), f2_pack(v[0], v[1]));
#pragma unroll
            for (int i = 2; i < 16; i += 2) acc = f2_fma(f2_pack(v[i], v[i + 1]), f2_pack(v[i], v[i + 1]), acc);
            const float2 a = f2_unpack(acc);
            vsq_run += a.x + a.y;
          } else {
            const int c_last = (c0 + TC2_RG < nch ? c0 + TC2_RG : nch) - 1;
            const int b0 = c0 - TC2_NA;
            if (c_last - TC2_NA >= 0) {
              float v[16];
              uint32_t ad[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int b = b0 + i;
                ad[i] = dq + 16u * static_cast<uint32_t>(b >= 0 && b <= c_last - TC2_NA ? b : 0);
              }
              tc::tmem_ld4x4(ad[0], ad[1], ad[2], ad[3], v);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int b = b0 + i;
                if (b >= 0 && b <= c_last - TC2_NA)
                  vsq_run = fmaf(v[4 * i], v[4 * i],
                                 fmaf(v[4 * i + 1], v[4 * i + 1], fmaf(v[4 * i + 2], v[4 * i + 2], fmaf(v[4 * i + 3], v[4 * i + 3], vsq_run))));
              }
            }
          }
        }
    };
    auto flush_part = [&](int u, unsigned long long mu2, unsigned long long sb2, unsigned long long kk2) {
      const float2 m_ = f2_unpack(mu2), s_ = f2_unpack(sb2), k_ = f2_unpack(kk2);
      const float mu_p = m_.x + m_.y, sb_p = s_.x + s_.y, kk_p = k_.x + k_.y;
      // each thread owns its slot (no atomics: the four quarters of a candidate used to contend)
      float* mp = m_part + ((u % LY::PS) * TC_JQ + jq) * 3 * TC_ROWS;
      mp[cand] = mu_p * T2.k_unscale;
      mp[TC_ROWS + cand] = sb_p * T2.k_unscale;
      mp[2 * TC_ROWS + cand] = kk_p * (T2.k_unscale * T2.k_unscale);
    };

    // Tile loop.  Before the epilogue of tile t (which waits for all of t's MMAs) the producers
    // already produce the first NA chunks of tile t+1 into the A ring, so the MMA drain of tile t
    // overlaps useful work and the MMAs of t+1 start as soon as the accumulator is read out.
    unsigned long long mu_c = 0ull, sb_c = 0ull, kk_c = 0ull;  // tile t's running sums (packed pairs)
    float vsq_c = 0.f, vsq_t = 0.f;
    if (ND == 2) {
      // lag mode (Mp16 <= 128, two accumulators): iteration t publishes t + 1, produces every chunk of
      // tile t (its R2 groups were issued one iteration earlier) and reads the accumulator of tile
      // t - 1 (its MMAs completed while tile t was produced): neither MMA round trip is exposed
      for (int t = 0; t <= my_tiles; ++t) {
        const bool have = t < my_tiles;
        // slots of tile t - 3 (meta (t + 1) % 4, partial sums t % 3, |v|^2 (t - 1) & 1) released --
        // also in the final epilogue-only iteration: its f_ready arrival reuses tile t - 3's phase
        // slot, and arriving before the finalize warps consumed that phase aliases the parity
        if (t >= 3) tc::mbar_wait(f_free + ((t - 3) & 1), ((t - 3) >> 1) & 1);
        if (have) {
          TR(t, 0);
          publish(t + 1);
          TR(t, 1);
          produce(t, 0, nch, mu_c, sb_c, kk_c, vsq_c);
          TR(t, 2);
          flush_part(t, mu_c, sb_c, kk_c);
          mu_c = sb_c = kk_c = 0ull;
        }
        if (t >= 1) {
          TR(t - 1, 3);
          epilogue_read(t - 1, vsq_t);          // hands tile t - 1 to the finalize warps
        }
        vsq_t = vsq_c;
        vsq_c = 0.f;
        if (!have) break;
      }
    } else {
    // One instruction copy of each chunk range (the chunk loop is unrolled, and the code must stay
    // small for the instruction cache): iteration t = -1 only produces the head of tile 0.
    constexpr int HEADC = NCH < TC2_NA ? NCH : TC2_NA;
    const int head = NCH > 0 ? HEADC : (nch < TC2_NA ? nch : TC2_NA);   // multiple of the R2 group size, or all of nch
    int n_next = n_cur;                                       // rows of tile t + 1
    n_cur = 0;                                                // rows of tile t
    for (int t = -1; t < 0 || n_cur > 0; ++t) {
      if (t >= 0) {
        TR(t, 0);
        // slots of tile t - 2 (meta (t + 1) % 4, partial sums t % 3, |v|^2 t & 1) released by the finalize warps
        if (t >= 2) tc::mbar_wait(f_free + (t & 1), ((t >> 1) + 1) & 1);
        n_next = publish(t + 1);
        TR(t, 1);
        if (NCH > 0) produce(t, HEADC, NCH, mu_c, sb_c, kk_c, vsq_c);
        else produce(t, head, nch, mu_c, sb_c, kk_c, vsq_c);
        TR(t, 2);
        flush_part(t, mu_c, sb_c, kk_c);
        vsq_t = vsq_c;
        mu_c = sb_c = kk_c = 0ull;
        vsq_c = 0.f;
      }
      if (n_next > 0) {
        if (NCH > 0) produce(t + 1, 0, HEADC, mu_c, sb_c, kk_c, vsq_c);
        else produce(t + 1, 0, head, mu_c, sb_c, kk_c, vsq_c);
      }
      if (t >= 0) {
        TR(t, 3);
        epilogue_read(t, vsq_t);              // hands tile t to the finalize warps
      }
      n_cur = n_next;
    }
    }
  } else {
  tc::setmaxnreg_dec<TC2_AUX_REGS>();
  if (warp == TC_PROD_WARPS) {
    // =========================================================== MMA issuer
    // The whole warp runs this loop in lock-step (warp-uniform state); one elected lane issues the
    // MMAs / commits (elect.sync inside the asm).  All bulk copies are the loader warp's, so this
    // warp never waits on a ring refill.
    uint32_t g = 0;                  // L^-1 chunks consumed
    auto tile_exists = [&](int u) -> bool { return u < my_tiles; };
    __syncwarp();
    const uint64_t dB = tc::sdesc(sB0, 128, (TC_KCH / 8) * 128);
    long long wa_acc = 0, wb_acc = 0;
    for (int t = 0; tile_exists(t); ++t) {
      TR(t, 8);
      tc::mbar_wait(d_empty + (ND == 2 ? (t & 1) : 0), ((ND == 2 ? (t >> 1) : t) & 1) ^ 1);
      TR(t, 9);
      tc::fence_after_sync();
      // one chunk: operand waits, 3 MMAs + 2 commits (rolled: unrolling it gained nothing once the
      // producers' code fit the instruction cache, and it spilled at 48 registers)
      auto mma_chunk = [&](int c) {
        const uint32_t ga = static_cast<uint32_t>(t) * static_cast<uint32_t>(nch) + static_cast<uint32_t>(c);
        const int sa = ga % TC2_NA, sbb = g % TC2_NB;
        const long long w0 = trace != nullptr ? clock64() : 0;
        tc::mbar_wait(a_full + sa, (ga / TC2_NA) & 1);
        const long long w1 = trace != nullptr ? clock64() : 0;
        tc::mbar_wait(b_full + sbb, (g / TC2_NB) & 1);
        if (trace != nullptr) {
          wa_acc += w1 - w0;
          wb_acc += clock64() - w1;
        }
        if (c == TC2_NA) TR(t, 11);
        tc::fence_after_sync();
        const int N = Mp16 - c * TC_KCH;
        const uint32_t idesc = tc::idesc_f16(TC_ROWS, N);
        const uint32_t a_h = tmem + A0col + 16u * sa, a_l = a_h + 8;
        const uint64_t bh = dB + ((sbb * b_stage_bytes) >> 4);
        const uint64_t bl = bh + ((N * TC_KCH * 2) >> 4);
        const uint32_t d = tmem + dcol(t) + c * TC_KCH;
        // 3-term FP16 split: hi.hi + hi.lo + lo.hi (one K = 16 step each), then release A and B
        tc::mma3_f16_ts_commit2_w(d, a_h, a_l, bh, bl, idesc, c > 0 ? 1u : 0u, a_empty + sa, b_empty + sbb);
        ++g;
      };
      if (NCH > 0) {
#pragma unroll 1
        for (int c = 0; c < (NCH > 0 ? NCH : 1); ++c) mma_chunk(c);
      } else {
        for (int c = 0; c < nch; ++c) mma_chunk(c);
      }
      tc::mma_commit_w(d_full + (ND == 2 ? (t & 1) : 0));
      TR(t, 10);
      if (trace != nullptr && lane == 0 && t < TC2_TR_TILES) {   // MMA warp: cycles waiting on A / B per tile
        trace[(static_cast<size_t>(t) * TC2_TR_EV + 12) * TC2_TR_W + warp] = static_cast<unsigned long long>(wa_acc);
        trace[(static_cast<size_t>(t) * TC2_TR_EV + 13) * TC2_TR_W + warp] = static_cast<unsigned long long>(wb_acc);
      }
      wa_acc = wb_acc = 0;
    }
    __syncwarp();
  } else if (warp == TC_PROD_WARPS + 2) {
    // =========================================================== R2 issuer (sub-partition 2)
    // R2 group x = D_R[x % RS] = E[tile & 1] T_g^T (N = 64; 2 FP16 pieces x Kp/16 k-steps), issued
    // as soon as its tile's E rows are published, its TMEM slot is free and its T stage is loaded:
    // an MMA stream independent of the L^-1 chunks (separate accumulators), on its own warp so
    // that neither stream waits for the other and the MMA warp's sub-partition carries only the
    // L^-1 issue.
    __syncwarp();
    const uint32_t sbo16 = (Kp / 8) * 128;
    const uint64_t dE = tc::sdesc(sE0, 128, sbo16), dT = tc::sdesc(sT0, 128, sbo16);
    const uint32_t piece16 = ((TC2_RG * TC_KCH) * Kp * 2) >> 4;   // descriptor units (16 B)
    const uint32_t idesc_r = tc::idesc_f16(TC_ROWS, TC2_RG * TC_KCH);
    const int ksteps_r = Kp / 16;
    uint32_t x = 0;
    for (int ru = 0; ru < my_tiles; ++ru) {
      tc::mbar_wait(t_ready + (ru % TC_TI), (ru / TC_TI) & 1);
      for (int rgi = 0; rgi < ng; ++rgi, ++x) {
        const int rs = x % TC2_RS, st_ = x % TC2_NT;
        tc::mbar_wait(r_empty + rs, ((x / TC2_RS) & 1u) ^ 1u);
        tc::mbar_wait(x_full + st_, (x / TC2_NT) & 1u);
        tc::fence_after_sync();
        const uint32_t dR = tmem + R0col + 64u * rs;
        const uint64_t ad = dE + (((ru & 1) * e_bytes) >> 4), bd = dT + ((st_ * t_stage_bytes) >> 4);
        for (int ks = 0; ks < ksteps_r; ++ks)
          tc::mma2_f16_w(dR, ad + 16 * ks, bd + 16 * ks, bd + piece16 + 16 * ks, idesc_r, ks > 0 ? 1u : 0u);
        tc::mma_commit_w(r_full + rs);
        tc::mma_commit_w(x_empty + st_);
      }
    }
    __syncwarp();
  } else if (warp == TC_PROD_WARPS + 3) {
    // =========================================================== L^-1 chunk loader (sub-partition 3)
    // The MMA warp's critical operand: refill a ring slot the moment its MMAs complete (blocking
    // wait, no polling back-off) -- the polling loader made the MMA warp wait ~7300 cycles per
    // tile on b_full (CTA-0 trace), three times its wait for the producers' A stages.
    if (lane == 0) {
      const uint32_t tot_L = static_cast<uint32_t>(my_tiles) * nch;
      int lc = 0;
      for (uint32_t gl = 0; gl < tot_L; ++gl) {
        const int s_ = gl % TC2_NB;
        tc::mbar_wait(b_empty + s_, ((gl / TC2_NB) & 1u) ^ 1u);
        const uint32_t bytes = 2u * (Mp16 - lc * TC_KCH) * TC_KCH * 2;
        tc::mbar_arrive_expect_tx(b_full + s_, bytes);
        tc::bulk_g2s(B0 + static_cast<size_t>(s_) * b_stage_bytes, T2.wch + T2.woff[lc], bytes, b_full + s_);
        if (++lc == nch) lc = 0;
      }
    }
    __syncwarp();
  } else if (warp == TC_PROD_WARPS + 1) {
    // =========================================================== loader (lane 0)
    // T groups in ring order with blocking waits: refill a stage once its R2 MMAs completed, and
    // zero a tile's one-hot buffer once the last R2 group of that tile completed.  Exactly the CTA's
    // totals are loaded, so nothing is left in flight at exit.
    if (lane == 0) {
      const uint32_t tot_T = static_cast<uint32_t>(my_tiles) * ng;
      int xc = 0;
      for (uint32_t xl = 0; xl < tot_T; ++xl) {
        const int s_ = xl % TC2_NT;
        tc::mbar_wait(x_empty + s_, ((xl / TC2_NT) & 1u) ^ 1u);
        if (xl >= TC2_NT) {
          // R2 group xl - NT has completed; if it was the last group of its tile u, the one-hot
          // buffer E[u & 1] is free: zero it for tile u + 2 (every u + 2 < my_tiles gets here)
          const uint32_t xg = xl - TC2_NT;
          const int u = static_cast<int>(xg / ng);
          if (xg % ng == static_cast<uint32_t>(ng - 1) && u + 2 < my_tiles) {
            tc::mbar_arrive_expect_tx(ez_full + (u & 1), e_bytes);
            tc::bulk_g2s(E0 + (u & 1) * e_bytes, T2.ezero, e_bytes, ez_full + (u & 1));
          }
        }
        tc::mbar_arrive_expect_tx(x_full + s_, t_stage_bytes);
        tc::bulk_g2s(T0 + static_cast<size_t>(s_) * t_stage_bytes,
                     T2.tch + static_cast<size_t>(xc) * (t_stage_bytes / 2), t_stage_bytes, x_full + s_);
        if (++xc == ng) xc = 0;
      }
    }
    __syncwarp();
  } else {
    // =========================================================== finalize (warps 20-23)
    const int pt = tid - FW0 * 32;                       // row of the tile
    double* scratch = TB.scratch + (static_cast<size_t>(blockIdx.x) * TC_EPI_WARPS + (warp & 3)) * Mp16;
    // ---- finalize (row = pt): FP32 screen + bound of tile u's rows and lazy admission.  Keys that
    // lose against tau lower this thread's drop_r instead of a shared atomicMin
    // per row (min is order-free; reduced once at the end, and tc2_prune lowers ts.drop as before).
    uint64_t drop_r = KEY_NONE;
    // list records of tile sl into staging slot sl & 1 once publish(sl - 2) consumed it (lane 0 of
    // the first finalize warp; publish(sl) waits on s_full)
    auto stage = [&](int sl) {
      const int ss = sl % LY::NS;
      tc::mbar_wait(s_empty + ss, ((sl / LY::NS) & 1u) ^ 1u);
      const uint64_t r0 = (blockIdx.x + static_cast<uint64_t>(sl) * gridDim.x) * TC_ROWS;
      const uint32_t n = static_cast<uint32_t>(n_list - r0 < TC_ROWS ? n_list - r0 : TC_ROWS);
      const uint32_t b4 = (n * 4 + 15) & ~15u, b8 = (n * 8 + 15) & ~15u;   // bulk sizes: multiples of 16 B
      unsigned char* sg = stg + ss * TC2_STG_BYTES;
      uint64_t* bar = s_full + ss;
      tc::mbar_arrive_expect_tx(bar, 2 * b4 + 4 * b8);
      tc::bulk_g2s(sg + TC2_STG_CVI, L.cvi + r0, b4, bar);
      tc::bulk_g2s(sg + TC2_STG_J, L.j + r0, b4, bar);
      tc::bulk_g2s(sg + TC2_STG_M0, L.m0 + r0, b8, bar);
      tc::bulk_g2s(sg + TC2_STG_DV0, L.dv0 + r0, b8, bar);
      tc::bulk_g2s(sg + TC2_STG_DV1, L.dv1 + r0, b8, bar);
      tc::bulk_g2s(sg + TC2_STG_DV2, L.dv2 + r0, b8, bar);
    };
    const bool stager = warp == FW0 && lane == 0;
    auto finalize = [&](int u, int n) {
      const int us = u % LY::PS, ms = u % LY::TI, vs_slot = u & 1;
      uint64_t key = KEY_NONE;
      bool sensitive = false;
      const int row = pt;
      float mu32 = 0.f, sb = 0.f, kk = 0.f, vv = 0.f, mu = 0.f, s2 = 0.f, d_mu = 0.f, d_s2 = 0.f;
      double cm0 = 0.0;
      bool early = false;
      if (pt < n) {
#pragma unroll
        for (int q = 0; q < TC_JQ; ++q) {
          const float* mp = m_part + (us * TC_JQ + q) * 3 * TC_ROWS;
          mu32 += mp[row];
          sb += mp[TC_ROWS + row];
          kk += mp[2 * TC_ROWS + row];
          vv += vpart[(vs_slot * TC_JQ + q) * TC_ROWS + row];
        }
        cm0 = m_m0[ms * TC_ROWS + row];
        TR(u, 13);
        mu = static_cast<float>(cm0 + G.b) + mu32;
        const float vs = vv;
        s2 = static_cast<float>(G.sf2) - vs;
        // FP32 k + 3xTF32 contraction: error coefficient 8x the SIMT one
        const float eps = 8.0f * static_cast<float>(G.eps);
        d_mu = eps * sb + 2e-7f * (1.0f + fabsf(mu));
        const float ew = eps * static_cast<float>(G.w_fro);
        d_s2 = 2.5f * ew * sqrtf(vs * kk) + ew * ew * kk + eps * vs + 8.0f * U32 * G.sf2f;
        // Early rejection (EI, bench path only): a cheap upper bound of the admission score,
        //   ln sigma + ln h(z),  h(z) <= phi(z) / (1 + z^2) for z <= 0 (Mills ratio
        //   Q(x) >= x phi(x) / (1 + x^2)),  h(z) <= z + phi(0) for z > 0,
        // at the same (mu - d_mu, s2 + d_s2) as the exact screen, plus slack covering twice the
        // screen's evaluation margin and its own MUFU rounding: its key never exceeds the exact
        // admission key, so key >= tau rejects exactly the rows the exact screen would reject, and
        // the (smaller) cheap key is a valid entry for the best-dropped bound.
        const uint64_t tau = ts.tau;
        if (A.acq == 0 && !A.d_scores && !A.d_screen && tau != KEY_NONE) {
          const float s2p = s2 + d_s2;
          if (s2p > 0.0f) {
            const float z = (static_cast<float>(G.fstar) - (mu - d_mu) - static_cast<float>(A.xi)) * rsqrtf(s2p);
            const float lnhb = z > 0.0f ? __logf(z + 0.3989422804014327f)
                                        : -0.5f * z * z - 0.9189385332046727f - __logf(1.0f + z * z);
            const float cheap = 0.5f * __logf(s2p) + lnhb;
            const float cheap_ub = cheap + 2e-5f * (1.0f + fabsf(cheap) + z * z);
            const uint64_t kc = make_key(cheap_ub, m_cvi[ms * TC_ROWS + row]);
            if (kc >= tau) {
              early = true;
              if (kc < drop_r) drop_r = kc;
            }
          }
        }
      }
      const bool warp_early = __all_sync(0xffffffffu, early || pt >= n);
      if (pt < n && !early && !warp_early) {
        const float fstar = static_cast<float>(G.fstar), m0f = static_cast<float>(cm0);
        float m2;
        float ub = acquisition32(A.acq, mu - d_mu, s2 + d_s2, m0f, fstar, static_cast<float>(A.xi),
                                 static_cast<float>(A.kappa), m2);
        ub += m2;
        if (A.d_screen) {   // parity / debug output of the screen (never on the bench path)
          float m3;
          const float scr = acquisition32(A.acq, mu, s2, m0f, fstar, static_cast<float>(A.xi),
                                          static_cast<float>(A.kappa), m3);
          *reinterpret_cast<float4*>(A.d_screen + 4ull * m_j[ms * TC_ROWS + row]) = make_float4(mu, s2, scr, ub);
        }
        TR(u, 14);
        if (A.d_scores) {
          const double mud = cm0 + G.b + static_cast<double>(mu32);
          const double s2d = G.sf2 - static_cast<double>(vv);
          if (A.acq == 0) {
            if (s2d > 0.0) {
              const double sg = sqrt(s2d), z = (G.fstar - mud - A.xi) / sg;
              if (z >= -3.2) {
                const double Phi = 0.5 * erfc(-z * INV_SQRT2);
                const double h = exp(-0.5 * z * z) * INV_SQRT_2PI + z * Phi;
                const double uu = static_cast<double>(U32);
                // R2 from the tensor cores: mu error model 4u(1 + sb)
                const double e_s = (1.0 - z * Phi / h) / (2.0 * s2d) * 160.0 * uu * static_cast<double>(vv) +
                                   Phi / (sg * h) * 4.0 * uu * (1.0 + static_cast<double>(sb));
                sensitive = e_s > 5e-6;
              }
            } else {
              sensitive = true;
            }
          }
          if (!sensitive)
            A.d_scores[m_j[ms * TC_ROWS + row]] =
                static_cast<float>(acquisition(A.acq, mud, s2d, cm0, G.fstar, A.xi, A.kappa));
        }
        if (!sensitive && ub > -INFINITY) key = make_key(ub, m_cvi[ms * TC_ROWS + row]);
      }
      {
        unsigned fl = __ballot_sync(0xffffffffu, sensitive);
        while (fl) {
          const int src = __ffs(fl) - 1;
          fl &= fl - 1;
          const int row = (warp - FW0) * 32 + src;
          const uint32_t cvi = m_cvi[ms * TC_ROWS + row];
          DV dv;
          uint32_t act;
          uint64_t raw;
          decode_dev(S, cvi, dv, act, raw);
          double kalpha, vq;
          posterior64_warp(S, G, dv, lane, scratch, kalpha, vq);
          if (lane == src) {
            const double cm0 = m_m0[ms * TC_ROWS + row];
            const double sc = acquisition(A.acq, cm0 + G.b + kalpha, G.sf2 - vq, cm0, G.fstar, A.xi, A.kappa);
            const double ub = sc + 1e-12 * fmax(1.0, fabs(sc));
            A.d_scores[m_j[ms * TC_ROWS + row]] = static_cast<float>(sc);
            if (ub > -INFINITY) key = make_key(__double2float_ru(ub), cvi);
          }
        }
      }
      TR(u, 6);
      if (key != KEY_NONE) {
        if (key < ts.tau) {
          const int pos = atomicAdd(&ts.n_add, 1);
          arr[ts.n_list + pos] = key;
        } else if (key < drop_r) {
          drop_r = key;
        }
      }
      TR(u, 7);
    };

    if (stager)
      for (int sl = 0; sl < LY::AHEAD && sl < my_tiles; ++sl) stage(sl);   // the last waits for publish(0)
    __syncwarp();
    for (int t = 0; t < my_tiles; ++t) {
      tc::mbar_wait(f_ready + (t & 1), (t >> 1) & 1);      // tile t handed over
      if (stager && t + LY::AHEAD < my_tiles) stage(t + LY::AHEAD);   // publish(t + 1) done: slot free
      __syncwarp();
      const uint64_t r0 = (blockIdx.x + static_cast<uint64_t>(t) * gridDim.x) * TC_ROWS;
      const int n = static_cast<int>(n_list - r0 < TC_ROWS ? n_list - r0 : TC_ROWS);
      finalize(t, n);
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(f_free + (t & 1));   // tile t's slots may be reused
      named_sync(2, TC_ROWS);                              // admissions done: uniform prune decision
      if (ts.n_list + ts.n_add > out.P - TC_ROWS) tc2_prune(arr, ts, out.KC, pt, TC_ROWS, 2);
      else named_sync(2, TC_ROWS);                         // decision read before the next tile's admissions
    }
    // ---- best dropped key, CTA list (final prune: sorted, at most KC entries)
    if (drop_r != KEY_NONE)
      atomicMin(reinterpret_cast<unsigned long long*>(&ts.drop), static_cast<unsigned long long>(drop_r));
    named_sync(2, TC_ROWS);
    tc2_prune(arr, ts, out.KC, pt, TC_ROWS, 2);
    const int n = ts.n_list;
    uint64_t* dst = out.lists + static_cast<size_t>(blockIdx.x) * out.KC;
    for (int i = pt; i < n; i += TC_ROWS) dst[i] = arr[i];
    if (pt == 0) {
      out.counts[blockIdx.x] = n;
      out.drop[blockIdx.x] = ts.drop;
    }
  }
  }
  // ---- teardown
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, tmem_cols);
  }
}

}  // namespace as
