// Candidate generation kernel: index -> configuration -> validity -> simulator,
// writing the VALID candidates of a slice of the batch as a compact list (SoA) for the
// tensor-core score kernel.  Decode + simulator are latency-bound integer / FP64 work; run as a
// separate high-occupancy kernel they no longer stall the producer warps of the score kernel
// (which has one 544-thread CTA per SM), and the score kernel sees full 128-row tiles only.
//
// Per candidate j of the slice [j0, j0 + nj):
//   p = begin + j (RANGE) or pi_seed(begin + j) (SAMPLE; reading R3)
//   (dv, act, raw) = CVI decode of p (SMEM structure index)
//   (cost, ok)     = simulator + FP64 resource check (R7)
//   d_raw[j] = raw; invalid: d_scores[j] = -inf; valid: append (cvi, j, ln cost, dv) to the list.
#pragma once
#include "kernels.cuh"

namespace as {

constexpr int GEN_THREADS = 256;
constexpr int GEN_CI_MAX = 4096;             // SMEM structure index entries (32 KB)

struct CandList {
  uint32_t* cvi;                // [cap + 128]
  uint32_t* j;                  // [cap + 128]   index in the batch (d_scores / d_raw slot)
  double* m0;                   // [cap + 128]   ln cost (GP prior mean, R9)
  uint64_t* dv0;                // [cap + 128]   digit vector words
  uint64_t* dv1;
  uint64_t* dv2;
  unsigned long long* count;    // number of records
};

// ENS: GP prior mean from the regression-simulator ensemble (NEXT-1) instead of ln cost_sim; a
// template parameter so the default instantiation carries no trace of it (register allocation).
// NC: tail-group count as a compile-time constant (decode_tail_nc; 0 = any count, runtime loop)
template <bool ENS, int NC>
#ifndef AS_GEN_OCC
#define AS_GEN_OCC 3
#endif
__global__ void __launch_bounds__(GEN_THREADS, AS_GEN_OCC)
gen_kernel(DevSpace S, BatchArgs A, uint64_t j0, uint64_t nj, CandList L, int ci_n, unsigned long long* valid_total) {
  extern __shared__ __align__(16) uint64_t gen_cidx[];
  __shared__ unsigned int blk_valid;         // this block's valid candidates (< 2^32 per slice)
  const int tid = threadIdx.x, lane = tid & 31;
  // ci_n < 0: SMEM copies of the whole prefix table (n_struct + 1) and the bucket index (decode by
  // bucket); else a coarse index of ci_n entries
  const bool by_bucket = ci_n < 0;
  uint32_t* gen_bkt = reinterpret_cast<uint32_t*>(gen_cidx + (S.n_struct + 1));
  if (tid == 0) blk_valid = 0;
  if (by_bucket) {
    for (int i = tid; i <= S.n_struct; i += GEN_THREADS) gen_cidx[i] = __ldg(S.prefix + i);
    for (int i = tid; i <= S.n_bucket; i += GEN_THREADS) gen_bkt[i] = __ldg(S.bucket + i);
  } else {
    load_cidx_n(S, gen_cidx, ci_n, tid, GEN_THREADS);
  }
  __syncthreads();
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * GEN_THREADS;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * GEN_THREADS; base < nj; base += stride) {
    const uint64_t jj = base + tid;
    const bool in = jj < nj;
    bool ok = false;
    DV dv;
    uint32_t act = 0;
    uint64_t raw = 0, pcvi = 0;
    double cost = 1.0;
    const uint64_t j = j0 + jj;
    if (in) {
      bool pin;
      pcvi = assign_pos(A, j, pin);
      int sidx = 0;
      uint64_t memok = 0;
      if (by_bucket) {
        // the structure's resource-check bits are requested before the tail decode (its loads
        // would otherwise queue behind the tuple loads and the check would wait a second L2 trip)
        sidx = find_struct_bucket(S, gen_cidx, gen_bkt, pcvi);
        if (S.srec != nullptr) memok = __ldg(&S.srec[sidx].memok);
        decode_tail_nc<NC>(S, sidx, static_cast<uint32_t>(pcvi - gen_cidx[sidx]), dv, act, raw);
      } else {
        decode_dev_ci(S, gen_cidx, ci_n, pcvi, dv, act, raw, &sidx);
        if (S.srec != nullptr) memok = __ldg(&S.srec[sidx].memok);
      }
      if (S.srec != nullptr) {
        // per-structure products + tabulated resource check (derived mode)
        SimRec r;
        const double2* rp = reinterpret_cast<const double2*>(S.srec + sidx);
        const double2 a = __ldg(rp), b = __ldg(rp + 1), c = __ldg(rp + 2), e = __ldg(rp + 3);
        r.comp = a.x; r.bub = a.y; r.tp = b.x; r.dp = b.y; r.ep = c.x; r.cp = c.y; r.vi_tp = e.x;
        r.tpgt1 = static_cast<uint32_t>(__double_as_longlong(e.y));
        r.memok = memok;
        sim_fast(S.sim, S.sf, S.val, S.lg2, r, dv, act, cost, ok);
      } else {
        sim_dev(S, dv, act, cost, ok);
      }
      if (!pin) {
        ok = false;
        raw = ~0ull;
      }
      if (A.d_raw) A.d_raw[j] = raw;
      if (!ok && A.d_scores) A.d_scores[j] = -INFINITY;
    }
    // warp-aggregated append of the valid lanes
    const unsigned vb = __ballot_sync(0xffffffffu, in && ok);
    if (vb) {
      unsigned long long wbase = 0;
      if (lane == 0) wbase = atomicAdd(L.count, static_cast<unsigned long long>(__popc(vb)));
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (in && ok) {
        const uint64_t slot = wbase + __popc(vb & ((1u << lane) - 1u));
        L.cvi[slot] = static_cast<uint32_t>(pcvi);
        L.j[slot] = static_cast<uint32_t>(j);
        L.m0[slot] = ENS ? ensemble_m0_dev(S.ens_tab, S.ens_c0, S.d, dv.w[0], dv.w[1], dv.w[2]) : log(cost);
        L.dv0[slot] = dv.w[0];
        L.dv1[slot] = dv.w[1];
        L.dv2[slot] = dv.w[2];
      }
      // valid count straight into shared memory (a RED, no return value): a per-lane 64-bit
      // counter live across the loop was spilled, and its reload cost ~7 % of the kernel's samples
      if (lane == 0) atomicAdd(&blk_valid, static_cast<unsigned int>(__popc(vb)));
    }
  }
  __syncthreads();
  if (tid == 0 && blk_valid) {
    atomicAdd(valid_total, static_cast<unsigned long long>(blk_valid));
    if (A.d_valid_count) atomicAdd(reinterpret_cast<unsigned long long*>(A.d_valid_count), static_cast<unsigned long long>(blk_valid));
  }
}

}  // namespace as
