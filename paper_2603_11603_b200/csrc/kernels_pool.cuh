// Device-resident sharded exchange: every rank packs its refined
// pool into a device buffer, one all_gather_into_tensor (NCCL over NVLink) concatenates the ranks'
// buffers, and the merge + global certificate run on the device -- the pools never pass through
// host memory; only the final top-k (k + 2 entries) is read back.
//
// Packed pool (PoolEntry = {double score; uint64 raw}, 16 B), cap + 2 entries:
//   [0] header {score = number of entries n (as double), raw = 1 if locally certified}
//   [1] cut: an entry that every candidate this rank scored but did not export ranks after or
//       equals in the total order (score = an upper bound on its score; -INF = nothing dropped)
//   [2, 2 + n) the refined entries, ordered (score desc, raw asc), one per configuration;
//   [2 + n, 2 + cap) filler {-INF, UINT64_MAX}.
// Order: PAPER.md:265 top-K re-evaluation, ties by the lower raw index (R11).
#pragma once
#include "kernels.cuh"

namespace as {

struct PoolEntry {
  double score;
  unsigned long long raw;
};
constexpr int POOL_THREADS = 1024;

__device__ __forceinline__ bool pe_before(const PoolEntry& a, const PoolEntry& b) {   // a strictly first
  return a.score > b.score || (a.score == b.score && a.raw < b.raw);
}
__device__ __forceinline__ PoolEntry pe_none() { return PoolEntry{-INFINITY, ~0ull}; }

// bitonic sort of buf[0, n2) into the total order (filler last); all threads of the block
__device__ __forceinline__ void pe_bitonic(PoolEntry* buf, int n2) {
  for (int k = 2; k <= n2; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (n2 >> 1); i += blockDim.x) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo | j;
        const bool asc = (lo & k) == 0;
        const PoolEntry a = buf[lo], b = buf[hi];
        if (pe_before(b, a) == asc) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
      __syncthreads();
    }
}

// Pack this rank's refined pool (refine_kernel output: n_pool scores / raws; the running cut key).
// n2 = next power of two >= n_pool; dynamic smem n2 * 16 B.  flag_out (device int): 1 if the
// local top-k is certified (the k-th entry precedes the cut), so the host can grow k' without
// reading the pool.
__global__ void __launch_bounds__(POOL_THREADS)
pool_pack_kernel(DevSpace S, const double* ref_score, const uint64_t* ref_raw, const int* pool_n, const uint64_t* cut_key,
                 int n2, int k, int cap, PoolEntry* out, int* flag_out) {
  extern __shared__ __align__(16) PoolEntry pbuf[];
  const int n_pool = *pool_n;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    PoolEntry e = pe_none();
    if (i < n_pool && isfinite(ref_score[i])) e = PoolEntry{ref_score[i], ref_raw[i]};
    pbuf[i] = e;
  }
  __syncthreads();
  pe_bitonic(pbuf, n2);
  if (threadIdx.x == 0) {
    PoolEntry cut = pe_none();
    const uint64_t key = *cut_key;
    if (key != KEY_NONE) {
      DV dv;
      uint32_t act;
      uint64_t raw;
      decode_dev(S, key & 0xFFFFFFFFull, dv, act, raw);
      const uint32_t ord = ~static_cast<uint32_t>(key >> 32);
      const uint32_t u = (ord & 0x80000000u) ? (ord & 0x7FFFFFFFu) : ~ord;
      cut = PoolEntry{static_cast<double>(__uint_as_float(u)), raw};
    }
    // one entry per configuration (equal raws are adjacent after the sort), at most cap exported;
    // the best entry not exported bounds every other dropped one
    int n = 0;
    unsigned long long last = ~0ull;
    bool first = true;
    for (int i = 0; i < n2; ++i) {
      const PoolEntry e = pbuf[i];
      if (e.raw == ~0ull && e.score == -INFINITY) break;
      if (!first && e.raw == last) continue;
      first = false;
      last = e.raw;
      if (n < cap) {
        out[2 + n] = e;
        ++n;
      } else {
        if (pe_before(e, cut)) cut = e;
        break;
      }
    }
    for (int i = n; i < cap; ++i) out[2 + i] = pe_none();
    const bool cert = (cut.score == -INFINITY && cut.raw == ~0ull) || (n >= k && pe_before(out[2 + k - 1], cut));
    out[0] = PoolEntry{static_cast<double>(n), cert ? 1ull : 0ull};
    out[1] = cut;
    *flag_out = cert ? 1 : 0;
  }
}

// Merge n_pools gathered packed pools ([n_pools][cap + 2]) into the global top-k with the global
// certificate: out[0] = {n, certified}, out[1] = the best cut over all ranks, out[2, 2 + k) entries.
// buf: n2 = next_pow2(n_pools * cap) entries of scratch (shared memory when it fits, else global).
__global__ void __launch_bounds__(POOL_THREADS)
pool_merge_kernel(const PoolEntry* pools, int n_pools, int cap, int k, int n2, PoolEntry* gbuf, PoolEntry* out) {
  extern __shared__ __align__(16) PoolEntry mbuf[];
  PoolEntry* buf = gbuf != nullptr ? gbuf : mbuf;
  const int stride = cap + 2;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    PoolEntry e = pe_none();
    if (i < n_pools * cap) {
      const int p = i / cap, j = i - p * cap;
      if (j < static_cast<int>(pools[static_cast<size_t>(p) * stride].score)) e = pools[static_cast<size_t>(p) * stride + 2 + j];
    }
    buf[i] = e;
  }
  __syncthreads();
  pe_bitonic(buf, n2);
  if (threadIdx.x == 0) {
    PoolEntry cut = pe_none();
    bool any_cut = false;
    for (int p = 0; p < n_pools; ++p) {
      const PoolEntry c = pools[static_cast<size_t>(p) * stride + 1];
      if (c.score != -INFINITY) {
        if (!any_cut || pe_before(c, cut)) cut = c;
        any_cut = true;
      }
    }
    int n = 0, total = 0;
    unsigned long long last = ~0ull;
    for (int i = 0; i < n2; ++i) {
      const PoolEntry e = buf[i];
      if (e.raw == ~0ull && e.score == -INFINITY) break;
      if (total > 0 && e.raw == last) continue;     // the same configuration from two pools
      last = e.raw;
      ++total;
      if (n < k) out[2 + n++] = e;
      else break;
    }
    for (int i = n; i < k; ++i) out[2 + i] = pe_none();
    const bool cert = !any_cut || (n >= k && pe_before(out[2 + k - 1], cut));
    out[0] = PoolEntry{static_cast<double>(n), cert ? 1ull : 0ull};
    out[1] = cut;
  }
}

}  // namespace as
