// numeric.cuh -- steps a6 (numeric hash accumulation) and a7 (optional sort).
// "In numeric phase, however, we need to store the resulting value data.
// Once the computation on the hash table finishes, the results are sorted by
// column indices in ascending order (if necessary), and stored to memory as
// output.".  Table size T = lowest 2^n >= 2 nnz(c_i) (reading R6).
#pragma once
#include "spg_internal.cuh"
#include "symbolic.cuh"

namespace spg {

// Shared-memory tables: chunked probing (probe_chunk).
__device__ __forceinline__ uint32_t num_probe_smem(uint32_t *keys, uint32_t c, int logT) {
  bool isnew = false;
  return probe_chunk(keys, c, logT, &isnew);
}

// Probe for key c, inserting it if absent; returns its slot (global tables).
__device__ __forceinline__ uint32_t num_probe(uint32_t *keys, uint32_t c, int logT) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
    const uint32_t k = ((volatile uint32_t *)keys)[h];
    if (k == c) return h;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(keys + h, kEmpty, c);
      if (old == kEmpty || old == c) return h;
    }
    h = (h + 1u) & mask;
  }
}

// Lanes of a round holding the same key c combine their values into the
// lowest such lane; returns true for the lanes that then hold a key to apply
// (active, first of their key).  Summation order inside a round is free
// (reading R4).
__device__ __forceinline__ bool warp_combine(bool act, uint32_t c, double &v) {
  const int lane = lane_id();
  const unsigned grp = __match_any_sync(kFull, act ? c : (0x80000000u | lane));
  const int leader = __ffs(grp) - 1;
  const int gmax = (int)__reduce_max_sync(kFull, (unsigned)__popc(grp));
  if (gmax > 1) {
    unsigned rem = lane == leader ? grp & ~(1u << lane) : 0u;
    for (int it = 1; it < gmax; ++it) {
      const int src = rem ? __ffs(rem) - 1 : lane;
      const double o = __shfl_sync(kFull, v, src);
      if (rem) {
        v += o;
        rem &= rem - 1;
      }
    }
  }
  return act && lane == leader;
}

// Warp emit of a warp-private table keys/vals[0, T) holding nnz keys to
// out_base: unsorted = ballot compaction in slot order; sorted (a7) =
// bucket (counting) sort: buckets b(c) = (c - min) >> sh are monotone in the
// column, T buckets for nnz <= T/2 keys, each key's position = bucket offset
// + its rank among the (few) keys of its bucket.  cnt[T] is scratch.
__device__ __forceinline__ void warp_emit(uint32_t *keys, double *vals, uint32_t *cnt, int T,
                                          int logT, int nnz, int64_t rp0,
                                          int32_t *__restrict__ c_col,
                                          double *__restrict__ c_val, int sorted) {
  const int lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  if (!sorted) {
    int base = 0;
    for (int s0 = 0; s0 < T; s0 += 32) {
      const uint32_t k = keys[s0 + lane];
      const bool occ = k != kEmpty;
      const unsigned bal = __ballot_sync(kFull, occ);
      if (occ) {
        const int64_t o = rp0 + base + __popc(bal & lt_mask);
        c_col[o] = (int32_t)k;
        c_val[o] = vals[s0 + lane];
      }
      base += __popc(bal);
    }
  } else {
    // a7: ascending columns by a bucket (counting) sort.  Buckets
    // are monotone in the column: b(c) = (c - min) >> sh, T buckets for
    // nnz <= T/2 keys; each key's position = bucket offset + its rank
    // among the (few) keys of its bucket.
    // 1. compact occupied slots to the front (destination <= source)
    int base = 0;
    for (int s0 = 0; s0 < T; s0 += 32) {
      const uint32_t k = keys[s0 + lane];
      const double v = vals[s0 + lane];
      const bool occ = k != kEmpty;
      const unsigned bal = __ballot_sync(kFull, occ);
      __syncwarp();
      if (occ) {
        const int d = base + __popc(bal & lt_mask);
        keys[d] = k;
        vals[d] = v;
      }
      base += __popc(bal);
      __syncwarp();
    }
    // 2. key range and bucket shift
    unsigned mn = 0xFFFFFFFFu, mx = 0u;
    for (int e = lane; e < nnz; e += 32) {
      const unsigned k = keys[e];
      mn = k < mn ? k : mn;
      mx = k > mx ? k : mx;
    }
    mn = __reduce_min_sync(kFull, mn);
    mx = __reduce_max_sync(kFull, mx);
    int sh = log2_ceil64(uint64_t(mx - mn) + 1) - logT;
    sh = sh < 0 ? 0 : sh;
    for (int b = lane; b < T; b += 32) cnt[b] = 0u;
    __syncwarp();
    uint32_t *loc = reinterpret_cast<uint32_t *>(vals + (T >> 1));  // free half
    uint32_t *grp = keys + (T >> 1);                                  // free half
    for (int e = lane; e < nnz; e += 32) loc[e] = atomicAdd(cnt + ((keys[e] - mn) >> sh), 1u);
    __syncwarp();
    // 3. exclusive scan of the bucket counts, 32 consecutive buckets per step
    //    (lane l reads bucket q + l: conflict-free)
    int carry = 0;
    for (int q = 0; q < T; q += 32) {
      const int v = (int)cnt[q + lane];
      const int incl = warp_incl_scan(v);
      cnt[q + lane] = (uint32_t)(carry + incl - v);
      carry += __shfl_sync(kFull, incl, 31);
    }
    __syncwarp();
    // 4. group keys by bucket, 5. rank inside the bucket and store
    for (int e = lane; e < nnz; e += 32) {
      const uint32_t k = keys[e];
      grp[cnt[(k - mn) >> sh] + loc[e]] = k;
    }
    __syncwarp();
    for (int e = lane; e < nnz; e += 32) {
      const uint32_t k = keys[e];
      const uint32_t b = (k - mn) >> sh;
      const int lo = (int)cnt[b];
      const int hi = (int)b + 1 < T ? (int)cnt[b + 1] : nnz;
      int rnk = 0;
      for (int q = lo; q < hi; ++q) rnk += grp[q] < k;
      c_col[rp0 + lo + rnk] = (int32_t)k;
      c_val[rp0 + lo + rnk] = vals[e];
    }
  }
}

// ---------------------------------------------------------------------------
// W tier: one warp per row, warp-private keys[TMAX] + vals[TMAX] (+ cnt[TMAX]
// bucket counters for the sort) in smem.
// Distinct keys of one round go to distinct slots, so the value add is a
// plain read-modify-write; lanes that share a key in a round (found with
// __match_any_sync) use the atomic add.  Rounds are separated by __syncwarp.
// ---------------------------------------------------------------------------
template <int TMAX, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_num_warp(const int32_t *__restrict__ rows,
                                                         int64_t nrows, DevCSR A, DevCSR B,
                                                         const int64_t *__restrict__ flop,
                                                         const int64_t *__restrict__ c_rp,
                                                         int32_t *__restrict__ c_col,
                                                         double *__restrict__ c_val,
                                                         int sorted) {
  extern __shared__ double s_dyn_f64[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *vals = s_dyn_f64 + w * TMAX;
  uint32_t *keys = reinterpret_cast<uint32_t *>(s_dyn_f64 + WARPS * TMAX) + w * TMAX;
  uint32_t *cnt = reinterpret_cast<uint32_t *>(s_dyn_f64 + WARPS * TMAX) + WARPS * TMAX + w * TMAX;
  for (int64_t r = int64_t(blockIdx.x) * WARPS + w; r < nrows; r += int64_t(gridDim.x) * WARPS) {
    const int i = rows[r];
    const int64_t rp0 = c_rp[i];
    const int nnz = (int)(c_rp[i + 1] - rp0);
    const int logT = num_log2(nnz);
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) { keys[s] = kEmpty; vals[s] = 0.0; }
    __syncwarp();
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    if (use_seq(flop[i], ae - as)) {
      // keys of a round are distinct: plain read-modify-write of the value
      for_row<true, true, 2>(A, B, as, ae, 0, 1, [&](bool act, uint32_t c, double v) {
        if (act) vals[num_probe(keys, c, logT)] += v;   // c_ij <- c_ij + value (l.8)
        __syncwarp();
      });
    } else {
      for_row<false, true, 2>(A, B, as, ae, 0, 1, [&](bool act, uint32_t c, double v) {
        uint32_t slot = 0;
        if (act) slot = num_probe(keys, c, logT);
        const unsigned grp = __match_any_sync(kFull, act ? c : (0x80000000u | lane));
        if (act) {
          if (__popc(grp) == 1) vals[slot] += v;   // c_ij <- c_ij + value (l.8)
          else atomicAdd(vals + slot, v);
        }
        __syncwarp();
      });
    }
    warp_emit(keys, vals, cnt, T, logT, nnz, rp0, c_col, c_val, sorted);
    __syncwarp();
  }
}

// Block-wide unordered compaction of occupied slots of a table into C row.
__device__ __forceinline__ void block_emit_unsorted(const uint32_t *keys, const double *vals,
                                                    int64_t T, int64_t rp0, int32_t *c_col,
                                                    double *c_val, int *s_cnt) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t s0 = int64_t(threadIdx.x & ~31); s0 < T; s0 += blockDim.x) {
    const int64_t s = s0 + lane;
    const uint32_t k = s < T ? keys[s] : kEmpty;
    const bool occ = k != kEmpty;
    const unsigned bal = __ballot_sync(kFull, occ);
    int base = 0;
    if (lane == 0 && bal) base = atomicAdd(s_cnt, __popc(bal));
    base = __shfl_sync(kFull, base, 0);
    if (occ) {
      const int64_t o = rp0 + base + __popc(bal & lt_mask);
      c_col[o] = (int32_t)k;
      c_val[o] = vals[s];
    }
  }
}

__device__ __forceinline__ int block_excl_scan_int(int v, int *s_warp, int *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int incl = warp_incl_scan(v);
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int x = lane < NW ? s_warp[lane] : 0;
    const int xi = warp_incl_scan(x);
    if (lane < NW) s_warp[lane] = xi - x;
    if (lane == 31) s_warp[32] = xi;
  }
  __syncthreads();
  const int r = s_warp[w] + incl - v;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

// a7 for a block-shared table: the row's nnz <= T/2 (key, value)
// pairs sit compacted in keys/vals[0, nnz); store them to C at rp0 in
// ascending column order by a bucket (counting) sort: T/2 buckets monotone in
// the column, b(c) = (c - min) >> sh; position = bucket offset + rank among
// the few keys of the bucket.  Scratch: keys[T/2, T) (bucket counters) and
// vals[T/2, T) (per-key rank in bucket, keys grouped by bucket); s_red[66].
__device__ __forceinline__ void block_bucket_sort_store(const uint32_t *keys, const double *vals,
                                                        int T, int nnz, int64_t rp0,
                                                        int32_t *__restrict__ c_col,
                                                        double *__restrict__ c_val, int *s_red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int NB = T >> 1;
  uint32_t *cnt = const_cast<uint32_t *>(keys) + NB;
  uint32_t *loc = reinterpret_cast<uint32_t *>(const_cast<double *>(vals) + NB);
  uint32_t *grp = loc + NB;
  unsigned mn = 0xFFFFFFFFu, mx = 0u;
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    const unsigned k = keys[e];
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  mn = __reduce_min_sync(kFull, mn);
  mx = __reduce_max_sync(kFull, mx);
  if (lane == 0) { s_red[w] = (int)mn; s_red[32 + w] = (int)mx; }
  for (int b = threadIdx.x; b < NB; b += blockDim.x) cnt[b] = 0u;
  __syncthreads();
  if (w == 0) {
    unsigned a = lane < NW ? (unsigned)s_red[lane] : 0xFFFFFFFFu;
    unsigned z = lane < NW ? (unsigned)s_red[32 + lane] : 0u;
    a = __reduce_min_sync(kFull, a);
    z = __reduce_max_sync(kFull, z);
    if (lane == 0) { s_red[64] = (int)a; s_red[65] = (int)z; }
  }
  __syncthreads();
  mn = (unsigned)s_red[64];
  mx = (unsigned)s_red[65];
  int sh = log2_ceil64(uint64_t(mx - mn) + 1) - (log2_ceil64(uint64_t(NB)));
  sh = sh < 0 ? 0 : sh;
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) loc[e] = atomicAdd(cnt + ((keys[e] - mn) >> sh), 1u);
  __syncthreads();
  // exclusive scan of cnt[0, NB): thread owns a contiguous range
  const int per = (NB + blockDim.x - 1) / blockDim.x;
  const int b0 = min(NB, (int)threadIdx.x * per), b1 = min(NB, b0 + per);
  int mine = 0;
  for (int b = b0; b < b1; ++b) mine += (int)cnt[b];
  int tot;
  int ex = block_excl_scan_int(mine, s_red, &tot);
  for (int b = b0; b < b1; ++b) {
    const int v = (int)cnt[b];
    cnt[b] = (uint32_t)ex;
    ex += v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    const uint32_t k = keys[e];
    grp[cnt[(k - mn) >> sh] + loc[e]] = k;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nnz; e += blockDim.x) {
    const uint32_t k = keys[e];
    const uint32_t b = (k - mn) >> sh;
    const int lo = (int)cnt[b];
    const int hi = (int)b + 1 < NB ? (int)cnt[b + 1] : nnz;
    int rnk = 0;
    for (int q = lo; q < hi; ++q) rnk += grp[q] < k;
    c_col[rp0 + lo + rnk] = (int32_t)k;
    c_val[rp0 + lo + rnk] = vals[e];
  }
}

// ---------------------------------------------------------------------------
// B tier: one block per row, keys/vals of T slots in dynamic smem, shared by
// the block (atomic CAS for keys, atomic fp64 add for values).  Sorted output:
// emit unordered into C, reload the row into smem, bucket-sort it into C (a7).
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_num_block(const int32_t *__restrict__ rows,
                                                       int64_t nrows, DevCSR A, DevCSR B,
                                                       const int64_t *__restrict__ flop,
                                                       const int64_t *__restrict__ c_rp,
                                                       int32_t *__restrict__ c_col,
                                                       double *__restrict__ c_val, int sorted,
                                                       int tmax) {
  extern __shared__ double s_dyn_f64[];
  __shared__ int s_cnt;
  __shared__ int s_red[66];
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5;
  double *vals = s_dyn_f64;
  uint32_t *keys = reinterpret_cast<uint32_t *>(s_dyn_f64 + tmax);
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int64_t rp0 = c_rp[i];
    const int nnz = (int)(c_rp[i + 1] - rp0);
    const int logT = num_log2(nnz);
    const int T = 1 << logT;
    for (int s = threadIdx.x; s < T; s += THREADS) { keys[s] = kEmpty; vals[s] = 0.0; }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto acc = [&](bool act, uint32_t c, double v) {
        if (act) atomicAdd(vals + num_probe_smem(keys, c, logT), v);  // c_ij <- c_ij + value (l.8)
      };
      auto acc_comb = [&](bool act, uint32_t c, double v) {  // keys may repeat in a round
        if (warp_combine(act, c, v)) atomicAdd(vals + num_probe_smem(keys, c, logT), v);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, true>(A, B, as, ae, w, NW, acc);
      else for_row<false, true>(A, B, as, ae, w, NW, acc_comb);
    }
    __syncthreads();
    block_emit_unsorted(keys, vals, T, rp0, c_col, c_val, &s_cnt);
    if (sorted) {
      __syncthreads();
      for (int s = threadIdx.x; s < nnz; s += THREADS) {
        keys[s] = (uint32_t)c_col[rp0 + s];
        vals[s] = c_val[rp0 + s];
      }
      __syncthreads();
      block_bucket_sort_store(keys, vals, T, nnz, rp0, c_col, c_val, s_red);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// G tier: one block per row, keys/vals in a per-block global slab (L2
// atomics: CAS for keys, native fp64 RED for values).  Sorted output by a
// bitmap rank over column chunks of kRankBits: set a bit per present column,
// prefix-popcount, each key's output position is its rank.
// ---------------------------------------------------------------------------
constexpr int kRankBits = 1 << 20;               // columns per rank chunk
constexpr int kRankWords = kRankBits / 32;       // 32768 words = 128 KB
constexpr int kRankGroup = 64;                   // words per u16 prefix group
constexpr int kRankGroups = kRankWords / kRankGroup;
constexpr size_t kRankSmem = size_t(kRankWords) * 4 + size_t(kRankWords) * 2 +
                             size_t(kRankGroups) * 4;

// Sorted emit by bitmap rank (block-wide): the keys of table [0, T) that lie
// in [cbase, cbase + nbits) (nbits <= 32 * words of bm) are written to
// out_col/out_val at out_base + (number of smaller keys in the range).
// Returns the number of such keys (same value in every thread).
__device__ __forceinline__ int block_rank_emit(const uint32_t *keys, const double *vals,
                                               int64_t T, int64_t cbase, int64_t nbits,
                                               uint32_t *bm, uint16_t *wpre, int *gpre,
                                               int *s_tot, int64_t out_base,
                                               int32_t *__restrict__ c_col,
                                               double *__restrict__ c_val) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int nwords = (int)((nbits + 31) >> 5);
  for (int s = threadIdx.x; s < nwords; s += blockDim.x) bm[s] = 0u;
  __syncthreads();
  for (int64_t s = threadIdx.x; s < T; s += blockDim.x) {
    const uint32_t k = keys[s];
    if (k != kEmpty && int64_t(k) >= cbase && int64_t(k) - cbase < nbits) {
      const uint32_t off = (uint32_t)(int64_t(k) - cbase);
      atomicOr(bm + (off >> 5), 1u << (off & 31u));
    }
  }
  __syncthreads();
  const int ngroups = (nwords + kRankGroup - 1) / kRankGroup;
  for (int g = w; g < ngroups; g += NW) {  // u16 prefix inside each 64-word group
    const int w0 = g * kRankGroup + 2 * lane;
    const int c0 = w0 < nwords ? __popc(bm[w0]) : 0;
    const int c1 = w0 + 1 < nwords ? __popc(bm[w0 + 1]) : 0;
    const int incl = warp_incl_scan(c0 + c1);
    const int ex = incl - c0 - c1;
    if (w0 < nwords) wpre[w0] = (uint16_t)ex;
    if (w0 + 1 < nwords) wpre[w0 + 1] = (uint16_t)(ex + c0);
    if (lane == 31) gpre[g] = incl;
  }
  __syncthreads();
  if (w == 0) {  // exclusive scan of the group totals
    int carry = 0;
    for (int g0 = 0; g0 < ngroups; g0 += 32) {
      const int g = g0 + lane;
      const int v = g < ngroups ? gpre[g] : 0;
      const int incl = warp_incl_scan(v);
      if (g < ngroups) gpre[g] = carry + incl - v;
      carry += __shfl_sync(kFull, incl, 31);
    }
    if (lane == 0) *s_tot = carry;
  }
  __syncthreads();
  for (int64_t s = threadIdx.x; s < T; s += blockDim.x) {
    const uint32_t k = keys[s];
    if (k != kEmpty && int64_t(k) >= cbase && int64_t(k) - cbase < nbits) {
      const uint32_t off = (uint32_t)(int64_t(k) - cbase);
      const uint32_t wd = off >> 5;
      const int pos = gpre[wd / kRankGroup] + wpre[wd] +
                      __popc(bm[wd] & ((1u << (off & 31u)) - 1u));
      c_col[out_base + pos] = (int32_t)k;
      c_val[out_base + pos] = vals[s];
    }
  }
  const int tot = *s_tot;
  __syncthreads();
  return tot;
}

// Emit of a part's table from its insertion list slot_of[0, n): unsorted =
// list order (coalesced stores); sorted = bitmap rank over [cbase, cbase +
// nbits), nbits <= 32 * words of bm.
__device__ __forceinline__ void block_list_emit(const uint32_t *keys, const double *vals,
                                                const uint16_t *slot_of, int n, int64_t cbase,
                                                int64_t nbits, uint32_t *bm, uint16_t *wpre,
                                                int *gpre, int *s_tot, int64_t out_base,
                                                int32_t *__restrict__ c_col,
                                                double *__restrict__ c_val, int sorted) {
  if (!sorted) {
    for (int p = threadIdx.x; p < n; p += blockDim.x) {
      const int s = slot_of[p];
      c_col[out_base + p] = (int32_t)keys[s];
      c_val[out_base + p] = vals[s];
    }
    return;
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int nwords = (int)((nbits + 31) >> 5);
  for (int q = threadIdx.x; q < nwords; q += blockDim.x) bm[q] = 0u;
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const uint32_t off = (uint32_t)(int64_t(keys[slot_of[p]]) - cbase);
    atomicOr(bm + (off >> 5), 1u << (off & 31u));
  }
  __syncthreads();
  const int ngroups = (nwords + kRankGroup - 1) / kRankGroup;
  for (int g = w; g < ngroups; g += NW) {
    const int w0 = g * kRankGroup + 2 * lane;
    const int c0 = w0 < nwords ? __popc(bm[w0]) : 0;
    const int c1 = w0 + 1 < nwords ? __popc(bm[w0 + 1]) : 0;
    const int incl = warp_incl_scan(c0 + c1);
    const int ex = incl - c0 - c1;
    if (w0 < nwords) wpre[w0] = (uint16_t)ex;
    if (w0 + 1 < nwords) wpre[w0 + 1] = (uint16_t)(ex + c0);
    if (lane == 31) gpre[g] = incl;
  }
  __syncthreads();
  if (w == 0) {
    int carry = 0;
    for (int g0 = 0; g0 < ngroups; g0 += 32) {
      const int g = g0 + lane;
      const int v = g < ngroups ? gpre[g] : 0;
      const int incl = warp_incl_scan(v);
      if (g < ngroups) gpre[g] = carry + incl - v;
      carry += __shfl_sync(kFull, incl, 31);
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    const int s = slot_of[p];
    const uint32_t k = keys[s];
    const uint32_t off = (uint32_t)(int64_t(k) - cbase);
    const uint32_t wd = off >> 5;
    const int pos = gpre[wd / kRankGroup] + wpre[wd] + __popc(bm[wd] & ((1u << (off & 31u)) - 1u));
    c_col[out_base + pos] = (int32_t)k;
    c_val[out_base + pos] = vals[s];
  }
  (void)s_tot;
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_num_global(const int32_t *__restrict__ rows,
                                                        int64_t nrows, DevCSR A, DevCSR B,
                                                        const int64_t *__restrict__ flop,
                                                        const int64_t *__restrict__ c_rp,
                                                        int32_t *__restrict__ c_col,
                                                        double *__restrict__ c_val, int sorted,
                                                        uint32_t *__restrict__ slab_keys,
                                                        double *__restrict__ slab_vals,
                                                        int64_t slabT) {
  extern __shared__ uint32_t s_dyn_u32[];
  __shared__ int s_cnt;
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5;
  uint32_t *keys = slab_keys + int64_t(blockIdx.x) * slabT;
  double *vals = slab_vals + int64_t(blockIdx.x) * slabT;
  uint32_t *bm = s_dyn_u32;                                          // [kRankWords]
  uint16_t *wpre = reinterpret_cast<uint16_t *>(bm + kRankWords);    // [kRankWords]
  int *gpre = reinterpret_cast<int *>(wpre + kRankWords);           // [kRankGroups]
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int64_t rp0 = c_rp[i];
    const int64_t nnz = c_rp[i + 1] - rp0;
    const int logT = num_log2(nnz);
    const int64_t T = int64_t(1) << logT;
    for (int64_t s = threadIdx.x; s < T; s += THREADS) { keys[s] = kEmpty; vals[s] = 0.0; }
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto acc = [&](bool act, uint32_t c, double v) {
        if (act) atomicAdd(vals + num_probe(keys, c, logT), v);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, true>(A, B, as, ae, w, NW, acc);
      else for_row<false, true>(A, B, as, ae, w, NW, acc);
    }
    __syncthreads();
    if (!sorted) {
      block_emit_unsorted(keys, vals, T, rp0, c_col, c_val, &s_cnt);
    } else {
      int64_t done = 0;
      for (int64_t cbase = 0; cbase < B.ncols; cbase += kRankBits) {
        const int64_t nbits = (B.ncols - cbase) < kRankBits ? (B.ncols - cbase) : kRankBits;
        done += block_rank_emit(keys, vals, T, cbase, nbits, bm, wpre, gpre, &s_cnt, rp0 + done,
                                c_col, c_val);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// G tier, column-range parts (B rows sorted, parts from the BM symbolic): one
// block per row at a time (dynamic row queue), the row's parts in column
// order.  For part [lo, hi) every a_ik's B row contributes the segment of
// columns in [lo, hi): it starts where the previous part's segment ended and
// ends at the first column >= hi (galloping search).  The part's <= kPartKeys
// keys are accumulated in an smem hash table of kPartT slots and emitted at
// C_row_ptr[i] + (keys of the row before lo) -- in order, by a bitmap rank
// over [lo, lo + kPartWidth), when sorted.  No global atomics.
// ---------------------------------------------------------------------------
constexpr int kPartT = 2 * kPartKeys;               // table slots (load <= 1/2)
constexpr int kSegSmem = 1024;                      // a_ik whose segments live in smem
constexpr int kSegBytes = 32;                       // pos, rend (int64), a (f64), nx, pre (int32)
constexpr int kPartRankWords = int(kPartWidth / 32);
constexpr size_t kPartSmem = size_t(kPartT) * 12 + size_t(kSegSmem) * kSegBytes + 16 +
                             size_t(kPartRankWords) * 6 +
                             size_t(kPartRankWords / kRankGroup) * 4 + size_t(kPartKeys) * 2;

// Per-entry state of a row walked part by part (smem, or per-block global
// scratch for rows with many a_ik).  Entry j = the row's j-th a_ik; its B row
// occupies [B.rp[k], B.rp[k+1]) = [.., rend[j]).
struct Segs {
  int64_t *pos;   // absolute start of the current part's segment in B.col / B.val
  int64_t *rend;  // absolute end of the B row
  double *a;      // a_ik
  int32_t *nx;    // length of the current part's segment
  int32_t *pre;   // exclusive prefix of nx over j (na + 1 entries)
};

__device__ __forceinline__ Segs segs_at(void *base, int cap) {
  Segs g;
  g.pos = reinterpret_cast<int64_t *>(base);
  g.rend = g.pos + cap;
  g.a = reinterpret_cast<double *>(g.rend + cap);
  g.nx = reinterpret_cast<int32_t *>(g.a + cap);
  g.pre = g.nx + cap;  // cap + 1 entries
  return g;
}

// Entry state at the start of row [as, as + na): one pass, cached for all parts.
__device__ __forceinline__ void seg_init(const DevCSR &A, const DevCSR &B, int64_t as, int na,
                                         const Segs &sg, int tid, int nth) {
  for (int j = tid; j < na; j += nth) {
    const int k = __ldg(A.col + as + j);
    sg.pos[j] = __ldg(B.rp + k);
    sg.rend[j] = __ldg(B.rp + k + 1);
    sg.a[j] = __ldg(A.val + as + j);
    sg.nx[j] = 0;
  }
}

// first q in [s, r) with col[q] >= hi (col sorted), given col[s-1] < hi
__device__ __forceinline__ int64_t gallop_abs(const int32_t *__restrict__ col, int64_t s,
                                              int64_t r, int64_t hi) {
  if (s >= r || int64_t(__ldg(col + s)) >= hi) return s;
  int64_t lo = s, step = 1;  // invariant: col[lo] < hi
  while (lo + step < r && int64_t(__ldg(col + lo + step)) < hi) {
    lo += step;
    step <<= 1;
  }
  int64_t x = lo + 1, y = lo + step < r ? lo + step : r;
  while (x < y) {
    const int64_t m = (x + y) >> 1;
    if (int64_t(__ldg(col + m)) < hi) x = m + 1; else y = m;
  }
  return x;
}

// Segment ends of one part [lo, hi) for all entries of a team of nth threads
// (a block or one warp): nx[j] = (first q >= pos[j] in the B row with
// col[q] >= hi) - pos[j]; the last part takes the rest of every B row.
// Latency-tolerant (the searches are chains of dependent loads):
//  - few entries: G = 2^g lanes per entry run a G-ary search (one ballot per
//    step narrows the range G+1 times: ~log_{G+1}(len) dependent loads);
//  - many entries: a thread takes 4 entries at a time and reads 4 consecutive
//    columns of each (16 independent loads in flight), which settles the short
//    segments of long rows at once; longer ones gallop on.
__device__ __forceinline__ void seg_search(const int32_t *__restrict__ bcol, const Segs &sg, int na,
                                           int64_t hi, bool last, int tid, int nth) {
  // every entry first moves past the previous part's segment (pos += nx)
  if (last) {
    for (int j = tid; j < na; j += nth) {
      const int64_t p = sg.pos[j] + sg.nx[j];
      sg.pos[j] = p;
      sg.nx[j] = (int)(sg.rend[j] - p);
    }
    return;
  }
  int G = 1;
  while (G < 32 && int64_t(G) * 2 * na <= nth) G <<= 1;
  if (G >= 4) {
    const int lane = tid & 31;
    const int gb = lane & ~(G - 1), gl = lane & (G - 1);
    const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << gb);
    const int ngroups = nth / G;
    for (int j = tid / G; j < na; j += ngroups) {  // same j sequence for the whole group
      const int64_t p0 = sg.pos[j] + sg.nx[j];
      int64_t lo = p0, up = sg.rend[j];  // the answer lies in [lo, up]
      while (up > lo) {
        const int64_t len = up - lo;
        if (len <= G) {
          const bool ge = gl < len && int64_t(__ldg(bcol + lo + gl)) >= hi;
          const unsigned b = __ballot_sync(gmask, ge) >> gb;
          lo = b ? lo + __ffs(b) - 1 : up;
          break;
        }
        const int64_t q = lo + (len * (gl + 1)) / (G + 1);  // strictly increasing in gl
        const bool ge = int64_t(__ldg(bcol + q)) >= hi;
        const unsigned b = (__ballot_sync(gmask, ge) >> gb) & (G == 32 ? kFull : ((1u << G) - 1u));
        const int f = b ? __ffs(b) - 1 : G;  // first probe >= hi
        const int64_t nlo = f > 0 ? lo + (len * f) / (G + 1) + 1 : lo;
        if (f < G) up = lo + (len * (f + 1)) / (G + 1);
        lo = nlo;
      }
      __syncwarp(gmask);
      if (gl == 0) {
        sg.pos[j] = p0;
        sg.nx[j] = (int)(lo - p0);
      }
    }
    return;
  }
  for (int j0 = tid; j0 < na; j0 += 4 * nth) {
    int64_t p[4], r[4];
    int32_t c[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * nth;
      p[u] = j < na ? sg.pos[j] + sg.nx[j] : 0;
      r[u] = j < na ? sg.rend[j] : 0;
#pragma unroll
      for (int d = 0; d < 4; ++d)
        c[u][d] = p[u] + d < r[u] ? __ldg(bcol + p[u] + d) : INT32_MAX;  // INT32_MAX >= any hi
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = j0 + u * nth;
      if (j >= na) continue;
      int d = 0;
#pragma unroll
      for (int t = 3; t >= 0; --t)
        if (int64_t(c[u][t]) >= hi) d = t;
      int64_t e;
      if (int64_t(c[u][0]) >= hi) e = p[u];
      else if (int64_t(c[u][3]) >= hi) e = p[u] + d;
      else e = gallop_abs(bcol, p[u] + 4, r[u], hi);
      sg.pos[j] = p[u];
      sg.nx[j] = (int)(e - p[u]);
    }
  }
}

// Number of lanes whose (nondecreasing across lanes) value wv is <= x: 0..32.
__device__ __forceinline__ int count_le(int wv, int x) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const int v = __shfl_sync(kFull, wv, pos + s - 1);
    if (v <= x) pos += s;
  }
  const int last = __shfl_sync(kFull, wv, 31);  // (all lanes shuffle)
  if (pos == 31 && last <= x) pos = 32;
  return pos;
}

// Owner entry of product x (x < P): the last j with pre[j] <= x, searched
// from entry jb (pre[jb] <= every product of the round) in windows of 32
// boundaries pre[jb+1 .. jb+32] loaded by the warp at once.  All lanes call.
__device__ __forceinline__ int part_owner(const int32_t *__restrict__ pre, int na, int jb, int x,
                                          bool act) {
  const int lane = lane_id();
  int own = act ? -1 : 0;
  while (true) {
    const int e = jb + 1 + lane;
    const int wv = e <= na ? pre[e] : INT32_MAX;
    const int c = count_le(wv, x);
    if (own < 0 && c < 32) own = jb + c;
    if (__all_sync(kFull, own >= 0)) break;
    jb += 32;
  }
  return own;
}

// Flat enumeration of the products of one part: product p (0 <= p < P) lies
// in the segment of entry j with pre[j] <= p < pre[j+1].  Rounds [g0, g1) of
// 32 consecutive products, owners found by part_owner windows.
constexpr int kPartChunk = 8;  // rounds a warp takes at a time in the block-part kernel
constexpr int kWalkMinEntries = 512;
constexpr int kWalkU = 2;  // entries a thread walks at once  // rows with >= this many a_ik: entry walk per part

template <int kD = 4, typename F>
__device__ __forceinline__ void for_part_rounds(const DevCSR &B, const Segs &sg, int na, int P,
                                                int g0, int g1, F &&f) {
  if (g0 >= g1) return;
  const int lane = lane_id();
  int jb;  // owner of the next round's first product (warp-uniform)
  {
    const int x = g0 * 32;
    int lo = 0, hi = na;  // last j with pre[j] <= x
    while (hi - lo > 1) {
      const int m = (lo + hi) >> 1;
      if (sg.pre[m] <= x) lo = m; else hi = m;
    }
    jb = lo;
  }
  // batches of kD rounds: owners and gather addresses of all kD rounds first,
  // then the kD gathers (independent loads in flight), then the kD updates
  for (int g = g0; g < g1; g += kD) {
    uint32_t c[kD];
    double v[kD];
    bool act[kD];
    int64_t q[kD];
    double a[kD];
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      const int x = (g + d) * 32 + lane;
      act[d] = (g + d < g1) && x < P;
      const int j = part_owner(sg.pre, na, jb, x, act[d]);
      jb = __shfl_sync(kFull, act[d] ? j : jb, 31);
      q[d] = act[d] ? sg.pos[j] + (x - sg.pre[j]) : 0;
      a[d] = act[d] ? sg.a[j] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      c[d] = act[d] ? (uint32_t)__ldg(B.col + q[d]) : 0u;
      v[d] = act[d] ? __ldg(B.val + q[d]) : 0.0;
    }
#pragma unroll
    for (int d = 0; d < kD; ++d) f(act[d], c[d], a[d] * v[d]);  // a_ik * b_kj (Fig:code_spgemm l.5)
  }
}

// ---------------------------------------------------------------------------
// G tier, column-range BLOCK parts (rows with many a_ik, B rows sorted; parts
// from the BM symbolic): one block per row at a time (dynamic row queue), the
// row's parts in column order.  Per part [lo, hi): every a_ik's B row
// contributes the segment of columns in [lo, hi) -- it starts where the
// previous part's segment ended and ends at the first column >= hi (galloping
// search); one block scan of the segment lengths makes the part's products a
// flat list, cut into equal contiguous ranges of 32-product rounds, one per
// warp.  The part's <= kPartKeys keys are accumulated in an smem hash table
// and emitted at C_row_ptr[i] + (keys of the row before lo) -- in order, by a
// bitmap rank over [lo, lo + kPartWidth), when sorted.  No global atomics.
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_num_part(
    const int32_t *__restrict__ rows, int64_t nrows, DevCSR A, DevCSR B,
    const int64_t *__restrict__ flop, const int64_t *__restrict__ c_rp,
    int32_t *__restrict__ c_col, double *__restrict__ c_val, int sorted,
    const int2 *__restrict__ parts, const int32_t *__restrict__ part_off,
    const int32_t *__restrict__ part_n, char *__restrict__ seg_scratch, int64_t seg_cap,
    unsigned long long *row_counter, int tune, unsigned long long *dbg) {
  extern __shared__ double s_dyn_f64[];
  __shared__ int s_cnt, s_round;
  __shared__ int s_warp[33];
  __shared__ long long s_row;
  double *vals = s_dyn_f64;
  uint32_t *keys = reinterpret_cast<uint32_t *>(vals + kPartT);
  char *seg_smem = reinterpret_cast<char *>(keys + kPartT);
  uint32_t *bm = reinterpret_cast<uint32_t *>(seg_smem + size_t(kSegSmem) * kSegBytes + 16);
  uint16_t *wpre = reinterpret_cast<uint16_t *>(bm + kPartRankWords);
  int *gpre = reinterpret_cast<int *>(wpre + kPartRankWords);
  uint16_t *slot_of = reinterpret_cast<uint16_t *>(gpre + kPartRankWords / kRankGroup);
  const int lane = threadIdx.x & 31;
  while (true) {
    if (threadIdx.x == 0) s_row = (long long)atomicAdd(row_counter, 1ull);
    __syncthreads();
    const int64_t r = s_row;
    if (r >= nrows) break;
    const int i = rows[r];
    const int64_t rp0 = c_rp[i];
    const int nnz = (int)(c_rp[i + 1] - rp0);
    const int64_t as = A.rp[i];
    const int na = (int)(A.rp[i + 1] - as);
    const int np = part_n[i];
    const int2 *pr = parts + part_off[i];
    Segs sg = na <= kSegSmem ? segs_at(seg_smem, kSegSmem)
                             : segs_at(seg_scratch + int64_t(blockIdx.x) * seg_cap * kSegBytes,
                                       (int)seg_cap);
    seg_init(A, B, as, na, sg, threadIdx.x, THREADS);
    const int per = (na + THREADS - 1) / THREADS;  // entries per thread for the scan
    const bool walk = na >= kWalkMinEntries && (tune & 4);  // (entry walk: measurement only)
    for (int p = 0; p < np; ++p) {
      const int2 Pp = pr[p];
      const int64_t hi = p + 1 < np ? int64_t(pr[p + 1].x) : B.ncols;
      const int cnt = (p + 1 < np ? pr[p + 1].y : nnz) - Pp.y;
      const int logT = num_log2(cnt);
      const int T = 1 << logT;
      const bool instr = (tune & 8) && threadIdx.x == 0;
      const long long t0 = instr ? clock64() : 0;
      for (int s = threadIdx.x; s < T; s += THREADS) { keys[s] = kEmpty; vals[s] = 0.0; }
      if (threadIdx.x == 0) {
        s_cnt = 0;
        s_round = 0;
      }
      __syncthreads();  // seg_init / the previous part's pos update are visible
      long long t1 = 0, t2 = 0;
      if (walk) {
        // entry walk (rows with many a_ik: short segments per part): thread
        // per entry, kWalkU entries at a time, 4 columns read ahead each; the
        // products c < hi of the B row are applied in place and pos[j] moves
        // past them.  No search, scan or owner lookup.
        t1 = t2 = instr ? clock64() : 0;
        auto ins = [&](uint32_t c, double v) {
          bool isnew = false;
          const uint32_t slot = probe_chunk(keys, c, logT, &isnew);
          atomicAdd(vals + slot, v);  // c_ij <- c_ij + value (l.8)
          if (isnew) slot_of[atomicAdd(&s_cnt, 1)] = (uint16_t)slot;
        };
        for (int j0 = threadIdx.x; j0 < na; j0 += kWalkU * THREADS) {
          int64_t q[kWalkU], r[kWalkU];
          double aa[kWalkU];
          bool live[kWalkU];
#pragma unroll
          for (int u = 0; u < kWalkU; ++u) {
            const int j = j0 + u * THREADS;
            live[u] = j < na;
            q[u] = live[u] ? sg.pos[j] : 0;
            r[u] = live[u] ? sg.rend[j] : 0;
            aa[u] = live[u] ? sg.a[j] : 0.0;
          }
          while (true) {
            bool any = false;
#pragma unroll
            for (int u = 0; u < kWalkU; ++u) any |= live[u];
            if (!any) break;
            int32_t c[kWalkU][4];
#pragma unroll
            for (int u = 0; u < kWalkU; ++u)
#pragma unroll
              for (int d = 0; d < 4; ++d)
                c[u][d] = (live[u] && q[u] + d < r[u]) ? __ldg(B.col + q[u] + d) : INT32_MAX;
#pragma unroll
            for (int u = 0; u < kWalkU; ++u) {
              if (!live[u]) continue;
              int n = 0;
#pragma unroll
              for (int d = 0; d < 4; ++d) n += int64_t(c[u][d]) < hi;  // sorted: a prefix
              double v[4];
#pragma unroll
              for (int d = 0; d < 4; ++d) v[d] = d < n ? __ldg(B.val + q[u] + d) : 0.0;
#pragma unroll
              for (int d = 0; d < 4; ++d)
                if (d < n) ins((uint32_t)c[u][d], aa[u] * v[d]);  // a_ik * b_kj (l.5)
              q[u] += n;
              if (n < 4) {
                live[u] = false;
                sg.pos[j0 + u * THREADS] = q[u];
              }
            }
          }
        }
      } else {
      seg_search(B.col, sg, na, hi, p + 1 == np, threadIdx.x, THREADS);
      __syncthreads();
      t1 = instr ? clock64() : 0;
      // exclusive prefix of the segment lengths (thread owns entries [t*per, t*per + per))
      const int jlo = min(na, threadIdx.x * per), jhi = min(na, jlo + per);
      int mine = 0;
      for (int j = jlo; j < jhi; ++j) mine += sg.nx[j];
      int P;
      int ex = block_excl_scan_int(mine, s_warp, &P);  // (contains the barriers)
      for (int j = jlo; j < jhi; j += 8) {  // nx loads batched ahead of the pre stores
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = j + u < jhi ? sg.nx[j + u] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j + u < jhi) {
            sg.pre[j + u] = ex;
            ex += v[u];
          }
      }
      if (threadIdx.x == 0) sg.pre[na] = P;
      __syncthreads();
      t2 = instr ? clock64() : 0;
      const int R = (P + 31) >> 5;
      // accumulate: flat rounds of 32 products, equal contiguous ranges of
      // rounds per warp (SPG_TUNE bit 2: chunks from a shared counter; bit 1:
      // combine equal keys of a round first); newly inserted keys are
      // appended to the insertion list
      const bool comb = (tune & 1) != 0;
      auto acc = [&](bool act, uint32_t c, double v) {
        const bool lead = comb ? warp_combine(act, c, v) : act;
        bool isnew = false;
        uint32_t slot = 0;
        if (lead) {
          slot = probe_chunk(keys, c, logT, &isnew);
          if (tune & 48) {  // measurement only (wrong values): 16 racy add, 32 no add
            if (tune & 16) vals[slot] += v;
          } else {
            atomicAdd(vals + slot, v);  // c_ij <- c_ij + value (l.8)
          }
        }
        const unsigned m = __ballot_sync(kFull, isnew);
        if (m) {
          const int leader = __ffs(m) - 1;
          int base = 0;
          if (lane == leader) base = atomicAdd(&s_cnt, __popc(m));
          base = __shfl_sync(kFull, base, leader);
          if (isnew) slot_of[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)slot;
        }
      };
      if (!(tune & 2)) {
        const int w = threadIdx.x >> 5, NW = THREADS / 32;
        for_part_rounds(B, sg, na, P, (int)((int64_t)R * w / NW), (int)((int64_t)R * (w + 1) / NW), acc);
      } else {
        while (true) {
          int g0 = 0;
          if (lane == 0) g0 = atomicAdd(&s_round, kPartChunk);
          g0 = __shfl_sync(kFull, g0, 0);
          if (g0 >= R) break;
          for_part_rounds(B, sg, na, P, g0, min(g0 + kPartChunk, R), acc);
        }
      }
      }
      __syncthreads();  // every warp is done reading this part's segments
      long long t3 = instr ? clock64() : 0;
      const int64_t width = (hi - Pp.x) < kPartWidth ? (hi - Pp.x) : kPartWidth;
      block_list_emit(keys, vals, slot_of, cnt, Pp.x, width, bm, wpre, gpre, &s_cnt, rp0 + Pp.y,
                      c_col, c_val, sorted);
      __syncthreads();
      if (instr) {
        const long long t4 = clock64();
        atomicAdd(dbg + 0, 1ull);                              // parts
        atomicAdd(dbg + 1, (unsigned long long)(t1 - t0));     // init + segment search
        atomicAdd(dbg + 2, (unsigned long long)(t2 - t1));     // scan
        atomicAdd(dbg + 3, (unsigned long long)(t3 - t2));     // accumulate
        atomicAdd(dbg + 4, (unsigned long long)(t4 - t3));     // emit
        atomicAdd(dbg + 5, (unsigned long long)walk);          // parts walked
        atomicAdd(dbg + 6, (unsigned long long)na);            // entries walked
      }
    }
  }
}

// ---------------------------------------------------------------------------
// G tier, WARP parts (rows with <= kWPartMaxEntries a_ik, B rows sorted):
// one warp per row at a time (dynamic row queue), the row's parts of
// kWPartKeys keys in column order, each accumulated in a warp-private smem
// table (plain fp64 read-modify-write; lanes sharing a key in a round found
// with __match_any_sync) and emitted at C_row_ptr[i] + (keys before the part)
// -- sorted by the warp bucket sort when requested.  Segments and the flat
// product list as in the block parts, per warp.
// ---------------------------------------------------------------------------
constexpr int kWPartT = 2 * kWPartKeys;
constexpr size_t kWPartSmemPerWarp =  // multiple of 16 B: 128-bit chunk loads stay aligned
    (size_t(kWPartT) * 16 + size_t(kWPartMaxEntries) * kSegBytes + 16 + 15) & ~size_t(15);

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_num_wpart(
    const int32_t *__restrict__ rows, int64_t nrows, DevCSR A, DevCSR B,
    const int64_t *__restrict__ flop, const int64_t *__restrict__ c_rp,
    int32_t *__restrict__ c_col, double *__restrict__ c_val, int sorted,
    const int2 *__restrict__ parts, const int32_t *__restrict__ part_off,
    const int32_t *__restrict__ part_n, unsigned long long *row_counter) {
  extern __shared__ double s_dyn_f64[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char *base = reinterpret_cast<char *>(s_dyn_f64) + size_t(w) * kWPartSmemPerWarp;
  double *vals = reinterpret_cast<double *>(base);
  uint32_t *keys = reinterpret_cast<uint32_t *>(vals + kWPartT);
  uint32_t *cnt = keys + kWPartT;
  Segs sg = segs_at(cnt + kWPartT, kWPartMaxEntries);
  while (true) {
    long long r = 0;
    if (lane == 0) r = (long long)atomicAdd(row_counter, 1ull);
    r = __shfl_sync(kFull, r, 0);
    if (r >= nrows) break;
    const int i = rows[r];
    const int64_t rp0 = c_rp[i];
    const int nnz = (int)(c_rp[i + 1] - rp0);
    const int64_t as = A.rp[i];
    const int na = (int)(A.rp[i + 1] - as);
    const int np = -part_n[i];
    const int2 *pr = parts + part_off[i];
    seg_init(A, B, as, na, sg, lane, 32);
    __syncwarp();
    for (int p = 0; p < np; ++p) {
      const int2 Pp = pr[p];
      const int64_t hi = p + 1 < np ? int64_t(pr[p + 1].x) : B.ncols;
      const int cntp = (p + 1 < np ? pr[p + 1].y : nnz) - Pp.y;
      const int logT = num_log2(cntp);
      const int T = 1 << logT;
      for (int s = lane; s < T; s += 32) { keys[s] = kEmpty; vals[s] = 0.0; }
      seg_search(B.col, sg, na, hi, p + 1 == np, lane, 32);
      __syncwarp();
      int carry = 0;
      for (int j0 = 0; j0 < na; j0 += 32) {  // exclusive prefix of the segment lengths
        const int j = j0 + lane;
        const int L = j < na ? sg.nx[j] : 0;
        const int incl = warp_incl_scan(L);
        if (j < na) sg.pre[j] = carry + incl - L;
        carry += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) sg.pre[na] = carry;
      __syncwarp();
      const int P = carry;
      for_part_rounds(B, sg, na, P, 0, (P + 31) >> 5, [&](bool act, uint32_t c, double v) {
        uint32_t slot = 0;
        if (act) slot = num_probe_smem(keys, c, logT);
        const unsigned grp = __match_any_sync(kFull, act ? c : (0x80000000u | lane));
        if (act) {
          if (__popc(grp) == 1) vals[slot] += v;  // c_ij <- c_ij + value (l.8)
          else atomicAdd(vals + slot, v);
        }
        __syncwarp();
      });
      warp_emit(keys, vals, cnt, T, logT, cntp, rp0 + Pp.y, c_col, c_val, sorted);
      __syncwarp();
    }
  }
}

}  // namespace spg
