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

// Warp-cooperative bitonic sort of P (power of two) (key, val) pairs in smem.
__device__ __forceinline__ void warp_bitonic(uint32_t *keys, double *vals, int P) {
  const int lane = lane_id();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < (P >> 1); t += 32) {
        const int i0 = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int i1 = i0 + j;
        const bool up = (i0 & k) == 0;
        const uint32_t a = keys[i0], b = keys[i1];
        if ((a > b) == up) {
          keys[i0] = b; keys[i1] = a;
          const double va = vals[i0];
          vals[i0] = vals[i1]; vals[i1] = va;
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void block_bitonic(uint32_t *keys, double *vals, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
        const int i0 = ((t & ~(j - 1)) << 1) | (t & (j - 1));
        const int i1 = i0 + j;
        const bool up = (i0 & k) == 0;
        const uint32_t a = keys[i0], b = keys[i1];
        if ((a > b) == up) {
          keys[i0] = b; keys[i1] = a;
          const double va = vals[i0];
          vals[i0] = vals[i1]; vals[i1] = va;
        }
      }
      __syncthreads();
    }
  }
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

// ---------------------------------------------------------------------------
// B tier: one block per row, keys/vals of T slots in dynamic smem, shared by
// the block (atomic CAS for keys, atomic fp64 add for values).  Sorted output:
// emit unordered into C, reload the row into smem, bitonic sort, store.
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
        if (act) atomicAdd(vals + num_probe_smem(keys, c, logT), v);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, true>(A, B, as, ae, w, NW, acc);
      else for_row<false, true>(A, B, as, ae, w, NW, acc);
    }
    __syncthreads();
    block_emit_unsorted(keys, vals, T, rp0, c_col, c_val, &s_cnt);
    if (sorted) {
      __syncthreads();
      int P = 1;
      while (P < nnz) P <<= 1;
      for (int s = threadIdx.x; s < P; s += THREADS) {
        if (s < nnz) { keys[s] = (uint32_t)c_col[rp0 + s]; vals[s] = c_val[rp0 + s]; }
        else keys[s] = kEmpty;
      }
      __syncthreads();
      block_bitonic(keys, vals, P);
      for (int s = threadIdx.x; s < nnz; s += THREADS) {
        c_col[rp0 + s] = (int32_t)keys[s];
        c_val[rp0 + s] = vals[s];
      }
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
constexpr int kSegBytes = 28;                       // sb, se, pre (int32), sabs (int64), a (f64)
constexpr int kPartRankWords = int(kPartWidth / 32);
constexpr size_t kPartSmem = size_t(kPartT) * 12 + size_t(kSegSmem) * kSegBytes + 16 +
                             size_t(kPartRankWords) * 6 +
                             size_t(kPartRankWords / kRankGroup) * 4 + size_t(kPartKeys) * 2;

// first q in [s, len) with col[q] >= hi (col sorted), searching from s
__device__ __forceinline__ int gallop_lb(const int32_t *__restrict__ col, int s, int len,
                                         int64_t hi) {
  if (s >= len || int64_t(__ldg(col + s)) >= hi) return s;
  int lo = s, step = 1;  // invariant: col[lo] < hi
  while (lo + step < len && int64_t(__ldg(col + lo + step)) < hi) {
    lo += step;
    step <<= 1;
  }
  int a = lo + 1, b = min(lo + step, len);
  while (a < b) {
    const int m = (a + b) >> 1;
    if (int64_t(__ldg(col + m)) < hi) a = m + 1; else b = m;
  }
  return a;
}

// Per-entry segment arrays of a part (smem or global scratch).
struct Segs {
  int32_t *sb, *se, *pre;  // begin / end offsets in the B row; exclusive prefix of lengths
  int64_t *sabs;           // absolute position of the segment start in B.col / B.val
  double *a;               // a_ik
};

__device__ __forceinline__ Segs segs_at(void *base, int cap) {
  Segs g;
  g.sabs = reinterpret_cast<int64_t *>(base);
  g.a = reinterpret_cast<double *>(g.sabs + cap);
  g.sb = reinterpret_cast<int32_t *>(g.a + cap);
  g.se = g.sb + cap;
  g.pre = g.se + cap;  // cap + 1 entries
  return g;
}

// Flat enumeration of the products of one part: product p (0 <= p < P) lies
// in the segment of entry j with pre[j] <= p < pre[j+1].  Rounds [g0, g1) of
// 32 consecutive products; each lane keeps its owner entry j and advances it
// (products of a lane increase by 32 per round).  Two rounds in flight.
template <typename F>
__device__ __forceinline__ void for_part_rounds(const DevCSR &B, const Segs &sg, int na, int P,
                                                int g0, int g1, F &&f) {
  if (g0 >= g1) return;
  const int lane = lane_id();
  int p = g0 * 32 + lane;
  int lo = 0, hi = na;  // owner: last j with pre[j] <= p
  while (hi - lo > 1) {
    const int m = (lo + hi) >> 1;
    if (sg.pre[m] <= p) lo = m; else hi = m;
  }
  int j = lo;
  for (int g = g0; g < g1; g += 2, p += 64) {
    const bool act0 = p < P;
    const bool act1 = (g + 1 < g1) && (p + 32 < P);
    uint32_t c0 = 0u, c1 = 0u;
    double v0 = 0.0, v1 = 0.0;
    if (act0) {
      while (j + 1 < na && sg.pre[j + 1] <= p) ++j;
      const int64_t q = sg.sabs[j] + (p - sg.pre[j]);
      c0 = (uint32_t)__ldg(B.col + q);
      v0 = sg.a[j] * __ldg(B.val + q);  // value <- a_ik * b_kj (Fig:code_spgemm l.5)
    }
    if (act1) {
      while (j + 1 < na && sg.pre[j + 1] <= p + 32) ++j;
      const int64_t q = sg.sabs[j] + (p + 32 - sg.pre[j]);
      c1 = (uint32_t)__ldg(B.col + q);
      v1 = sg.a[j] * __ldg(B.val + q);
    }
    f(act0, c0, v0);
    f(act1, c1, v1);
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
    unsigned long long *row_counter) {
  extern __shared__ double s_dyn_f64[];
  __shared__ int s_cnt;
  __shared__ int s_warp[33];
  __shared__ long long s_row;
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5;
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
    for (int j = threadIdx.x; j < na; j += THREADS) {
      sg.sb[j] = 0;
      const int k = __ldg(A.col + as + j);
      sg.sabs[j] = __ldg(B.rp + k);  // B row start (the segment offset is added per part)
      sg.a[j] = __ldg(A.val + as + j);
    }
    __syncthreads();
    const int per = (na + THREADS - 1) / THREADS;  // entries per thread for the scan
    for (int p = 0; p < np; ++p) {
      const int2 Pp = pr[p];
      const int64_t hi = p + 1 < np ? int64_t(pr[p + 1].x) : B.ncols;
      const int cnt = (p + 1 < np ? pr[p + 1].y : nnz) - Pp.y;
      const int logT = num_log2(cnt);
      const int T = 1 << logT;
      for (int s = threadIdx.x; s < T; s += THREADS) { keys[s] = kEmpty; vals[s] = 0.0; }
      // segment ends and lengths (thread owns entries [t*per, t*per + per))
      int mine = 0;
      for (int j = threadIdx.x * per; j < na && j < (threadIdx.x + 1) * per; ++j) {
        const int k = __ldg(A.col + as + j);
        const int len = (int)(__ldg(B.rp + k + 1) - __ldg(B.rp + k));
        const int64_t bs0 = __ldg(B.rp + k);
        const int e = p + 1 == np ? len : gallop_lb(B.col + bs0, sg.sb[j], len, hi);
        sg.se[j] = e;
        sg.sabs[j] = bs0 + sg.sb[j];  // absolute segment start for this part
        mine += e - sg.sb[j];
      }
      int P;
      int ex = block_excl_scan_int(mine, s_warp, &P);  // (contains the barriers)
      for (int j = threadIdx.x * per; j < na && j < (threadIdx.x + 1) * per; ++j) {
        sg.pre[j] = ex;
        ex += sg.se[j] - sg.sb[j];
      }
      if (threadIdx.x == 0) {
        sg.pre[na] = P;
        s_cnt = 0;
      }
      __syncthreads();
      const int R = (P + 31) >> 5;
      // accumulate; newly inserted keys are appended to the insertion list
      for_part_rounds(B, sg, na, P, (int)((int64_t)R * w / NW), (int)((int64_t)R * (w + 1) / NW),
                      [&](bool act, uint32_t c, double v) {
                        bool isnew = false;
                        uint32_t slot = 0;
                        if (act) {
                          slot = probe_chunk(keys, c, logT, &isnew);
                          atomicAdd(vals + slot, v);  // c_ij <- c_ij + value (l.8)
                        }
                        const unsigned m = __ballot_sync(kFull, isnew);
                        if (m) {
                          const int leader = __ffs(m) - 1;
                          int base = 0;
                          if (lane == leader) base = atomicAdd(&s_cnt, __popc(m));
                          base = __shfl_sync(kFull, base, leader);
                          if (isnew) slot_of[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)slot;
                        }
                      });
      for (int j = threadIdx.x; j < na; j += THREADS) sg.sb[j] = sg.se[j];
      __syncthreads();
      const int64_t width = (hi - Pp.x) < kPartWidth ? (hi - Pp.x) : kPartWidth;
      block_list_emit(keys, vals, slot_of, cnt, Pp.x, width, bm, wpre, gpre, &s_cnt, rp0 + Pp.y,
                      c_col, c_val, sorted);
      __syncthreads();
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
    (size_t(kWPartT) * 16 + size_t(kWPartMaxEntries) * kSegBytes + 8 + 15) & ~size_t(15);

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
    for (int j = lane; j < na; j += 32) {
      sg.sb[j] = 0;
      sg.a[j] = __ldg(A.val + as + j);
    }
    __syncwarp();
    for (int p = 0; p < np; ++p) {
      const int2 Pp = pr[p];
      const int64_t hi = p + 1 < np ? int64_t(pr[p + 1].x) : B.ncols;
      const int cntp = (p + 1 < np ? pr[p + 1].y : nnz) - Pp.y;
      const int logT = num_log2(cntp);
      const int T = 1 << logT;
      for (int s = lane; s < T; s += 32) { keys[s] = kEmpty; vals[s] = 0.0; }
      int carry = 0;
      for (int j0 = 0; j0 < na; j0 += 32) {  // segment ends, exclusive prefix of lengths
        const int j = j0 + lane;
        int L = 0;
        if (j < na) {
          const int k = __ldg(A.col + as + j);
          const int64_t bs0 = __ldg(B.rp + k);
          const int len = (int)(__ldg(B.rp + k + 1) - bs0);
          const int e = p + 1 == np ? len : gallop_lb(B.col + bs0, sg.sb[j], len, hi);
          sg.se[j] = e;
          sg.sabs[j] = bs0 + sg.sb[j];
          L = e - sg.sb[j];
        }
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
      for (int j = lane; j < na; j += 32) sg.sb[j] = sg.se[j];
      __syncwarp();
    }
  }
}

}  // namespace spg
