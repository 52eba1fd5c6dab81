// plan.cuh -- steps a1 (flop), a2 (bins), a4 (scan), a8 (partition), a9 (mask
// sum) and validation.  Included once by spgemm.cu.
#pragma once
#include "spg_internal.cuh"

namespace spg {

// ---------------------------------------------------------------------------
// a1, nonzero-parallel form (balanced whatever the row lengths): every thread
// owns kFlopRun consecutive stored a_ik, finds the row of the first one by a
// binary search of A.rp inside its block's row range, sums nnz(b_k*) along
// its run, and adds each row's partial sum with a segmented warp reduction
// + one atomicAdd per row segment.  flop[] must be zeroed first.
// ---------------------------------------------------------------------------
constexpr int kFlopRun = 8;
constexpr int kFlopThreads = 256;
constexpr int kFlopTile = kFlopRun * kFlopThreads;

__device__ __forceinline__ int64_t row_of(const int64_t *__restrict__ rp, int64_t lo, int64_t hi,
                                          int64_t j) {
  // last r in [lo, hi] with rp[r] <= j
  while (hi - lo > 0) {
    const int64_t mid = lo + (hi - lo + 1) / 2;
    if (__ldg(rp + mid) <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// last r' in [r, hi] with rp[r'] <= j, given rp[r] <= j (galloping: cheap
// when few rows lie between, logarithmic across long runs of empty rows)
__device__ __forceinline__ int64_t advance_row(const int64_t *__restrict__ rp, int64_t r, int64_t hi,
                                               int64_t j) {
  if (r >= hi || __ldg(rp + r + 1) > j) return r;
  int64_t lo = r + 1, step = 1;  // invariant: rp[lo] <= j
  while (lo + step <= hi && __ldg(rp + lo + step) <= j) {
    lo += step;
    step <<= 1;
  }
  int64_t up = lo + step <= hi ? lo + step - 1 : hi;  // answer in [lo, up]
  while (up > lo) {
    const int64_t m = lo + (up - lo + 1) / 2;
    if (__ldg(rp + m) <= j) lo = m; else up = m - 1;
  }
  return lo;
}

// Row of the first a_ik of every tile of kFlopTile consecutive a_ik (one
// thread per tile, all searches in parallel), plus the row of the last a_ik:
// the nonzero-parallel kernels read their tile's row range from it instead
// of searching row_ptr per tile.
__global__ void __launch_bounds__(256) k_tile_rows(DevCSR A, int64_t cap, int64_t *__restrict__ trow) {
  // trow[t] for t < min(ntile, cap) (+ the last row at index ntile if it fits)
  const int64_t base = A.rp[0], nz = A.rp[A.nrows] - base;
  const int64_t ntile = (nz + kFlopTile - 1) / kFlopTile;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t <= ntile && t <= cap;
       t += int64_t(gridDim.x) * blockDim.x) {
    if (nz == 0) break;
    const int64_t j = t < ntile ? base + t * kFlopTile : base + nz - 1;
    trow[t] = row_of(A.rp, 0, A.nrows - 1, j);
  }
}

// Rows of the first and last entries of the tile starting at t0 into
// s_r[0..1]: from the tile-row index (last row of tile t = first row of tile
// t + 1, or the row of the last a_ik), else by binary search.
__device__ __forceinline__ void tile_rows(const DevCSR &A, int64_t base, int64_t t0, int64_t nz,
                                          long long *s_r, const int64_t *__restrict__ trow,
                                          int64_t cap) {
  if (threadIdx.x < 2) {
    const int64_t t = t0 / kFlopTile;
    if (trow && t + 1 <= cap) {
      s_r[threadIdx.x] = threadIdx.x == 0 ? trow[t] : trow[t + 1];
    } else {
      const int64_t tl = (nz - t0) < kFlopTile ? (nz - t0) : kFlopTile;
      const int64_t j = base + t0 + (threadIdx.x == 0 ? 0 : tl - 1);
      s_r[threadIdx.x] = row_of(A.rp, 0, A.nrows - 1, j);
    }
  }
}

__global__ void __launch_bounds__(kFlopThreads) k_flop_nz(DevCSR A, const int64_t *__restrict__ b_rp,
                                                          int64_t b_nrows,
                                                          const uint32_t *__restrict__ b_nonempty,
                                                          unsigned long long *__restrict__ flop,
                                                          PlanInfo *info,
                                                          unsigned long long *__restrict__ useful_row,
                                                          const int64_t *__restrict__ trow, int64_t tcap,
                                                          uint32_t *__restrict__ useful_bits,
                                                          int64_t bits_cap) {
  __shared__ long long s_r[2];
  __shared__ unsigned long long s_maxb, s_useful;
  const int lane = threadIdx.x & 31;
  const int64_t base = A.rp[0], nz = A.rp[A.nrows] - base;
  // mostly-empty B (e.g. a tall-skinny frontier): test the nonempty-row bitmap
  // before gathering B.rp (decided on the device: no host round trip)
  const bool use_bm = b_nonempty != nullptr && 2 * (int64_t)info->b_empty > b_nrows;
  unsigned long long maxb = 0, useful = 0;
  if (threadIdx.x == 0) { s_maxb = 0; s_useful = 0; }
  __syncthreads();
  const int64_t jend = base + nz;
  if (use_bm) {
    // (no block barriers on this path: the warps stream their chunks
    // independently; a useful a_ik -- rare -- finds its row from the tile-row
    // index itself.  Measured on C4: 39% of the stall samples were the two
    // per-tile barriers of the row lookup below)
    for (int64_t t0 = int64_t(blockIdx.x) * kFlopTile; t0 < nz; t0 += int64_t(gridDim.x) * kFlopTile) {
      // mostly-empty B: most a_ik gather nothing, so a warp takes 32
      // consecutive a_ik at a time (coalesced column loads) and finds rows
      // only for the useful ones (one atomic each); the ballot of useful
      // entries is the pruning bitmask: word (tile, chunk), bit = lane
      // (the column loads of all of a warp's chunks are issued before any is
      // used, then the bitmap words: one load in flight per lane kept this
      // pass at 1.2 TB/s on C4's 126 MB of A.col)
      constexpr int kNW = kFlopThreads / 32, kPerWarp = kFlopTile / 32 / kNW;
      const int w = threadIdx.x >> 5;
      int kk[kPerWarp];
      uint32_t bw[kPerWarp];
#pragma unroll
      for (int u = 0; u < kPerWarp; ++u) {
        const int64_t j = base + t0 + int64_t(w + u * kNW) * 32 + lane;
        kk[u] = j < jend ? __ldg(A.col + j) : -1;
      }
#pragma unroll
      for (int u = 0; u < kPerWarp; ++u) bw[u] = kk[u] >= 0 ? __ldg(b_nonempty + (kk[u] >> 5)) : 0u;
#pragma unroll
      for (int u = 0; u < kPerWarp; ++u) {
        const int ch = w + u * kNW;
        const int64_t j = base + t0 + int64_t(ch) * 32 + lane;
        const int k = kk[u];
        unsigned long long len = 0;
        if (k >= 0 && ((bw[u] >> (k & 31)) & 1u))
          len = (unsigned long long)(__ldg(b_rp + k + 1) - __ldg(b_rp + k));
        const unsigned bal = __ballot_sync(kFull, len > 0);
        const int64_t word = (t0 / kFlopTile) * (kFlopTile / 32) + ch;
        if (useful_bits != nullptr && word < bits_cap && lane == 0) useful_bits[word] = bal;
        if (!bal) continue;
        if (len > 0) {
          int64_t rlo = 0, rhi = A.nrows - 1;
          const int64_t t = t0 / kFlopTile;
          if (trow && t + 1 <= tcap) {
            rlo = trow[t];
            rhi = trow[t + 1];
          }
          const int64_t r = row_of(A.rp, rlo, rhi, j);
          atomicAdd(flop + r, len);
          if (useful_row) atomicAdd(useful_row + r, 1ull);
          useful += 1;
          maxb = len > maxb ? len : maxb;
        }
      }
    }
  }
  for (int64_t t0 = int64_t(blockIdx.x) * kFlopTile; t0 < nz && !use_bm;
       t0 += int64_t(gridDim.x) * kFlopTile) {
    __syncthreads();
    tile_rows(A, base, t0, nz, s_r, trow, tcap);
    __syncthreads();
    const int64_t rlo = s_r[0], rhi = s_r[1];
    const int64_t j0 = base + t0 + int64_t(threadIdx.x) * kFlopRun;
    int64_t r = j0 < jend ? row_of(A.rp, rlo, rhi, j0) : rhi;
    int64_t rend = __ldg(A.rp + r + 1);
    unsigned long long acc = 0;
    // walk the run; flush acc at each row boundary (all but the last segment)
    for (int u = 0; u < kFlopRun; ++u) {
      const int64_t j = j0 + u;
      if (j >= jend) break;
      if (j >= rend) {
        if (acc) atomicAdd(flop + r, acc);
        acc = 0;
        r = advance_row(A.rp, r + 1, rhi, j);
        rend = __ldg(A.rp + r + 1);
      }
      const int k = __ldg(A.col + j);
      const unsigned long long len = (unsigned long long)(__ldg(b_rp + k + 1) - __ldg(b_rp + k));
      acc += len;
      useful += len > 0;
      maxb = len > maxb ? len : maxb;
    }

    // last segment: lanes holding the same row combine before the atomic
    const unsigned long long key = (unsigned long long)r;
    const unsigned grp = __match_any_sync(kFull, j0 < jend ? key : ~0ull);
    const int leader = __ffs(grp) - 1;
    // segmented suffix sum inside the group (groups are contiguous lane ranges
    // because rows are nondecreasing across lanes): after the step with offset
    // o, lane i holds the sum over lanes [i, i + 2o) of its group
    unsigned long long sum = acc;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_down_sync(kFull, sum, o);
      if (lane + o < 32 && ((grp >> (lane + o)) & 1u)) sum += v;
    }
    if (lane == leader && j0 < jend && sum) atomicAdd(flop + r, sum);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(kFull, maxb, o);
    maxb = t > maxb ? t : maxb;
  }
  useful = warp_sum(useful);
  if (lane == 0) {
    atomicMax(&s_maxb, maxb);
    if (useful) atomicAdd(&s_useful, useful);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&info->max_brow, s_maxb);
    if (s_useful) atomicAdd(&info->useful, s_useful);
    if (blockIdx.x == 0) info->a_nnz = (unsigned long long)nz;
  }
}

// Nonempty-row bitmap of B (bit k = B row k has entries) and its count of
// empty rows (info->b_empty): one thread per row, words built by warp ballots.
__global__ void __launch_bounds__(256) k_b_rowmask(DevCSR B, uint32_t *__restrict__ bm,
                                                   PlanInfo *info) {
  const int lane = threadIdx.x & 31;
  unsigned long long empty = 0;
  const int64_t nr32 = ((B.nrows + 31) >> 5) << 5;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nr32;
       k += int64_t(gridDim.x) * blockDim.x) {
    const bool valid = k < B.nrows;
    const bool ne = valid && B.rp[k + 1] > B.rp[k];
    const unsigned word = __ballot_sync(kFull, ne);
    if (lane == 0) bm[k >> 5] = word;
    empty += (valid && !ne) ? 1ull : 0ull;
  }
  empty = warp_sum(empty);
  if (lane == 0 && empty) atomicAdd(&info->b_empty, empty);
}

// Pruning of A for a mostly-empty B: a_ik whose B row is empty contribute no
// product, so C = A'*B with A' = A restricted to the useful a_ik.  The row
// counts of A' come from k_flop_nz (useful_row); k_prune_scatter writes, for
// each useful a_ik, its column and its index in A at a per-row cursor (order
// inside a row arbitrary); k_prune_values gathers A' values from the index.
__global__ void __launch_bounds__(kFlopThreads) k_prune_scatter(DevCSR A, const uint32_t *__restrict__ bnz,
                                                                unsigned long long *__restrict__ cursor,
                                                                const int64_t *__restrict__ rp2,
                                                                int32_t *__restrict__ col2,
                                                                int64_t *__restrict__ idx2,
                                                                const int64_t *__restrict__ trow,
                                                                int64_t tcap) {
  __shared__ long long s_r[2];
  const int64_t base = A.rp[0], nz = A.rp[A.nrows] - base;
  for (int64_t t0 = int64_t(blockIdx.x) * kFlopTile; t0 < nz; t0 += int64_t(gridDim.x) * kFlopTile) {
    __syncthreads();
    tile_rows(A, base, t0, nz, s_r, trow, tcap);
    __syncthreads();
    const int64_t j0 = base + t0 + int64_t(threadIdx.x) * kFlopRun;
    const int64_t jend = base + nz;
    if (j0 >= jend) continue;
    int64_t r = row_of(A.rp, s_r[0], s_r[1], j0);
    int64_t rend = __ldg(A.rp + r + 1);
    for (int u = 0; u < kFlopRun; ++u) {
      const int64_t j = j0 + u;
      if (j >= jend) break;
      if (j >= rend) {
        r = advance_row(A.rp, r + 1, s_r[1], j);
        rend = __ldg(A.rp + r + 1);
      }
      const int k = __ldg(A.col + j);
      if (!((__ldg(bnz + (k >> 5)) >> (k & 31)) & 1u)) continue;
      const int64_t pos = rp2[r] + (int64_t)atomicAdd(cursor + r, 1ull);
      col2[pos] = k;
      idx2[pos] = j;
    }
  }
}

// The same scatter from the useful-entry bitmask of k_flop_nz: only the
// useful a_ik are visited (their row by a search over the tile's row range).
__global__ void __launch_bounds__(256) k_prune_scatter_bits(DevCSR A, const uint32_t *__restrict__ bits,
                                                            int64_t nwords,
                                                            unsigned long long *__restrict__ cursor,
                                                            const int64_t *__restrict__ rp2,
                                                            int32_t *__restrict__ col2,
                                                            int64_t *__restrict__ idx2,
                                                            const int64_t *__restrict__ trow,
                                                            int64_t tcap) {
  const int64_t base = A.rp[0];
  constexpr int kWordsPerTile = kFlopTile / 32;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nwords;
       q += int64_t(gridDim.x) * blockDim.x) {
    uint32_t word = bits[q];
    if (!word) continue;
    const int64_t t = q / kWordsPerTile;
    const int ch = (int)(q % kWordsPerTile);
    int64_t rlo = 0, rhi = A.nrows - 1;
    if (trow && t + 1 <= tcap) {
      rlo = trow[t];
      rhi = trow[t + 1];
    }
    while (word) {
      const int lane = __ffs(word) - 1;
      word &= word - 1;
      const int64_t j = base + t * kFlopTile + int64_t(ch) * 32 + lane;
      const int64_t r = row_of(A.rp, rlo, rhi, j);
      const int k = __ldg(A.col + j);
      const int64_t pos = rp2[r] + (int64_t)atomicAdd(cursor + r, 1ull);
      col2[pos] = k;
      idx2[pos] = j;
    }
  }
}

__global__ void __launch_bounds__(256) k_prune_values(const double *__restrict__ aval,
                                                      const int64_t *__restrict__ idx2, int64_t n,
                                                      double *__restrict__ val2) {
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += int64_t(gridDim.x) * blockDim.x)
    val2[p] = __ldg(aval + idx2[p]);
}

// Per-row pass after k_flop_nz: symbolic bin counts, flop total / max, longest a_i.
__global__ void __launch_bounds__(256) k_flop_stats(DevCSR A, int64_t ncols,
                                                    const int64_t *__restrict__ flop,
                                                    PlanInfo *info, int count_bins) {
  __shared__ unsigned s_bins[kMaxBins];
  __shared__ unsigned long long s_sum, s_max, s_maxa;
  if (threadIdx.x < kMaxBins) s_bins[threadIdx.x] = 0;
  if (threadIdx.x == 0) { s_sum = 0; s_max = 0; s_maxa = 0; }
  __syncthreads();
  unsigned long long sum = 0, mx = 0, mxa = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < A.nrows;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t f = flop[i], na = A.rp[i + 1] - A.rp[i];
    sum += (unsigned long long)f;
    mx = (unsigned long long)f > mx ? (unsigned long long)f : mx;
    mxa = (unsigned long long)na > mxa ? (unsigned long long)na : mxa;
    if (count_bins) atomicAdd(&s_bins[count_bins == 2 ? onep_bin(f, ncols, na) : sym_bin(f, ncols, na)], 1u);
  }
  sum = warp_sum(sum);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long t = __shfl_xor_sync(kFull, mx, o);
    mx = t > mx ? t : mx;
    t = __shfl_xor_sync(kFull, mxa, o);
    mxa = t > mxa ? t : mxa;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_sum, sum);
    atomicMax(&s_max, mx);
    atomicMax(&s_maxa, mxa);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_sum) atomicAdd(&info->flop_total, s_sum);
    atomicMax(&info->max_flop, s_max);
    atomicMax(&info->max_arow, s_maxa);
  }
  if (count_bins && threadIdx.x < kMaxBins && s_bins[threadIdx.x])
    atomicAdd(&info->sym_count[threadIdx.x], (unsigned long long)s_bins[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// a2: group row ids by bin (counting sort on the bin id; block-aggregated
// atomics).  mode 0 = symbolic bins from flop[i] (skip rows get row_nnz = 0);
// mode 1 = numeric bins from nnz(c_i) = C_rp[i+1] - C_rp[i].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bin_scatter(int64_t m, const int64_t *__restrict__ key,
                                                     const int64_t *__restrict__ arp,
                                                     int64_t ncols, int mode, PlanInfo *info,
                                                     int32_t *__restrict__ rows_out,
                                                     int64_t *__restrict__ row_nnz,
                                                     const int64_t *__restrict__ flop = nullptr,
                                                     int accum = ACC_HASH, float cfac = 1.0f,
                                                     float hfac = 1.0f) {
  // mode 1: rows the heap tier takes (heap_pick) go to the BACK of their
  // bin's segment, the others to the front
  __shared__ unsigned s_cnt[kMaxBins], s_hcnt[kMaxBins];
  __shared__ unsigned long long s_base[kMaxBins], s_hbase[kMaxBins];
  if (threadIdx.x < kMaxBins) { s_cnt[threadIdx.x] = 0; s_hcnt[threadIdx.x] = 0; }
  __syncthreads();
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  int b = 0;
  bool hp = false;
  unsigned local = 0;
  if (i < m) {
    if (mode == 0 || mode == 2) {  // symbolic bins / one-phase bins (by flop)
      b = mode == 0 ? sym_bin(key[i], ncols, arp[i + 1] - arp[i])
                    : onep_bin(key[i], ncols, arp[i + 1] - arp[i]);
      if (b == SB_SKIP) row_nnz[i] = 0;
    } else {
      const int64_t nz = key[i + 1] - key[i], na = arp[i + 1] - arp[i];
      b = num_bin(nz, na);
      hp = flop != nullptr && heap_pick(b, flop[i], na, nz, accum, cfac, info->b_unsorted == 0, hfac);
    }
    if (b != 0) local = atomicAdd(hp ? &s_hcnt[b] : &s_cnt[b], 1u);
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t > 0 && t < kMaxBins && (s_cnt[t] || s_hcnt[t])) {
    const unsigned long long *cnt = mode != 1 ? info->sym_count : info->num_count;
    unsigned long long off = 0;
    for (int u = 1; u < t; ++u) off += cnt[u];
    if (s_cnt[t])
      s_base[t] = off + atomicAdd(&(mode != 1 ? info->cursor : info->num_cursor)[t],
                                  (unsigned long long)s_cnt[t]);
    if (s_hcnt[t])
      s_hbase[t] = off + cnt[t] - atomicAdd(&info->heap_cursor[t], (unsigned long long)s_hcnt[t]) -
                   s_hcnt[t];
  }
  __syncthreads();
  if (b != 0) rows_out[(hp ? s_hbase[b] : s_base[b]) + local] = (int32_t)i;
}

// ---------------------------------------------------------------------------
// a4: exclusive scan of per-row nnz into C_row_ptr (Fig:hash_spgemm
// "Allocate(cols_C, rpts_C[N_row])", implies the prefix sum).
// In place on data = C_row_ptr + 1 (inclusive scan of row_nnz there gives the
// exclusive row pointer).  Three passes: tile sums, scan of tile sums, tile
// scan + offset.  The last pass also counts numeric bins and max nnz(c_i).
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ long long block_excl_scan_1024(long long v, long long *s_warp,
                                                          long long *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long t = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += t;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0;
    long long yi = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long t = __shfl_up_sync(kFull, yi, o);
      if (lane >= o) yi += t;
    }
    s_warp[lane] = yi - y;  // exclusive warp offsets
    if (lane == 31) s_warp[32] = yi;
  }
  __syncthreads();
  long long r = s_warp[w] + x - v;
  *total = s_warp[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const int64_t *__restrict__ data,
                                                              int64_t n,
                                                              int64_t *__restrict__ partial) {
  __shared__ long long s_warp[33];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  long long s = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    const int64_t idx = base + int64_t(t) * kScanThreads + threadIdx.x;
    if (idx < n) s += data[idx];
  }
  long long tot;
  block_excl_scan_1024(s, s_warp, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(int64_t *__restrict__ partial,
                                                                int64_t nb) {
  __shared__ long long s_warp[33];
  long long carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    const int64_t idx = base + threadIdx.x;
    long long v = idx < nb ? partial[idx] : 0;
    long long tot;
    long long ex = block_excl_scan_1024(v, s_warp, &tot);
    if (idx < nb) partial[idx] = carry + ex;
    carry += tot;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(int64_t *__restrict__ data, int64_t n,
                                                            const int64_t *__restrict__ partial,
                                                            PlanInfo *info,
                                                            const int64_t *__restrict__ arp,
                                                            const int64_t *__restrict__ flop = nullptr,
                                                            int accum = ACC_HASH,
                                                            float cfac = 1.0f, float hfac = 1.0f) {
  __shared__ long long s_warp[33];
  __shared__ unsigned s_bins[kMaxBins], s_hbins[kMaxBins];
  __shared__ unsigned long long s_max;
  if (threadIdx.x < kMaxBins) { s_bins[threadIdx.x] = 0; s_hbins[threadIdx.x] = 0; }
  if (threadIdx.x == 0) s_max = 0;
  const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
  long long v[kScanItems];
  long long s = 0;
  unsigned long long mx = 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    const int64_t idx = base + t;
    v[t] = idx < n ? data[idx] : 0;
    s += v[t];
    mx = (unsigned long long)v[t] > mx ? (unsigned long long)v[t] : mx;
  }
  __syncthreads();
  const bool b_sorted = info->b_unsorted == 0;
#pragma unroll
  for (int t = 0; t < kScanItems; ++t)
    if (arp && base + t < n && v[t] > 0) {
      const int64_t na = arp[base + t + 1] - arp[base + t];
      const int b = num_bin(v[t], na);
      atomicAdd(&s_bins[b], 1u);
      if (flop && heap_pick(b, flop[base + t], na, v[t], accum, cfac, b_sorted, hfac))
        atomicAdd(&s_hbins[b], 1u);
    }
  long long tot;
  long long ex = block_excl_scan_1024(s, s_warp, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int t = 0; t < kScanItems; ++t) {
    const int64_t idx = base + t;
    ex += v[t];
    if (idx < n) data[idx] = ex;
    if (idx == n - 1) info->nnz_total = (unsigned long long)ex;
  }
  atomicMax(&s_max, mx);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&info->max_nnz, s_max);
  if (threadIdx.x > 0 && threadIdx.x < kMaxBins && s_bins[threadIdx.x])
    atomicAdd(&info->num_count[threadIdx.x], (unsigned long long)s_bins[threadIdx.x]);
  if (threadIdx.x > 0 && threadIdx.x < kMaxBins && s_hbins[threadIdx.x])
    atomicAdd(&info->heap_count[threadIdx.x], (unsigned long long)s_hbins[threadIdx.x]);
}

// ---------------------------------------------------------------------------
// Are all rows of B strictly increasing?  (Enables the column-range parts of
// the numeric G tier, which binary-search B rows.)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_check_sorted(DevCSR B, PlanInfo *info) {
  // info->b_unsorted += (descents col[q-1] >= col[q] over all q) - (descents
  // at the first entry of a nonempty row): nonzero iff some row is not
  // strictly increasing.  Two coalesced grid-stride passes (entries, rows)
  // instead of a warp per row.
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  const int64_t q0 = B.rp[0], q1 = B.rp[B.nrows];
  long long d = 0;
  for (int64_t q = q0 + 1 + tid; q < q1; q += nth) d += __ldg(B.col + q - 1) >= __ldg(B.col + q);
  for (int64_t r = tid; r < B.nrows; r += nth) {
    const int64_t s = B.rp[r];
    if (s > q0 && s < B.rp[r + 1]) d -= __ldg(B.col + s - 1) >= __ldg(B.col + s);
  }
  d = warp_sum(d);
  if ((threadIdx.x & 31) == 0 && d != 0) atomicAdd(&info->b_unsorted, (unsigned long long)d);
}

// ---------------------------------------------------------------------------
// Column-tile offsets of B (long-row tier; needs strictly increasing rows;
// positions fit int32, checked by the host).
// ---------------------------------------------------------------------------
// toff[t * nB + k] = first position of B row k (sorted) with column >= t *
// kTileCols, t in [0, ntiles] (TILE-MAJOR: the parts of one tile read one
// contiguous column of the table).  A block takes 32 consecutive B rows: a
// warp per row, lane l lower-bounds tiles l, l + 32, ... in the row (no
// serial walk over the tiles an entry skips) into smem, then the block
// writes each tile's 32 offsets as one coalesced 128-byte store.
constexpr int kToffRows = 32;
__global__ void __launch_bounds__(256) k_tile_offsets(DevCSR B, int ntiles, int32_t *__restrict__ toff) {
  extern __shared__ int32_t s_toff[];  // [(ntiles + 1) * 33]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nB = B.nrows;
  for (int64_t k0 = int64_t(blockIdx.x) * kToffRows; k0 < nB; k0 += int64_t(gridDim.x) * kToffRows) {
    for (int kk = w; kk < kToffRows; kk += 8) {
      const int64_t k = k0 + kk;
      if (k >= nB) break;
      const int64_t s = B.rp[k], e = B.rp[k + 1];
      for (int t = lane; t <= ntiles; t += 32) {
        const int64_t key = int64_t(t) << kTileLog;
        int64_t lo = s, hi = e;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if ((int64_t)__ldg(B.col + mid) < key) lo = mid + 1; else hi = mid;
        }
        s_toff[t * 33 + kk] = (int32_t)lo;
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < (ntiles + 1) * kToffRows; idx += blockDim.x) {
      const int t = idx / kToffRows, kk = idx % kToffRows;
      if (k0 + kk < nB) toff[int64_t(t) * nB + k0 + kk] = s_toff[t * 33 + kk];
    }
    __syncthreads();
  }
}

// Parts (three int4 records each) in processing order: bucket = t0 for single-tile (dense-window)
// parts, kMaxTiles + t0 for multi-tile (hash) parts; dense parts first, tile
// ascending (see k_num_tpart).  Counting sort: per-block smem histograms
// merged into hist[2 * kMaxTiles], one block scans it, then a scatter with a
// per-block reservation in every bucket.
constexpr int kPartBuckets = 2 * kMaxTiles;
__device__ __forceinline__ int part_bucket(int4 p) {
  const int t0 = p.y & 0xFFFF, t1 = p.y >> 16;
  return (t1 == t0 + 1 ? 0 : kMaxTiles) + t0;
}

__global__ void __launch_bounds__(256) k_parts_hist(const int4 *__restrict__ parts,
                                                    const PlanInfo *__restrict__ info,
                                                    unsigned *__restrict__ hist) {
  __shared__ unsigned h[kPartBuckets];
  for (int b = threadIdx.x; b < kPartBuckets; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const int64_t n = (int64_t)info->parts_pool;  // (slots handed out; holes have row -1)
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    const int4 v = parts[3 * p];
    if (v.x >= 0) atomicAdd(&h[part_bucket(v)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kPartBuckets; b += blockDim.x)
    if (h[b]) atomicAdd(&hist[b], h[b]);
}

__global__ void __launch_bounds__(kPartBuckets) k_parts_scan(unsigned *__restrict__ hist) {
  __shared__ int s_w[33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int v = (int)hist[threadIdx.x];
  const int inc = warp_incl_scan(v);
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int x = lane < kPartBuckets / 32 ? s_w[lane] : 0;
    const int xi = warp_incl_scan(x);
    if (lane < kPartBuckets / 32) s_w[lane] = xi - x;
  }
  __syncthreads();
  hist[threadIdx.x] = (unsigned)(s_w[w] + inc - v);  // exclusive: the bucket's first slot (cursor)
}

__global__ void __launch_bounds__(256) k_parts_scatter(const int4 *__restrict__ parts,
                                                       const PlanInfo *__restrict__ info,
                                                       unsigned *__restrict__ cursor,
                                                       int4 *__restrict__ out) {
  __shared__ unsigned h[kPartBuckets];
  for (int b = threadIdx.x; b < kPartBuckets; b += blockDim.x) h[b] = 0u;
  __syncthreads();
  const int64_t n = (int64_t)info->parts_pool;  // (slots handed out; holes have row -1)
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const int4 v = parts[3 * p];
    if (v.x >= 0) atomicAdd(&h[part_bucket(v)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kPartBuckets; b += blockDim.x)
    if (h[b]) h[b] = atomicAdd(&cursor[b], h[b]);  // this block's first slot in bucket b
  __syncthreads();
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n; p += stride) {
    const int4 v = parts[3 * p];
    if (v.x < 0) continue;
    const int4 v1 = parts[3 * p + 1], v2 = parts[3 * p + 2];
    const unsigned d = atomicAdd(&h[part_bucket(v)], 1u);
    out[3 * (int64_t)d] = v;
    out[3 * (int64_t)d + 1] = v1;
    out[3 * (int64_t)d + 2] = v2;
  }
}

// Bytes weight of every row for the bytes-balanced split:
// w_i = 16 + 12 (nnz(a_i) + flop_i + nnz(c_i)) -- the row's share of the
// minimal-bytes model (A row, gathered B rows, C row).
__global__ void __launch_bounds__(256) k_row_bytes(const int64_t *__restrict__ arp,
                                                   const int64_t *__restrict__ flop,
                                                   const int64_t *__restrict__ cnnz, int64_t m,
                                                   int64_t *__restrict__ w) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    w[i] = 16 + 12 * ((arp[i + 1] - arp[i]) + flop[i] + cnnz[i]);
}

// ---------------------------------------------------------------------------
// a8: lowbnd of floor(total*t/nparts) in the flop prefix (length m+1).
// ---------------------------------------------------------------------------
__global__ void k_lowbnd(const int64_t *__restrict__ ps, int64_t m, int64_t nparts,
                         int64_t *__restrict__ offsets) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > nparts) return;
  if (t == 0) { offsets[0] = 0; return; }
  if (t == nparts) { offsets[nparts] = m; return; }
  const int64_t total = ps[m];
  const int64_t q = total / nparts, r = total % nparts;
  const int64_t target = q * t + (r * t) / nparts;  // floor(total * t / nparts)
  int64_t lo = 0, hi = m + 1;                        // first id with ps[id] >= target
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (ps[mid] < target) lo = mid + 1; else hi = mid;
  }
  offsets[t] = lo;
}

// ---------------------------------------------------------------------------
// Validation (untimed): flags bit0 = row_ptr decreasing, bit1 = column out of
// range, bit2 = row not strictly increasing (only when check_sorted).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_validate(DevCSR M, int check_sorted,
                                                  unsigned long long *flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long f = 0;
  for (int64_t i = warp; i < M.nrows; i += nwarps) {
    const int64_t s = M.rp[i], e = M.rp[i + 1];
    if (e < s) { f |= 1; continue; }
    for (int64_t q = s + lane; q < e; q += 32) {
      const int c = M.col[q];
      if (c < 0 || (int64_t)c >= M.ncols) f |= 2;
      if (check_sorted && q > s && M.col[q - 1] >= c) f |= 4;
    }
  }
  if (f) atomicOr(flags, f);
}

}  // namespace spg
