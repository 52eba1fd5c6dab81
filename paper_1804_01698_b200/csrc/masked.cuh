// masked.cuh -- fused mask-and-sum (triangle counting,
// PAPER.md Sec 5.6 "L*U ... wedges", BASELINE config 5):
//
//     S = sum over (i, j) in pattern(G) of (A*B)(i, j)
//       = sum over products a_ik * b_kj of Gustavson's row i (Fig:code_spgemm)
//         whose column j is in row i of G,
//
// computed without forming C.  The hash table of the method holds the MASK:
// the columns of G's row i are inserted as keys (key = column, -1
// initialised, multiplicative hash, linear probing) and every product probes
// it; matching products are summed in registers (fp64, exact for the
// integer-valued triangle inputs).  Two tiers:
//   - warp tier (|G_i| <= kMaskWarpKeys): warp-private smem hash set;
//   - block tier (larger G rows): an ncols-bit smem bitmap (ncols <=
//     kBitmapMaxCols) whose bits are set for G_i and cleared again after the
//     row (no full clears), or -- for wider matrices -- a binary search of the
//     sorted G row in global memory.
// Rows are taken from a dynamic queue (row costs are power-law for R-MAT).
#pragma once
#include "spg_internal.cuh"
#include "symbolic.cuh"

namespace spg {

constexpr int kMaskWarpKeys = 256;             // G rows up to this size: warp tier
constexpr int kMaskWarpT = 2 * kMaskWarpKeys;  // warp hash-set slots (load <= 1/2)

// probe-only lookup in a warp-private smem hash set (no insertion)
__device__ __forceinline__ bool set_contains(const uint32_t *tab, uint32_t c, int logT) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
    const uint32_t k = tab[h];
    if (k == c) return true;
    if (k == kEmpty) return false;
    h = (h + 1u) & mask;  // linear probing
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_mask_sum_warp(DevCSR A, DevCSR B, DevCSR G,
                                                              int64_t g_row_begin,
                                                              unsigned long long *row_counter,
                                                              double *sum) {
  __shared__ uint32_t s_tab[WARPS][kMaskWarpT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_tab[w];
  double acc = 0.0;
  while (true) {
    long long r = 0;
    if (lane == 0) r = (long long)atomicAdd(row_counter, 1ull);
    r = __shfl_sync(kFull, r, 0);
    if (r >= A.nrows) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t as = A.rp[r], ae = A.rp[r + 1];
    const int64_t gn = ge - gs;
    if (gn == 0 || gn > kMaskWarpKeys || as == ae) continue;  // (block tier takes the long G rows)
    const int logT = log2_ceil64(uint64_t(2 * gn)) < kMinLogT ? kMinLogT : log2_ceil64(uint64_t(2 * gn));
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
    __syncwarp();
    for (int64_t q = gs + lane; q < ge; q += 32) sym_insert(tab, (uint32_t)__ldg(G.col + q), logT);
    __syncwarp();
    auto f = [&](bool act, uint32_t c, double v) {
      if (act && set_contains(tab, c, logT)) acc += v;  // mask hit: C(i,j) += a_ik b_kj
    };
    int64_t fl = 0;  // flop of the row, for the enumeration choice
    for (int64_t q = as + lane; q < ae; q += 32) {
      const int k = __ldg(A.col + q);
      fl += __ldg(B.rp + k + 1) - __ldg(B.rp + k);
    }
    fl = warp_sum(fl);
    if (use_seq(fl, ae - as)) for_row<true, true, 2>(A, B, as, ae, 0, 1, f);
    else for_row<false, true, 2>(A, B, as, ae, 0, 1, f);
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc != 0.0) atomicAdd(sum, acc);
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_mask_sum_block(DevCSR A, DevCSR B, DevCSR G,
                                                            int64_t g_row_begin,
                                                            unsigned long long *row_counter,
                                                            double *sum, int use_bitmap) {
  extern __shared__ uint32_t s_bm[];
  __shared__ long long s_row;
  __shared__ double s_acc[THREADS / 32];
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwords = (int)((B.ncols + 31) >> 5);
  if (use_bitmap)
    for (int s = threadIdx.x; s < nwords; s += THREADS) s_bm[s] = 0u;
  double acc = 0.0;
  while (true) {
    if (threadIdx.x == 0) s_row = (long long)atomicAdd(row_counter, 1ull);
    __syncthreads();
    const long long r = s_row;
    if (r >= A.nrows) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t as = A.rp[r], ae = A.rp[r + 1];
    if (ge - gs <= kMaskWarpKeys || as == ae) {
      __syncthreads();  // s_row is rewritten next iteration
      continue;
    }
    if (use_bitmap)
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        atomicOr(s_bm + (c >> 5), 1u << (c & 31u));
      }
    __syncthreads();
    auto f = [&](bool act, uint32_t c, double v) {
      if (!act) return;
      bool hit;
      if (use_bitmap) {
        hit = (s_bm[c >> 5] >> (c & 31u)) & 1u;
      } else {  // sorted G row: binary search
        int64_t lo = gs, hi = ge;
        while (lo < hi) {
          const int64_t m = (lo + hi) >> 1;
          if ((uint32_t)__ldg(G.col + m) < c) lo = m + 1; else hi = m;
        }
        hit = lo < ge && (uint32_t)__ldg(G.col + lo) == c;
      }
      if (hit) acc += v;  // mask hit: C(i,j) += a_ik b_kj
    };
    int64_t fl = 0;
    for (int64_t q = as + threadIdx.x; q < ae; q += THREADS) {
      const int k = __ldg(A.col + q);
      fl += __ldg(B.rp + k + 1) - __ldg(B.rp + k);
    }
    fl = warp_sum(fl);
    if (lane == 0) s_acc[w] = (double)fl;
    __syncthreads();
    double flt = 0.0;
    for (int u = 0; u < NW; ++u) flt += s_acc[u];
    if (use_seq((int64_t)flt, ae - as)) for_row<true, true>(A, B, as, ae, w, NW, f);
    else for_row<false, true>(A, B, as, ae, w, NW, f);
    __syncthreads();
    if (use_bitmap)  // clear exactly the bits of G_i for the next row
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        s_bm[c >> 5] = 0u;
      }
    __syncthreads();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc != 0.0) atomicAdd(sum, acc);
}

// ---------------------------------------------------------------------------
// a9 (triangle counting with C formed): sum over stored C(i,j) with
// (i,j) in pattern(G) of C(i,j).  Same mask structures as above: G's row is a
// warp-private hash set (short rows) or an ncols-bit block bitmap (long rows;
// binary search of the sorted G row when ncols > kBitmapMaxCols); the C row
// is read once, coalesced, and every entry probes the set.
// ---------------------------------------------------------------------------
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_csr_mask_sum_warp(DevCSR C, DevCSR G,
                                                                  int64_t g_row_begin,
                                                                  unsigned long long *row_counter,
                                                                  double *sum) {
  __shared__ uint32_t s_tab[WARPS][kMaskWarpT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_tab[w];
  double acc = 0.0;
  while (true) {
    long long r = 0;
    if (lane == 0) r = (long long)atomicAdd(row_counter, 1ull);
    r = __shfl_sync(kFull, r, 0);
    if (r >= C.nrows) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t cs = C.rp[r], ce = C.rp[r + 1];
    const int64_t gn = ge - gs;
    if (gn == 0 || gn > kMaskWarpKeys || cs == ce) continue;  // (block tier: long G rows)
    const int lg = log2_ceil64(uint64_t(2 * gn));
    const int logT = lg < kMinLogT ? kMinLogT : lg;
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
    __syncwarp();
    for (int64_t q = gs + lane; q < ge; q += 32) sym_insert(tab, (uint32_t)__ldg(G.col + q), logT);
    __syncwarp();
    for (int64_t q = cs + lane; q < ce; q += 32)
      if (set_contains(tab, (uint32_t)__ldg(C.col + q), logT)) acc += __ldg(C.val + q);
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc != 0.0) atomicAdd(sum, acc);
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_csr_mask_sum_block(DevCSR C, DevCSR G,
                                                                int64_t g_row_begin,
                                                                unsigned long long *row_counter,
                                                                double *sum, int use_bitmap) {
  extern __shared__ uint32_t s_bm[];
  __shared__ long long s_row;
  const int lane = threadIdx.x & 31;
  const int nwords = (int)((G.ncols + 31) >> 5);
  if (use_bitmap)
    for (int s = threadIdx.x; s < nwords; s += THREADS) s_bm[s] = 0u;
  double acc = 0.0;
  while (true) {
    if (threadIdx.x == 0) s_row = (long long)atomicAdd(row_counter, 1ull);
    __syncthreads();
    const long long r = s_row;
    if (r >= C.nrows) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t cs = C.rp[r], ce = C.rp[r + 1];
    if (ge - gs <= kMaskWarpKeys || cs == ce) {
      __syncthreads();
      continue;
    }
    if (use_bitmap)
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        atomicOr(s_bm + (c >> 5), 1u << (c & 31u));
      }
    __syncthreads();
    for (int64_t q = cs + threadIdx.x; q < ce; q += THREADS) {
      const uint32_t c = (uint32_t)__ldg(C.col + q);
      bool hit;
      if (use_bitmap) {
        hit = (s_bm[c >> 5] >> (c & 31u)) & 1u;
      } else {
        int64_t lo = gs, hi = ge;
        while (lo < hi) {
          const int64_t m = (lo + hi) >> 1;
          if ((uint32_t)__ldg(G.col + m) < c) lo = m + 1; else hi = m;
        }
        hit = lo < ge && (uint32_t)__ldg(G.col + lo) == c;
      }
      if (hit) acc += __ldg(C.val + q);
    }
    __syncthreads();
    if (use_bitmap)
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        s_bm[c >> 5] = 0u;
      }
    __syncthreads();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc != 0.0) atomicAdd(sum, acc);
}

}  // namespace spg
