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
constexpr int kMaskWarpT = 4 * kMaskWarpKeys;  // warp hash-set slots (load <= 1/4: most
                                               // probes miss, and a miss walks to an empty slot)

// Final reduction of one warp's fp64 partial (lane 0): into the fp64 sum and,
// exactly, into an int64 sum (triangle counts are reduced in int64, SURVEY
// §8(a) a9).  The int64 sum is exact when every partial is an integer below
// 2^53 in magnitude (then the fp64 partial itself was exact: integer-valued
// inputs); any other partial flags it inexact.
__device__ __forceinline__ void mask_reduce(double acc, PlanInfo *info) {
  if (acc == 0.0) return;
  atomicAdd(&info->mask_acc, acc);
  if (acc == rint(acc) && fabs(acc) < 9007199254740992.0)
    atomicAdd(&info->mask_isum, (unsigned long long)(long long)acc);
  else
    atomicOr(&info->mask_inexact, 1ull);
}

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

// Row lists of the two tiers: rows i with a nonempty row of the product's
// left operand (A, or C when formed) and a nonempty G row, split by |G_i|.
// Only these rows are visited by the sum kernels (most rows of a reordered
// or sparse graph have no work; a per-row queue pop for every row cost more
// than the sums).  Warp-aggregated appends; order within a list arbitrary.
__global__ void k_mask_rows(const int64_t *__restrict__ a_rp, int64_t nrows, DevCSR G,
                            int64_t g_row_begin, int32_t *__restrict__ list_w,
                            int32_t *__restrict__ list_b, unsigned long long *n) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t b = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * 32; b < nrows;
       b += nw * 32) {
    const int64_t r = b + lane;
    bool ok = r < nrows && a_rp[r + 1] > a_rp[r];
    const int64_t gn = ok ? G.rp[g_row_begin + r + 1] - G.rp[g_row_begin + r] : 0;
    const bool isw = ok && gn > 0 && gn <= kMaskWarpKeys, isb = ok && gn > kMaskWarpKeys;
    const unsigned bw = __ballot_sync(kFull, isw), bb = __ballot_sync(kFull, isb);
    unsigned long long ow = 0, ob = 0;
    if (lane == 0) {
      if (bw) ow = atomicAdd(n + 0, (unsigned long long)__popc(bw));
      if (bb) ob = atomicAdd(n + 1, (unsigned long long)__popc(bb));
    }
    ow = __shfl_sync(kFull, ow, 0);
    ob = __shfl_sync(kFull, ob, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (isw) list_w[ow + __popc(bw & lt)] = (int32_t)r;
    if (isb) list_b[ob + __popc(bb & lt)] = (int32_t)r;
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_mask_sum_warp(DevCSR A, DevCSR B, DevCSR G,
                                                              int64_t g_row_begin,
                                                              const int32_t *__restrict__ list,
                                                              const unsigned long long *nlist,
                                                              unsigned long long *row_counter,
                                                              PlanInfo *info) {
  __shared__ uint32_t s_tab[WARPS][kMaskWarpT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_tab[w];
  const long long nl = (long long)*nlist;
  double acc = 0.0;
  while (true) {
    long long q = 0;
    if (lane == 0) q = (long long)atomicAdd(row_counter, 1ull);
    q = __shfl_sync(kFull, q, 0);
    if (q >= nl) break;
    const int64_t r = list[q];  // (warp-tier row: 0 < |G_i| <= kMaskWarpKeys, A row nonempty)
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t as = A.rp[r], ae = A.rp[r + 1];
    const int64_t gn = ge - gs;
    const int logT = log2_ceil64(uint64_t(4 * gn)) < kMinLogT ? kMinLogT : log2_ceil64(uint64_t(4 * gn));
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
  if (lane == 0) mask_reduce(acc, info);
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_mask_sum_block(DevCSR A, DevCSR B, DevCSR G,
                                                            int64_t g_row_begin,
                                                            const int32_t *__restrict__ list,
                                                            const unsigned long long *nlist,
                                                            unsigned long long *row_counter,
                                                            PlanInfo *info, int use_bitmap) {
  extern __shared__ uint32_t s_bm[];
  __shared__ long long s_row;
  __shared__ double s_acc[THREADS / 32];
  __shared__ int s_next;
  __shared__ DeferList s_dl;  // long B rows walked by the whole block
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwords = (int)((B.ncols + 31) >> 5);
  if (use_bitmap)
    for (int s = threadIdx.x; s < nwords; s += THREADS) s_bm[s] = 0u;
  const long long nl = (long long)*nlist;
  double acc = 0.0;
  while (true) {
    // the list is walked from its end: for a degree-ordered graph the
    // heaviest rows have the largest ids and go first
    if (threadIdx.x == 0) {
      const long long q = (long long)atomicAdd(row_counter, 1ull);
      s_row = q < nl ? (long long)list[nl - 1 - q] : -1;
      s_next = 0;
    }
    __syncthreads();
    const long long r = s_row;
    if (r < 0) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t as = A.rp[r], ae = A.rp[r + 1];
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
    if (use_seq((int64_t)flt, ae - as)) for_row<true, true>(A, B, as, ae, w, NW, f, &s_next, &s_dl);
    else for_row<false, true>(A, B, as, ae, w, NW, f, &s_next, &s_dl);
    __syncthreads();
    if (use_bitmap)  // clear exactly the bits of G_i for the next row
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        s_bm[c >> 5] = 0u;
      }
    __syncthreads();
  }
  acc = warp_sum(acc);
  if (lane == 0) mask_reduce(acc, info);
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
                                                                  const int32_t *__restrict__ list,
                                                                  const unsigned long long *nlist,
                                                                  unsigned long long *row_counter,
                                                                  PlanInfo *info) {
  __shared__ uint32_t s_tab[WARPS][kMaskWarpT];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_tab[w];
  const long long nl = (long long)*nlist;
  double acc = 0.0;
  while (true) {
    long long q = 0;
    if (lane == 0) q = (long long)atomicAdd(row_counter, 1ull);
    q = __shfl_sync(kFull, q, 0);
    if (q >= nl) break;
    const int64_t r = list[q];  // (warp-tier row: 0 < |G_i| <= kMaskWarpKeys, C row nonempty)
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t cs = C.rp[r], ce = C.rp[r + 1];
    const int64_t gn = ge - gs;
    const int lg = log2_ceil64(uint64_t(4 * gn));
    const int logT = lg < kMinLogT ? kMinLogT : lg;
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
    __syncwarp();
    for (int64_t q = gs + lane; q < ge; q += 32) sym_insert(tab, (uint32_t)__ldg(G.col + q), logT);
    __syncwarp();
    // C rows are long (C5: ~18 K entries per row): kU coalesced column loads
    // in flight before the probes
    // (the next batch's loads are issued before this batch is probed)
    constexpr int kU = 8;
    uint32_t cc[kU], nc[kU];
    int64_t q0 = cs + lane;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t q = q0 + 32 * u;
      cc[u] = q < ce ? (uint32_t)__ldg(C.col + q) : kEmpty;
    }
    while (q0 < ce) {
      const int64_t q1 = q0 + 32 * kU;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t q = q1 + 32 * u;
        nc[u] = q < ce ? (uint32_t)__ldg(C.col + q) : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (cc[u] != kEmpty && set_contains(tab, cc[u], logT)) acc += __ldg(C.val + q0 + 32 * u);
#pragma unroll
      for (int u = 0; u < kU; ++u) cc[u] = nc[u];
      q0 = q1;
    }
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0) mask_reduce(acc, info);
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_csr_mask_sum_block(DevCSR C, DevCSR G,
                                                                int64_t g_row_begin,
                                                                const int32_t *__restrict__ list,
                                                                const unsigned long long *nlist,
                                                                unsigned long long *row_counter,
                                                                PlanInfo *info, int use_bitmap) {
  extern __shared__ uint32_t s_bm[];
  __shared__ long long s_row;
  const int lane = threadIdx.x & 31;
  const int nwords = (int)((G.ncols + 31) >> 5);
  if (use_bitmap)
    for (int s = threadIdx.x; s < nwords; s += THREADS) s_bm[s] = 0u;
  const long long nl = (long long)*nlist;
  double acc = 0.0;
  while (true) {
    if (threadIdx.x == 0) {
      const long long q = (long long)atomicAdd(row_counter, 1ull);
      s_row = q < nl ? (long long)list[nl - 1 - q] : -1;
    }
    __syncthreads();
    const long long r = s_row;
    if (r < 0) break;
    const int64_t gs = G.rp[g_row_begin + r], ge = G.rp[g_row_begin + r + 1];
    const int64_t cs = C.rp[r], ce = C.rp[r + 1];
    if (use_bitmap)
      for (int64_t q = gs + threadIdx.x; q < ge; q += THREADS) {
        const uint32_t c = (uint32_t)__ldg(G.col + q);
        atomicOr(s_bm + (c >> 5), 1u << (c & 31u));
      }
    __syncthreads();
    constexpr int kU = 4;
    for (int64_t q0 = cs + threadIdx.x; q0 < ce; q0 += THREADS * kU) {
      uint32_t cc[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t q = q0 + int64_t(THREADS) * u;
        cc[u] = q < ce ? (uint32_t)__ldg(C.col + q) : kEmpty;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
      const uint32_t c = cc[u];
      const int64_t q = q0 + int64_t(THREADS) * u;
      if (c == kEmpty) continue;
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
  if (lane == 0) mask_reduce(acc, info);
}

}  // namespace spg
