// relabel.cuh -- degree-ascending relabelling for triangle counting
// (Sec 5.6: "we reorder rows with
// increasing number of nonzeros.  The algorithm then splits the reordered
// matrix A as A = L + U").  Untimed preprocessing in the paper ("After
// preprocessing the input matrix, we compute SpGEMM between L and U").
//
// Given the pattern of a symmetric adjacency matrix G without diagonal:
//   new id of vertex v = rank of the key (deg(v), v) in ascending order
//   (ties by vertex id, so the order is unique);
//   G' = P G P^T, L' = strict lower triangle of G', U' = strict upper.
// Rows of L', U', G' are emitted with ascending columns.
//
// All sorting is done by the kernels below (no library sorts): every key to
// sort is a DISTINCT id in [0, n) inside a segment, so
//   * the vertex order (deg(v), v) = a counting sort by degree (histogram,
//     scan, scatter into degree buckets) followed by a sort of every bucket
//     by id;
//   * the rows of L', U', G' = sorts of their (distinct) new column ids;
// and k_segsort_* sort segments of distinct ids: a warp bitonic network in
// registers (<= 32 keys) or in shared memory (<= 1024 keys), and for longer
// segments a block sets one bit per key in an n-bit shared-memory bitmap and
// emits the set bits in order (a bitmap sort: O(len + n / 32) per segment).
#pragma once
#include "spg_internal.cuh"

namespace spg {

// cnt[deg(v)] += 1 (the degree histogram of the counting sort)
__global__ void k_rl_deghist(DevCSR G, unsigned long long *__restrict__ cnt) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < G.nrows;
       v += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + (G.rp[v + 1] - G.rp[v]), 1ull);
}

// bucket[start[deg(v)] + k] = v, k from the bucket's fill counter (order
// inside a bucket arbitrary: sorted by id next)
__global__ void k_rl_degscatter(DevCSR G, const int64_t *__restrict__ start,
                                unsigned long long *__restrict__ fill, int32_t *__restrict__ bucket) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < G.nrows;
       v += int64_t(gridDim.x) * blockDim.x) {
    const int64_t d = G.rp[v + 1] - G.rp[v];
    bucket[start[d] + (int64_t)atomicAdd(fill + d, 1ull)] = (int32_t)v;
  }
}

// perm[r] = old id of new vertex r (the sorted buckets); rank[v] = new id of v
__global__ void k_rl_rank(const int32_t *__restrict__ sorted_ids, int64_t n,
                          int32_t *__restrict__ perm, int32_t *__restrict__ rank) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t v = sorted_ids[r];
    perm[r] = v;
    rank[v] = (int32_t)r;
  }
}

// ---------------------------------------------------------------------------
// Segmented sort of distinct ids: out[seg[i] .. seg[i+1]) = in[...] ascending.
// Warp per segment: <= 32 keys bitonic in registers, <= kSegWarpMax keys
// bitonic in a warp's shared buffer; longer segments are appended to `longs`
// for k_segsort_long.
// ---------------------------------------------------------------------------
constexpr int kSegWarpMax = 1024;

__device__ __forceinline__ int32_t bitonic32(int32_t x) {
  const int lane = lane_id();
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int32_t o = __shfl_xor_sync(kFull, x, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      x = (lower == up) ? min(x, o) : max(x, o);
    }
  return x;
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_segsort_warp(const int32_t *__restrict__ in,
                                                             int32_t *__restrict__ out,
                                                             const int64_t *__restrict__ seg,
                                                             int64_t nseg, int32_t *__restrict__ longs,
                                                             unsigned long long *nlong) {
  __shared__ int32_t s_buf[WARPS][kSegWarpMax];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t *buf = s_buf[w];
  for (int64_t i = int64_t(blockIdx.x) * WARPS + w; i < nseg; i += int64_t(gridDim.x) * WARPS) {
    const int64_t s = seg[i], len = seg[i + 1] - s;
    if (len <= 1) {
      if (len == 1 && lane == 0) out[s] = in[s];
      continue;
    }
    if (len <= 32) {
      const int32_t x = bitonic32(lane < len ? in[s + lane] : INT32_MAX);
      if (lane < len) out[s + lane] = x;
      continue;
    }
    if (len > kSegWarpMax) {
      if (lane == 0) longs[atomicAdd(nlong, 1ull)] = (int32_t)i;
      continue;
    }
    int P = 64;
    while (P < len) P <<= 1;
    for (int q = lane; q < P; q += 32) buf[q] = q < len ? in[s + q] : INT32_MAX;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int t = lane; t < P / 2; t += 32) {  // pair (a, a + j)
          const int a = ((t / j) * 2 * j) + (t % j);
          const int32_t x = buf[a], y = buf[a + j];
          const bool up = (a & k) == 0;
          if ((x > y) == up) {
            buf[a] = y;
            buf[a + j] = x;
          }
        }
        __syncwarp();
      }
    for (int q = lane; q < len; q += 32) out[s + q] = buf[q];
    __syncwarp();
  }
}

// Block per long segment: bitmap sort over [0, n), in windows of 32 * wwords
// ids (wwords = the shared bitmap's words): per window, set one bit per key
// in the window, then emit the set bits in ascending order after a block
// scan of the per-thread popcounts.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_segsort_long(const int32_t *__restrict__ in,
                                                          int32_t *__restrict__ out,
                                                          const int64_t *__restrict__ seg,
                                                          const int32_t *__restrict__ longs,
                                                          const unsigned long long *nlong,
                                                          int64_t n, int wwords) {
  extern __shared__ uint32_t s_bits[];
  __shared__ int s_w[33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32;
  const long long nl = (long long)*nlong;
  const int64_t W = int64_t(wwords) * 32;
  for (long long li = blockIdx.x; li < nl; li += gridDim.x) {
    const int64_t i = longs[li];
    const int64_t s = seg[i], len = seg[i + 1] - s;
    int64_t done = 0;
    for (int64_t base = 0; base < n; base += W) {
      const int64_t nw64 = (n - base + 31) >> 5;
      const int nwords = (int)(nw64 < wwords ? nw64 : wwords);
      for (int q = threadIdx.x; q < nwords; q += THREADS) s_bits[q] = 0u;
      __syncthreads();
      for (int64_t q = threadIdx.x; q < len; q += THREADS) {
        const int64_t v = in[s + q] - base;
        if (v >= 0 && v < W) atomicOr(s_bits + (v >> 5), 1u << (v & 31));
      }
      __syncthreads();
      // thread t owns words [t * per, (t + 1) * per): popcounts, block scan, emit
      const int per = (nwords + THREADS - 1) / THREADS;
      const int q0 = min(nwords, (int)threadIdx.x * per), q1 = min(nwords, q0 + per);
      int mine = 0;
      for (int q = q0; q < q1; ++q) mine += __popc(s_bits[q]);
      const int incl = warp_incl_scan(mine);
      if (lane == 31) s_w[w] = incl;
      __syncthreads();
      if (w == 0) {
        const int x = lane < NW ? s_w[lane] : 0;
        const int xi = warp_incl_scan(x);
        if (lane < NW) s_w[lane] = xi - x;
        if (lane == NW - 1) s_w[32] = xi;
      }
      __syncthreads();
      int64_t o = s + done + s_w[w] + incl - mine;
      for (int q = q0; q < q1; ++q) {
        uint32_t b = s_bits[q];
        while (b) {
          const int t = __ffs(b) - 1;
          b &= b - 1;
          out[o++] = (int32_t)(base + q * 32 + t);
        }
      }
      done += s_w[32];
      __syncthreads();
    }
  }
}

// Warp per new row r (old vertex u = perm[r]): entries of L' row r = the
// neighbours with a smaller new id, U' row r = those with a larger one.
// Lc/Uc/Gc receive the row lengths (the caller's row_ptr + 1, scanned next);
// a diagonal entry (v == u) is counted in *bad.
__global__ void k_rl_count(DevCSR G, const int32_t *__restrict__ perm,
                           const int32_t *__restrict__ rank, int64_t *__restrict__ Lc,
                           int64_t *__restrict__ Uc, int64_t *__restrict__ Gc,
                           unsigned long long *bad) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < G.nrows; r += nw) {
    const int u = perm[r];
    const int64_t s = G.rp[u], e = G.rp[u + 1];
    int64_t cl = 0;
    int diag = 0;
    for (int64_t q = s + lane; q < e; q += 32) {
      const int v = __ldg(G.col + q);
      cl += __ldg(rank + v) < r;
      diag |= v == u;
    }
    cl = warp_sum(cl);
    diag = __any_sync(kFull, diag);
    if (lane == 0) {
      Lc[r] = cl;
      Uc[r] = (e - s) - cl;
      Gc[r] = e - s;
      if (diag) atomicAdd(bad, 1ull);
    }
  }
}

// Warp per new row r: scatter the new ids of u's neighbours into the L', U'
// and G' rows (order within a row fixed by the segmented sort that follows).
__global__ void k_rl_fill(DevCSR G, const int32_t *__restrict__ perm,
                          const int32_t *__restrict__ rank, const int64_t *__restrict__ Lrp,
                          const int64_t *__restrict__ Urp, const int64_t *__restrict__ Grp,
                          int32_t *__restrict__ Lt, int32_t *__restrict__ Ut,
                          int32_t *__restrict__ Gt) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < G.nrows; r += nw) {
    const int u = perm[r];
    const int64_t s = G.rp[u], e = G.rp[u + 1];
    int64_t lo = Lrp[r], uo = Urp[r];
    const int64_t go = Grp[r];
    for (int64_t q0 = s; q0 < e; q0 += 32) {
      const int64_t q = q0 + lane;
      const bool act = q < e;
      const int rv = act ? __ldg(rank + __ldg(G.col + q)) : 0;
      const bool isl = act && rv < r, isu = act && rv > r;
      const unsigned bl = __ballot_sync(kFull, isl), bu = __ballot_sync(kFull, isu);
      if (isl) Lt[lo + __popc(bl & lt)] = rv;
      if (isu) Ut[uo + __popc(bu & lt)] = rv;
      if (act) Gt[go + (q - s)] = rv;
      lo += __popc(bl);
      uo += __popc(bu);
    }
  }
}

__global__ void k_fill_f64(double *__restrict__ p, int64_t n, double v) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

}  // namespace spg
