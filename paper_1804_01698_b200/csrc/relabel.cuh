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
// The vertex order and the per-row column sorts use CUB (library sorts of
// the preprocessing step, like a library GEMM); the counting and scatter are
// the kernels below.
#pragma once
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include "spg_internal.cuh"

namespace spg {

// key[v] = deg(v) << 32 | v  (sorted ascending = the degree order)
__global__ void k_rl_keys(DevCSR G, unsigned long long *__restrict__ key) {
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < G.nrows;
       v += int64_t(gridDim.x) * blockDim.x)
    key[v] = ((unsigned long long)(G.rp[v + 1] - G.rp[v]) << 32) | (unsigned long long)v;
}

// perm[r] = old id of new vertex r; rank[v] = new id of old vertex v
__global__ void k_rl_rank(const unsigned long long *__restrict__ skey, int64_t n,
                          int32_t *__restrict__ perm, int32_t *__restrict__ rank) {
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t v = (int32_t)(skey[r] & 0xFFFFFFFFull);
    perm[r] = v;
    rank[v] = (int32_t)r;
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
