// symbolic.cuh -- step a3: nnz(c_i*) per row with open-addressing hash tables
// ("In symbolic phase, it is enough to insert keys to the hash table", P:285;
// key = column, table initialised to -1, (col * const) hashed into a 2^n
// table, linear probing).
//
// Products of a row are enumerated "flattened": a warp takes up to 32 stored
// a_ik of the row, scans the lengths of the B rows they select, and then each
// lane takes one product (a_ik, b_kj) per round, so a round is 32 products
// whatever the B-row lengths (coalesced gathers of consecutive b_kj).
#pragma once
#include "spg_internal.cuh"

namespace spg {

// Insert key c; returns 1 if c was new.  Table in shared or global memory.
__device__ __forceinline__ int sym_insert(uint32_t *tab, uint32_t c, int logT) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
    const uint32_t k = ((volatile uint32_t *)tab)[h];
    if (k == c) return 0;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(tab + h, kEmpty, c);
      if (old == kEmpty) return 1;
      if (old == c) return 0;
    }
    h = (h + 1u) & mask;  // linear probing
  }
}

// Bitmap variant for very long rows: column c -> bit c of an ncols-bit set.
__device__ __forceinline__ int sym_bitmap_insert(uint32_t *bm, uint32_t c) {
  const uint32_t bit = 1u << (c & 31u);
  return (atomicOr(bm + (c >> 5), bit) & bit) ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Product enumeration.  The products of row i are cut into ROUNDS of <= 32
// products; the NW warps of the row's owner (one warp in the W tier, a block
// in the B/G tiers) take rounds round-robin (round g goes to warp g % NW), so
// a row with few a_ik but long B rows still keeps every warp busy.  f(active,
// col, a_ik * b_kj) is called by all 32 lanes of a warp once per round.
//
//  - sequential rounds (kSeq): a round is <= 32 consecutive b_kj of ONE B row,
//    so the keys of a round are distinct (CSR rows hold unique columns);
//  - flattened rounds: 32 consecutive products of the row's product list,
//    whatever the B-row lengths (full lanes for short B rows).
// kVal = false skips the values (symbolic phase).
// ---------------------------------------------------------------------------
template <bool kSeq, bool kVal, typename F>
__device__ __forceinline__ void for_row(const DevCSR &A, const DevCSR &B, int64_t as,
                                        int64_t ae, int w, int NW, F &&f) {
  const int lane = lane_id();
  int64_t gbase = 0;  // rounds of the previous chunks
  for (int64_t cb = as; cb < ae; cb += 32) {
    const int64_t e = cb + lane;
    int len = 0;
    int64_t bs = 0;
    double a = 0.0;
    if (e < ae) {
      const int k = __ldg(A.col + e);
      if (kVal) a = __ldg(A.val + e);
      bs = __ldg(B.rp + k);
      len = (int)(__ldg(B.rp + k + 1) - bs);
    }
    if (kSeq && NW == 1) {
      // one warp owns the row: walk the nonempty entries directly
      unsigned pend = __ballot_sync(kFull, len > 0);
      while (pend) {
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        const int64_t jbs = shfl_i64(bs, j);
        const int L = __shfl_sync(kFull, len, j);
        const double aj = kVal ? shfl_f64(a, j) : 0.0;
        for (int t = 0; t < L; t += 32) {
          const bool act = t + lane < L;
          uint32_t c = 0u;
          double v = 0.0;
          if (act) {
            c = (uint32_t)__ldg(B.col + jbs + t + lane);
            if (kVal) v = aj * __ldg(B.val + jbs + t + lane);  // value <- a_ik*b_kj (l.5)
          }
          f(act, c, v);
        }
      }
      continue;
    }
    const int r = kSeq ? ((len + 31) >> 5) : len;  // rounds (seq) or products per entry
    const int incl = warp_incl_scan(r);
    const int excl = incl - r;
    const int total = __shfl_sync(kFull, incl, 31);
    const int nr = kSeq ? total : ((total + 31) >> 5);
    int g = (int)((w - gbase % NW + NW) % NW);
    for (; g < nr; g += NW) {
      int64_t q;
      double oa = 0.0;
      bool act;
      if (kSeq) {
        const int own = owner_lane(incl, g);
        const int t = (g - __shfl_sync(kFull, excl, own)) * 32 + lane;
        q = shfl_i64(bs, own) + t;
        act = t < __shfl_sync(kFull, len, own);
        if (kVal) oa = shfl_f64(a, own);
      } else {
        const int p = g * 32 + lane;
        const int own = owner_lane(incl, p);
        q = shfl_i64(bs, own) + (p - __shfl_sync(kFull, excl, own));
        act = p < total;
        if (kVal) oa = shfl_f64(a, own);
      }
      uint32_t c = 0u;
      double v = 0.0;
      if (act) {
        c = (uint32_t)__ldg(B.col + q);
        if (kVal) v = oa * __ldg(B.val + q);  // value <- a_ik * b_kj (Fig:code_spgemm l.5)
      }
      f(act, c, v);
    }
    gbase += nr;
  }
}

// Rows whose B rows average >= kSeqMinLen entries use the sequential
// enumeration (no owner search, distinct keys per round); shorter ones the
// flattened one (full 32-lane rounds).
constexpr int kSeqMinLen = 16;
__device__ __forceinline__ bool use_seq(int64_t flop, int64_t nnz_a) {
  return flop >= int64_t(kSeqMinLen) * nnz_a;
}

// ---------------------------------------------------------------------------
// W tier: one warp per row, warp-private table of T <= TMAX slots in smem.
// ---------------------------------------------------------------------------
template <int TMAX, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_sym_warp(const int32_t *__restrict__ rows,
                                                         int64_t nrows, DevCSR A, DevCSR B,
                                                         const int64_t *__restrict__ flop,
                                                         int64_t *__restrict__ row_nnz) {
  extern __shared__ uint32_t s_dyn_u32[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_dyn_u32 + w * TMAX;
  for (int64_t r = int64_t(blockIdx.x) * WARPS + w; r < nrows; r += int64_t(gridDim.x) * WARPS) {
    const int i = rows[r];
    const int logT = sym_log2_gpu(flop[i], B.ncols);
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
    __syncwarp();
    int cnt = 0;
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    auto ins = [&](bool act, uint32_t c, double) {
      if (act) cnt += sym_insert(tab, c, logT);
    };
    if (use_seq(flop[i], ae - as)) for_row<true, false>(A, B, as, ae, 0, 1, ins);
    else for_row<false, false>(A, B, as, ae, 0, 1, ins);
    cnt = warp_sum(cnt);
    if (lane == 0) row_nnz[i] = cnt;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// B tier: one block per row, table of T = 2^logT slots (dynamic smem) shared
// by the block; warps take interleaved chunks of 32 a_ik.
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_sym_block(const int32_t *__restrict__ rows,
                                                       int64_t nrows, DevCSR A, DevCSR B,
                                                       const int64_t *__restrict__ flop,
                                                       int64_t *__restrict__ row_nnz) {
  extern __shared__ uint32_t s_dyn_u32[];
  __shared__ int s_cnt;
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_dyn_u32;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int logT = sym_log2_gpu(flop[i], B.ncols);
    const int T = 1 << logT;
    for (int s = threadIdx.x; s < T; s += THREADS) tab[s] = kEmpty;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int cnt = 0;
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    auto ins = [&](bool act, uint32_t c, double) {
      if (act) cnt += sym_insert(tab, c, logT);
    };
    if (use_seq(flop[i], ae - as)) for_row<true, false>(A, B, as, ae, w, NW, ins);
    else for_row<false, false>(A, B, as, ae, w, NW, ins);
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) row_nnz[i] = s_cnt;
  }
}

// ---------------------------------------------------------------------------
// G tier, bitmap form (ncols small enough for an ncols-bit set in smem): the
// set of distinct columns of c_i* is exactly the set bits.
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_sym_bitmap(const int32_t *__restrict__ rows,
                                                        int64_t nrows, DevCSR A, DevCSR B,
                                                        int64_t *__restrict__ row_nnz) {
  extern __shared__ uint32_t s_dyn_u32[];
  __shared__ int s_cnt;
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwords = (int)((B.ncols + 31) >> 5);
  uint32_t *bm = s_dyn_u32;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    for (int s = threadIdx.x; s < nwords; s += THREADS) bm[s] = 0u;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int cnt = 0;
    for_row<false, false>(A, B, A.rp[i], A.rp[i + 1], w, NW, [&](bool act, uint32_t c, double) {
      if (act) cnt += sym_bitmap_insert(bm, c);
    });
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) row_nnz[i] = s_cnt;
  }
}

// ---------------------------------------------------------------------------
// G tier, global-memory hash (any ncols): one block per row, table in a
// per-block slab of the workspace (global atomics, L2).
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_sym_global(const int32_t *__restrict__ rows,
                                                        int64_t nrows, DevCSR A, DevCSR B,
                                                        const int64_t *__restrict__ flop,
                                                        int64_t *__restrict__ row_nnz,
                                                        uint32_t *__restrict__ slab,
                                                        int64_t slabT) {
  __shared__ int s_cnt;
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = slab + int64_t(blockIdx.x) * slabT;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int logT = sym_log2_gpu(flop[i], B.ncols);
    const int64_t T = int64_t(1) << logT;
    for (int64_t s = threadIdx.x; s < T; s += THREADS) tab[s] = kEmpty;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int cnt = 0;
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto ins = [&](bool act, uint32_t c, double) {
        if (act) cnt += sym_insert(tab, c, logT);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, false>(A, B, as, ae, w, NW, ins);
      else for_row<false, false>(A, B, as, ae, w, NW, ins);
    }
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) row_nnz[i] = s_cnt;
  }
}

}  // namespace spg
