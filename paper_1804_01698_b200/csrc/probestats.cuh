// probestats.cuh -- collision factor c of Eq:hash_est (PAPER.md P:362-365:
// "c is the average number of probes") measured on the GPU, for SURVEY.md
// §8(f) row 2 (HashVector analogue vs linear probing).  Measurement only: not
// on the hot path, no output matrix.
//
// For every row whose numeric table fits a warp (T = lowest 2^n >= 2 nnz(c_i)
// <= kProbeTMax, reading R6), the row's products are inserted (keys only, in
// the numeric phase's round order) into a warp-private table three times:
//   mode 0: linear probing, slot = HIGH bits of col * H (reading R5, the build)
//   mode 1: linear probing, slot = LOW bits of col * H (the literal remainder)
//   mode 2: 4-slot chunks (HashVector-style), chunk = high bits;
//           a probe = one chunk read
//   mode 3: 32-slot warp buckets (warp_bucket_insert, symbolic.cuh): the
//           warp probes one key at a time, a probe = one bucket read (one
//           slot per lane + ballots)
// and the probes of every insert are counted.  out[3 m] = probes, out[3 m + 1]
// = products, out[3 m + 2] = new keys (must equal nnz(C) of the rows).
#pragma once
#include <type_traits>

#include "spg_internal.cuh"
#include "symbolic.cuh"

namespace spg {

constexpr int kProbeTMax = 1024;

template <int MODE>
__device__ __forceinline__ int probe_count_insert(uint32_t *tab, uint32_t c, int logT, bool *isnew) {
  const uint32_t mask = (1u << logT) - 1u;
  int probes = 0;
  if (MODE == 2) {
    const uint32_t cmask = (1u << (logT - kChunkLog)) - 1u;
    uint32_t ch = (c * kHashMul) >> (32 - (logT - kChunkLog));
    while (true) {
      ++probes;
      const uint32_t b = ch << kChunkLog;
      const uint4 k = lds_volatile_v4(tab + b);
      if (k.x == c || k.y == c || k.z == c || k.w == c) return probes;
      const int e = k.x == kEmpty ? 0 : k.y == kEmpty ? 1 : k.z == kEmpty ? 2 : k.w == kEmpty ? 3 : 4;
      if (e < 4) {
        const uint32_t old = atomicCAS(tab + b + e, kEmpty, c);
        if (old == kEmpty) { *isnew = true; return probes; }
        if (old == c) return probes;
        continue;  // lost the slot: re-read the chunk (counted as a probe)
      }
      ch = (ch + 1u) & cmask;
    }
  }
  uint32_t h = MODE == 0 ? hash_slot(c, logT) : ((c * kHashMul) & mask);
  while (true) {
    ++probes;
    const uint32_t k = ((volatile uint32_t *)tab)[h];
    if (k == c) return probes;
    if (k == kEmpty) {
      const uint32_t old = atomicCAS(tab + h, kEmpty, c);
      if (old == kEmpty) { *isnew = true; return probes; }
      if (old == c) return probes;
      continue;  // lost the slot: re-read it (counted)
    }
    h = (h + 1u) & mask;
  }
}

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_probe_stats(DevCSR A, DevCSR B,
                                                            const int64_t *__restrict__ c_rp,
                                                            unsigned long long *out) {
  __shared__ uint32_t s_tab[WARPS][kProbeTMax];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_tab[w];
  unsigned long long acc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = int64_t(blockIdx.x) * WARPS + w; i < A.nrows; i += int64_t(gridDim.x) * WARPS) {
    const int64_t nnz = c_rp[i + 1] - c_rp[i];
    if (nnz == 0 || 2 * nnz > kProbeTMax) continue;
    const int logT = num_log2(nnz);
    const int T = 1 << logT;
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    int64_t fl = 0;
    for (int64_t q = as + lane; q < ae; q += 32) {
      const int k = __ldg(A.col + q);
      fl += __ldg(B.rp + k + 1) - __ldg(B.rp + k);
    }
    fl = warp_sum(fl);
    const bool seq = use_seq(fl, ae - as);
    auto run = [&](auto mode_tag) {
      constexpr int M = decltype(mode_tag)::value;
      for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
      __syncwarp();
      unsigned long long pr = 0, np = 0, nk = 0;
      auto ins = [&](bool act, uint32_t c, double) {
        if (!act) return;
        bool isnew = false;
        pr += (unsigned long long)probe_count_insert<M>(tab, c, logT, &isnew);
        ++np;
        nk += isnew;
      };
      if (seq) for_row<true, false, 2>(A, B, as, ae, 0, 1, ins);
      else for_row<false, false, 2>(A, B, as, ae, 0, 1, ins);
      __syncwarp();
      acc[3 * M] += pr;
      acc[3 * M + 1] += np;
      acc[3 * M + 2] += nk;
    };
    run(std::integral_constant<int, 0>());
    run(std::integral_constant<int, 1>());
    run(std::integral_constant<int, 2>());
    {  // mode 3: warp buckets (every lane ends with the warp's counts)
      for (int s = lane; s < T; s += 32) tab[s] = kEmpty;
      __syncwarp();
      unsigned long long pr = 0, np = 0, nk = 0;
      auto ins = [&](bool act, uint32_t c, double) {
        np += (unsigned long long)__popc(__ballot_sync(kFull, act));
        nk += (unsigned long long)warp_bucket_insert(tab, logT, act, c, &pr);
      };
      if (seq) for_row<true, false, 2>(A, B, as, ae, 0, 1, ins);
      else for_row<false, false, 2>(A, B, as, ae, 0, 1, ins);
      __syncwarp();
      if (lane == 0) {  // (warp-level counts: once per warp)
        acc[9] += pr;
        acc[10] += np;
        acc[11] += nk;
      }
    }
  }
#pragma unroll
  for (int m = 0; m < 12; ++m) {
    const unsigned long long v = warp_sum(acc[m]);
    if (lane == 0 && v) atomicAdd(out + m, v);
  }
}

}  // namespace spg
