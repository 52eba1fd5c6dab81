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

// CAS-first linear probing of a shared table: one ATOMS.CAS per probe decides
// hit / inserted / occupied.
__device__ __forceinline__ uint32_t num_probe_cas(uint32_t *keys, uint32_t c, int logT) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
    const uint32_t old = atomicCAS(keys + h, kEmpty, c);
    if (old == kEmpty || old == c) return h;
    h = (h + 1u) & mask;
  }
}

// The same for the warp tier's warp-private shared tables.  SPG_NUM_PROBE
// (switch): 0 = num_probe; 1 = the slot's occupant after an attempted
// insert decides (one exit test per step); 2 = CAS-first (no plain load: one
// ATOMS.CAS per probe decides hit / inserted / occupied).  Measured on C2
// (k_num_warp<256>, sorted): 1.156 / 1.105 / 1.025 ms: 2 is the default.
#ifndef SPG_NUM_PROBE
#define SPG_NUM_PROBE 2
#endif
__device__ __forceinline__ uint32_t num_probe_w(uint32_t *keys, uint32_t c, int logT) {
#if SPG_NUM_PROBE == 0
  return num_probe(keys, c, logT);
#else
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
#if SPG_NUM_PROBE == 1
    uint32_t k = ((volatile uint32_t *)keys)[h];
    if (k == kEmpty) {
      k = atomicCAS(keys + h, kEmpty, c);
      k = k == kEmpty ? c : k;
    }
    if (k == c) return h;
#else
    const uint32_t old = atomicCAS(keys + h, kEmpty, c);
    if (old == kEmpty || old == c) return h;
#endif
    h = (h + 1u) & mask;
  }
#endif
}

// Bank spreading of the fp64 accumulators (shared-memory CAS adds serialise
// per bank; measured 26 wavefronts per 32-lane ATOMS.CAST.64 on C3):
//  * dense window: column offset -> slot off ^ (bits 4-7) ^ (bits 8-11) ^
//    (bit 12) in the low 4 bits (a bijection on [0, 8192)); R-MAT columns
//    have each bit set with probability 0.24, so a third of them end in
//    0000 -- one bank pair -- without it;
//  * hash table values: slot s of chunk c = s >> 2, position e = s & 3 lives
//    at e * (T / 4) + c, so the first slots of the chunks (e = 0, the common
//    case) spread over all banks instead of every fourth.
__device__ __forceinline__ uint32_t dense_slot(uint32_t off) {
  return off ^ (((off >> 4) ^ (off >> 8) ^ (off >> 12)) & 15u);
}
__device__ __forceinline__ uint32_t hash_vslot(uint32_t s, int logT) {
  return ((s & 3u) << (logT - 2)) + (s >> 2);
}

// Dense windows start every slot at -0.0: -0.0 + v = v for every v, and a
// slot that received any product can never hold -0.0 again, because every
// product is first mapped through v + (+0.0) (which turns a -0.0 product into
// +0.0 and leaves every other value, NaN included, unchanged; the oracle's
// accumulator starts at +0.0, so the sums are the same).  So a slot is present
// iff its bits differ from -0.0: no occupancy bitmap, no second atomic per
// product.
// C (written once, never re-read by the multiply) goes out with evict-first
// stores so its 116 GB stream (config 3) does not push B's rows out of L2;
// the tile records (read once) come in with evict-first loads.
#ifndef SPG_STCS
#define SPG_STCS 1
#endif
template <typename T>
__device__ __forceinline__ void st_c(T *p, T v) {
#if SPG_STCS
  __stcs(p, v);
#else
  *p = v;
#endif
}
template <typename T>
__device__ __forceinline__ T ld_once(const T *p) {
#if SPG_STCS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}
constexpr unsigned long long kNegZeroBits = 0x8000000000000000ull;
__device__ __forceinline__ double nz_product(double v) { return __dadd_rn(v, 0.0); }
// fp64 add into shared memory at a 32-bit shared address (the LDS + CAS-spin
// loop sm_100a lowers it to; no generic-address arithmetic in the loop)
__device__ __forceinline__ void red_shared_f64(uint32_t saddr, double v) {
  asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(saddr), "d"(v) : "memory");
}

// Two independent fp64 adds into shared memory (SPG_ADD2 builds): both
// current values are loaded and both CAS issued before either result is
// tested, so the two read-modify-write round trips overlap (the lowered
// red.shared.add.f64 is a serial LDS + CAS-spin loop per add).  A failed CAS
// returns the slot's current bits, which seed the retry.
#ifndef SPG_ADD2
#define SPG_ADD2 0
#endif
__device__ __forceinline__ void add2_shared_f64(bool a0, uint32_t s0, double v0, bool a1, uint32_t s1,
                                                double v1) {
#if SPG_ADD2
  unsigned long long x0 = 0, x1 = 0;
  if (a0) asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x0) : "r"(s0) : "memory");
  if (a1) asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x1) : "r"(s1) : "memory");
  unsigned p0 = a0, p1 = a1;
  while (p0 | p1) {
    const unsigned long long n0 = (unsigned long long)__double_as_longlong(
        __dadd_rn(__longlong_as_double((long long)x0), v0));
    const unsigned long long n1 = (unsigned long long)__double_as_longlong(
        __dadd_rn(__longlong_as_double((long long)x1), v1));
    unsigned long long o0 = x0, o1 = x1;  // (an inactive side keeps x: done)
    // both CAS predicated, no branch between them
    asm volatile(
        "{\n\t.reg .pred q0, q1;\n\t"
        "setp.ne.u32 q0, %8, 0;\n\t"
        "setp.ne.u32 q1, %9, 0;\n\t"
        "@q0 atom.shared.cas.b64 %0, [%2], %4, %6;\n\t"
        "@q1 atom.shared.cas.b64 %1, [%3], %5, %7;\n\t}"
        : "+l"(o0), "+l"(o1)
        : "r"(s0), "r"(s1), "l"(x0), "l"(x1), "l"(n0), "l"(n1), "r"(p0), "r"(p1)
        : "memory");
    p0 = p0 && o0 != x0;
    p1 = p1 && o1 != x1;
    x0 = o0;
    x1 = o1;
  }
#else
  if (a0) red_shared_f64(s0, v0);
  if (a1) red_shared_f64(s1, v1);
#endif
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
                                          double *__restrict__ c_val, int sorted, int vlog = 0) {
  // (vlog > 0: the value of slot s is at hash_vslot(s, vlog))
  const int lane = lane_id();
  auto vs = [&](uint32_t s) -> uint32_t { return vlog ? hash_vslot(s, vlog) : s; };
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
        c_val[o] = vals[vs(s0 + lane)];
      }
      base += __popc(bal);
    }
  } else {
    if (nnz <= 128) {
      // <= 128 keys: bitonic sort in registers of packed
      // (column - min) << logT | slot, 4 per lane (element e = 4 lane + r);
      // the values stay in their slots until the store.  Needs a span
      // < 2^(32 - logT).
      unsigned mn = 0xFFFFFFFFu, mx = 0u;
      for (int s0 = 0; s0 < T; s0 += 32) {
        const unsigned k = keys[s0 + lane];
        if (k != kEmpty) {
          mn = k < mn ? k : mn;
          mx = k > mx ? k : mx;
        }
      }
      mn = __reduce_min_sync(kFull, mn);
      mx = __reduce_max_sync(kFull, mx);
      if (mx - mn < (1u << (32 - logT))) {
        uint32_t *pk_s = cnt;  // scratch: packed keys compacted to the front
        int base = 0;
        for (int s0 = 0; s0 < T; s0 += 32) {
          const uint32_t k = keys[s0 + lane];
          const bool occ = k != kEmpty;
          const unsigned bal = __ballot_sync(kFull, occ);
          if (occ) pk_s[base + __popc(bal & lt_mask)] = ((k - mn) << logT) | (uint32_t)(s0 + lane);
          base += __popc(bal);
        }
        for (int e = base + lane; e < 128; e += 32) pk_s[e] = 0xFFFFFFFFu;
        __syncwarp();
        const uint4 kk = reinterpret_cast<const uint4 *>(pk_s)[lane];
        uint32_t pk[4] = {kk.x, kk.y, kk.z, kk.w};
#pragma unroll
        for (int k = 2; k <= 128; k <<= 1) {
#pragma unroll
          for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 4) {  // partner: same r in lane ^ (j / 4)
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                const uint32_t o = __shfl_xor_sync(kFull, pk[r], j >> 2);
                const int e = 4 * lane + r;
                const bool keepmin = ((e & j) == 0) == ((e & k) == 0);
                pk[r] = keepmin ? min(pk[r], o) : max(pk[r], o);
              }
            } else {  // partner: register r ^ j of this lane
#pragma unroll
              for (int r = 0; r < 4; ++r) {
                if (r & j) continue;
                const int e = 4 * lane + r;
                const uint32_t a = pk[r], b = pk[r | j];
                const bool up = (e & k) == 0;
                if ((a > b) == up) { pk[r] = b; pk[r | j] = a; }
              }
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int e = 4 * lane + r;
          if (e < nnz) {
            c_col[rp0 + e] = (int32_t)(mn + (pk[r] >> logT));
            c_val[rp0 + e] = vals[vs(pk[r] & uint32_t(T - 1))];
          }
        }
        return;
      }
    }
    // a7: ascending columns by a bucket (counting) sort.  Buckets
    // are monotone in the column: b(c) = (c - min) >> sh, T buckets for
    // nnz <= T/2 keys; each key's position = bucket offset + its rank
    // among the (few) keys of its bucket.
    // 1. compact occupied slots to the front (destination <= source; with
    //    permuted values (vlog > 0, T <= 256) a lane first holds its slots'
    //    values in registers, so no write lands on an unread value)
    double vreg[8];
    if (vlog) {
#pragma unroll
      for (int j = 0; j < 8; ++j) vreg[j] = 32 * j < T ? vals[vs(32 * j + lane)] : 0.0;
      __syncwarp();
    }
    int base = 0;
    for (int s0 = 0; s0 < T; s0 += 32) {
      const uint32_t k = keys[s0 + lane];
      double v = 0.0;
      if (vlog) {
#pragma unroll
        for (int j = 0; j < 8; ++j) if (32 * j == s0) v = vreg[j];
      } else {
        v = vals[s0 + lane];
      }
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
// One-phase mode (§2, "allocate large
// enough memory space for output matrix and compute"): the numeric kernels
// run on the SYMBOLIC bins (table T = lowest 2^n > min(flop_i, ncols),
// P:302-305, so no symbolic pass is needed), read their bin's row count and
// offset from the device plan (persistent launch, no host round trip), write
// row i at the flop prefix fofs[i] of a flop-sized workspace and record
// nnz(c_i); a copy kernel later compacts the rows into the caller's C.
struct OnePhase {
  const PlanInfo *info;     // sym_count[] (device), flop_total
  const int64_t *fofs;      // exclusive prefix of flop (workspace row offsets)
  int64_t *row_nnz;         // out: nnz(c_i) (C_row_ptr + 1, scanned afterwards)
  unsigned long long cap;   // workspace capacity (products); larger flop: skip
  int bin;                  // symbolic bin this launch handles
};

// this launch's row-list offset (and *nrows); -1 when the workspace overflows
// (the host then grows it and reruns)
__device__ __forceinline__ long long onephase_rows(const OnePhase &op, int64_t *nrows) {
  if (op.info->flop_total > op.cap) return -1;
  long long off = 0;
  for (int u = 1; u < op.bin; ++u) off += (long long)op.info->sym_count[u];
  *nrows = (int64_t)op.info->sym_count[op.bin];
  return off;
}

template <int TMAX, int WARPS, int SORTED, bool ONEP = false>
__global__ void __launch_bounds__(WARPS * 32, (SORTED ? 40 : 48) / WARPS) k_num_warp(const int32_t *__restrict__ rows,
                                                         int64_t nrows, DevCSR A, DevCSR B,
                                                         const int64_t *__restrict__ flop,
                                                         const int64_t *__restrict__ c_rp,
                                                         int32_t *__restrict__ c_col,
                                                         double *__restrict__ c_val,
                                                         OnePhase op = OnePhase{}) {
  constexpr int sorted = SORTED;  // (separate instantiations: the sorted emit costs registers)
  extern __shared__ double s_dyn_f64[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *vals = s_dyn_f64 + w * TMAX;
  uint32_t *keys = reinterpret_cast<uint32_t *>(s_dyn_f64 + WARPS * TMAX) + w * TMAX;
  uint32_t *cnt = reinterpret_cast<uint32_t *>(s_dyn_f64 + WARPS * TMAX) + WARPS * TMAX + w * TMAX;
  if (ONEP) {
    const long long off = onephase_rows(op, &nrows);
    if (off < 0) return;
    rows += off;
  }
  for (int64_t r = int64_t(blockIdx.x) * WARPS + w; r < nrows; r += int64_t(gridDim.x) * WARPS) {
    const int i = rows[r];
    const int64_t rp0 = ONEP ? op.fofs[i] : c_rp[i];
    int nnz = ONEP ? 0 : (int)(c_rp[i + 1] - rp0);
    const int logT = ONEP ? onep_log2(flop[i], B.ncols) : num_log2(nnz);
    const int T = 1 << logT;
    for (int s = lane; s < T; s += 32) { keys[s] = kEmpty; vals[s] = 0.0; }
    __syncwarp();
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    // value slot of key c (chunked probing: the values of chunk position e
    // live at e T/4 + chunk, as in the block tiers, so a round's first-slot
    // values fall in distinct banks)
    // (tables of <= 256 slots: the emit can hold a lane's values in registers)
    const bool chunked = SPG_WARP_CHUNK && T <= 256;
    auto wslot = [&](uint32_t c) -> uint32_t {
      return chunked ? hash_vslot(num_probe_smem(keys, c, logT), logT) : num_probe_w(keys, c, logT);
    };
    if (use_seq(flop[i], ae - as)) {
      // keys of a round are distinct: plain read-modify-write of the value
      for_row<true, true, 2>(A, B, as, ae, 0, 1, [&](bool act, uint32_t c, double v) {
        if (act) vals[wslot(c)] += v;   // c_ij <- c_ij + value (l.8)
        __syncwarp();
      });
    } else {
      for_row<false, true, 2>(A, B, as, ae, 0, 1, [&](bool act, uint32_t c, double v) {
        uint32_t slot = 0;
        if (act) slot = wslot(c);
        const unsigned grp = __match_any_sync(kFull, act ? c : (0x80000000u | lane));
        if (act) {
          if (__popc(grp) == 1) vals[slot] += v;   // c_ij <- c_ij + value (l.8)
          else atomicAdd(vals + slot, v);
        }
        __syncwarp();
      });
    }
    if (ONEP) {  // nnz(c_i) = occupied slots
      for (int s0 = 0; s0 < T; s0 += 32) nnz += __popc(__ballot_sync(kFull, keys[s0 + lane] != kEmpty));
      if (lane == 0) op.row_nnz[i] = nnz;
    }
    warp_emit(keys, vals, cnt, T, logT, nnz, rp0, c_col, c_val, sorted, chunked ? logT : 0);
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Heap tier (§4.2.3 "Heap SpGEMM"):
// one THREAD per row of C.  "To construct c_i*, a heap of size nnz(a_i*) is
// allocated.  For every nonzero a_ik, the first nonzero entry in b_k* along
// with its column index is inserted into the heap.  The algorithm iteratively
// extracts an entry with the minimum column index from the heap, accumulates
// it to c_i*, and inserts the next nonzero entry from the last extracted row
// of B into the heap".  The heap lives in shared memory,
// interleaved by thread (entry e of thread t at [e * T + t]: conflict-free);
// key = column << 32 | entry index, so equal columns leave the heap in the
// stored order of their a_ik and every c_ij is summed in the oracle's
// canonical order with separate multiply and add roundings (bit-exact).
// Output is produced in ascending column order (no sort) straight into C at
// C_row_ptr[i] -- the symbolic phase fixed nnz(c_i).  Needs sorted B rows;
// rows are chosen by heap_pick (cost model Eq:heap_est vs Eq:hash_est).
// ---------------------------------------------------------------------------
struct HeapSegs {
  long long off[2];  // first row-list position of the heap rows of bins W256, W1024
  long long n[2];
};

template <int T>
__global__ void __launch_bounds__(T) k_num_heap(const int32_t *__restrict__ rows, HeapSegs segs,
                                                DevCSR A, DevCSR B,
                                                const int64_t *__restrict__ c_rp,
                                                int32_t *__restrict__ c_col,
                                                double *__restrict__ c_val) {
  extern __shared__ unsigned long long s_heap[];
  unsigned long long *hk = s_heap;                                         // heap keys
  long long *hp = reinterpret_cast<long long *>(s_heap + kHeapMax * T);    // head position
  long long *he = hp + kHeapMax * T;                                       // end of the B row
  double *ha = reinterpret_cast<double *>(he + kHeapMax * T);              // a_ik
  double *hb = ha + kHeapMax * T;                                          // head value b_kj
  const int t = threadIdx.x;
#define SPG_H(arr, e) arr[(e) * T + t]
  const long long total = segs.n[0] + segs.n[1];
  for (long long r = int64_t(blockIdx.x) * T + t; r < total; r += int64_t(gridDim.x) * T) {
    const int i = r < segs.n[0] ? rows[segs.off[0] + r] : rows[segs.off[1] + (r - segs.n[0])];
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    int n = 0;
    for (int64_t q = as; q < ae; ++q) {  // insert the head of every nonempty b_k*
      const int k = __ldg(A.col + q);
      const int64_t bs = __ldg(B.rp + k), be = __ldg(B.rp + k + 1);
      if (bs >= be) continue;
      const int j = n++;
      SPG_H(hp, j) = bs;
      SPG_H(he, j) = be;
      SPG_H(ha, j) = __ldg(A.val + q);
      SPG_H(hb, j) = __ldg(B.val + bs);
      const unsigned long long key = (unsigned long long)(uint32_t)__ldg(B.col + bs) << 32 | (unsigned)j;
      int pos = j;  // sift up
      while (pos > 0) {
        const int par = (pos - 1) >> 1;
        const unsigned long long kp = SPG_H(hk, par);
        if (kp <= key) break;
        SPG_H(hk, pos) = kp;
        pos = par;
      }
      SPG_H(hk, pos) = key;
    }
    int64_t out = c_rp[i];
    long long cur = -1;
    double acc = 0.0;
    while (n > 0) {
      const unsigned long long top = SPG_H(hk, 0);
      const int j = (int)(top & 0xFFFFu);
      const long long c = (long long)(top >> 32);
      const double v = __dmul_rn(SPG_H(ha, j), SPG_H(hb, j));  // a_ik * b_kj (Fig:code_spgemm l.5)
      if (c == cur) {
        acc = __dadd_rn(acc, v);  // accumulate to c_i*
      } else {
        if (cur >= 0) {
          c_col[out] = (int32_t)cur;
          c_val[out] = acc;
          ++out;
        }
        cur = c;
        acc = v;
      }
      // next entry of the extracted B row replaces the top, else the last leaf does
      const long long p = SPG_H(hp, j) + 1;
      unsigned long long key;
      if (p < SPG_H(he, j)) {
        SPG_H(hp, j) = p;
        SPG_H(hb, j) = __ldg(B.val + p);
        key = (unsigned long long)(uint32_t)__ldg(B.col + p) << 32 | (unsigned)j;
      } else {
        --n;
        key = SPG_H(hk, n);
      }
      int pos = 0;  // sift down
      while (true) {
        const int l = 2 * pos + 1;
        if (l >= n) break;
        int m = l;
        unsigned long long km = SPG_H(hk, l);
        if (l + 1 < n) {
          const unsigned long long kr = SPG_H(hk, l + 1);
          if (kr < km) { m = l + 1; km = kr; }
        }
        if (km >= key) break;
        SPG_H(hk, pos) = km;
        pos = m;
      }
      if (n > 0) SPG_H(hk, pos) = key;
    }
    if (cur >= 0) {
      c_col[out] = (int32_t)cur;
      c_val[out] = acc;
    }
  }
#undef SPG_H
}
constexpr int kHeapThreads = 64;
constexpr size_t kHeapSmem = size_t(kHeapMax) * kHeapThreads * 40;

// Block-wide unordered compaction of occupied slots of a table into C row
// (vlog > 0: the values are in the chunk-spread layout hash_vslot(., vlog)).
__device__ __forceinline__ void block_emit_unsorted(const uint32_t *keys, const double *vals,
                                                    int64_t T, int64_t rp0, int32_t *c_col,
                                                    double *c_val, int *s_cnt, int vlog = 0) {
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
      c_val[o] = vals[vlog ? hash_vslot((uint32_t)s, vlog) : (uint32_t)s];
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

// Two exclusive block scans sharing their barriers: returns a's prefix, b's in
// *exb; the totals in *ta / *tb.  s_wa / s_wb hold >= 33 ints each.
__device__ __forceinline__ int block_excl_scan_int2(int a, int b, int *s_wa, int *s_wb, int *ta,
                                                    int *tb, int *exb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int ia = warp_incl_scan(a), ib = warp_incl_scan(b);
  if (lane == 31) {
    s_wa[w] = ia;
    s_wb[w] = ib;
  }
  __syncthreads();
  if (w == 0) {
    const int xa = lane < NW ? s_wa[lane] : 0, xb = lane < NW ? s_wb[lane] : 0;
    const int xia = warp_incl_scan(xa), xib = warp_incl_scan(xb);
    if (lane < NW) {
      s_wa[lane] = xia - xa;
      s_wb[lane] = xib - xb;
    }
    if (lane == 31) {
      s_wa[32] = xia;
      s_wb[32] = xib;
    }
  }
  __syncthreads();
  const int ra = s_wa[w] + ia - a;
  *exb = s_wb[w] + ib - b;
  *ta = s_wa[32];
  *tb = s_wb[32];
  __syncthreads();
  return ra;
}

// a7, block-wide: nnz (key, value) pairs sit compacted in keys /
// vals[0, nnz); store them to C at out in ascending column order by a bucket
// (counting) sort: NB buckets (power of two >= nnz) monotone in the column,
// b(c) = (c - min) >> sh; position = bucket offset + rank among the few keys
// of the bucket.  Scratch: cnt[NB], loc[nnz], grp[nnz] (u32); s_red[66].
__device__ __forceinline__ void block_bucket_sort_to(const uint32_t *keys, const double *vals,
                                                     int nnz, int NB, uint32_t *cnt,
                                                     uint32_t *loc, uint32_t *grp, int64_t out,
                                                     int32_t *__restrict__ c_col,
                                                     double *__restrict__ c_val, int *s_red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
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
  // scatter into bucket order: grp[pos] = key, loc[pos] = its entry (the
  // positions are computed before loc is overwritten: <= kSortPer entries
  // per thread)
  constexpr int kSortPer = 16;
  int pos[kSortPer];
#pragma unroll
  for (int u = 0; u < kSortPer; ++u) {
    const int e = (int)threadIdx.x + u * (int)blockDim.x;
    pos[u] = e < nnz ? (int)cnt[(keys[e] - mn) >> sh] + (int)loc[e] : -1;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSortPer; ++u) {
    const int e = (int)threadIdx.x + u * (int)blockDim.x;
    if (pos[u] >= 0) {
      grp[pos[u]] = keys[e];
      loc[pos[u]] = (uint32_t)e;
    }
  }
  __syncthreads();
  // rank inside the bucket, walking the keys in bucket order (the lanes of a
  // warp sit in the same or neighbouring buckets: no lane waits on a lane of
  // a far larger bucket)
  for (int p = threadIdx.x; p < nnz; p += blockDim.x) {
    const uint32_t k = grp[p];
    const uint32_t b = (k - mn) >> sh;
    const int lo = (int)cnt[b];
    const int hi = (int)b + 1 < NB ? (int)cnt[b + 1] : nnz;
    int rnk = 0;
    for (int q = lo; q < hi; ++q) rnk += grp[q] < k;
    c_col[out + lo + rnk] = (int32_t)k;
    c_val[out + lo + rnk] = vals[loc[p]];
  }
}

// Block-shared table variant: pairs compacted in keys/vals[0, nnz) of a T-slot
// table (nnz <= T/2); scratch in the free upper halves.
__device__ __forceinline__ void block_bucket_sort_store(const uint32_t *keys, const double *vals,
                                                        int T, int nnz, int64_t rp0,
                                                        int32_t *__restrict__ c_col,
                                                        double *__restrict__ c_val, int *s_red) {
  const int NB = T >> 1;
  uint32_t *cnt = const_cast<uint32_t *>(keys) + NB;
  uint32_t *loc = reinterpret_cast<uint32_t *>(const_cast<double *>(vals) + NB);
  block_bucket_sort_to(keys, vals, nnz, NB, cnt, loc, loc + NB, rp0, c_col, c_val, s_red);
}

// ---------------------------------------------------------------------------
// B tier: one block per row, keys/vals of T slots in dynamic smem, shared by
// the block (atomic CAS for keys, atomic fp64 add for values).  Sorted output:
// emit unordered into C, reload the row into smem, bucket-sort it into C (a7).
// ---------------------------------------------------------------------------
template <int THREADS, bool ONEP = false>
__global__ void __launch_bounds__(THREADS, 1024 / THREADS) k_num_block(const int32_t *__restrict__ rows,
                                                       int64_t nrows, DevCSR A, DevCSR B,
                                                       const int64_t *__restrict__ flop,
                                                       const int64_t *__restrict__ c_rp,
                                                       int32_t *__restrict__ c_col,
                                                       double *__restrict__ c_val, int sorted,
                                                       int tmax, OnePhase op = OnePhase{},
                                                       const int64_t *__restrict__ list_off = nullptr,
                                                       const int32_t *__restrict__ lists = nullptr) {
  extern __shared__ double s_dyn_f64[];
  __shared__ int s_cnt, s_next;
  __shared__ DeferList s_dl;  // long B rows walked by the whole block
  __shared__ int s_red[66];
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5;
  double *vals = s_dyn_f64;
  uint32_t *keys = reinterpret_cast<uint32_t *>(s_dyn_f64 + tmax);
  if (ONEP) {
    const long long off = onephase_rows(op, &nrows);
    if (off < 0) return;
    rows += off;
  }
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int64_t rp0 = ONEP ? op.fofs[i] : c_rp[i];
    int nnz = ONEP ? 0 : (int)(c_rp[i + 1] - rp0);
    const int logT = ONEP ? onep_log2(flop[i], B.ncols) : num_log2(nnz);
    const int T = 1 << logT;
    // rows with a sorted column list from the bitmap symbolic: a key -> rank
    // table is built first (every key distinct: inserts do not collide on a
    // key), each product adds into vals2[rank] after a read-only probe, and
    // the emit copies the list and vals2 out (sorted, coalesced; no key CAS
    // per product, no sort).  One walk serves both kinds of rows (a uniform
    // branch in the accumulate: one instantiation of the walk, registers).
    const long long lo_ = (!ONEP && list_off != nullptr) ? list_off[i] : -1;
    const bool lrow = lo_ >= 0;
    const int32_t *L = lists + (lrow ? lo_ : 0);
    uint16_t *rank = reinterpret_cast<uint16_t *>(vals + (T >> 1));  // [T] (list rows)
    for (int s = threadIdx.x; s < T; s += THREADS) keys[s] = kEmpty;
    for (int s = threadIdx.x; s < (lrow ? nnz : T); s += THREADS) vals[s] = 0.0;
    if (threadIdx.x == 0) { s_cnt = 0; s_next = 0; }
    if (lrow) {
      __syncthreads();
      for (int r = threadIdx.x; r < nnz; r += THREADS) {
        bool isnew = false;
        rank[probe_chunk(keys, (uint32_t)__ldg(L + r), logT, &isnew)] = (uint16_t)r;
      }
    }
    __syncthreads();
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto slot_of = [&](uint32_t c) -> double * {
        return lrow ? vals + rank[probe_find(keys, c, logT)]
                    : vals + hash_vslot(SPG_BLOCK_CASFIRST ? num_probe_cas(keys, c, logT)
                                                           : num_probe_smem(keys, c, logT), logT);
      };
      auto acc = [&](bool act, uint32_t c, double v) {  // c_ij <- c_ij + value (l.8)
        if (act) atomicAdd(slot_of(c), v);
      };
      auto acc_comb = [&](bool act, uint32_t c, double v) {  // keys may repeat in a round
        if (warp_combine(act, c, v)) atomicAdd(slot_of(c), v);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, true>(A, B, as, ae, w, NW, acc, &s_next, &s_dl);
      else for_row<false, true>(A, B, as, ae, w, NW, acc_comb, &s_next, &s_dl);
    }
    __syncthreads();
    if (lrow) {
      for (int r = threadIdx.x; r < nnz; r += THREADS) {
        c_col[rp0 + r] = __ldg(L + r);
        c_val[rp0 + r] = vals[r];
      }
      __syncthreads();
      continue;
    }
    block_emit_unsorted(keys, vals, T, rp0, c_col, c_val, &s_cnt, logT);
    if (ONEP) {  // nnz(c_i) = the emitted count
      __syncthreads();
      nnz = s_cnt;
      if (threadIdx.x == 0) op.row_nnz[i] = nnz;
    }
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
  __shared__ int s_cnt, s_next;
  __shared__ DeferList s_dl;  // long B rows walked by the whole block
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
    if (threadIdx.x == 0) { s_cnt = 0; s_next = 0; }
    __syncthreads();
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto acc = [&](bool act, uint32_t c, double v) {
        if (act) atomicAdd(vals + num_probe(keys, c, logT), v);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, true>(A, B, as, ae, w, NW, acc, &s_next, &s_dl);
      else for_row<false, true>(A, B, as, ae, w, NW, acc, &s_next, &s_dl);
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
// G tier, column-tile parts (B rows sorted; parts from the BM symbolic, tile
// offsets from k_tile_offsets).  The blocked SPA the paper cites for long
// rows, on one SM per part: a long row of C is cut into PARTS =
// column ranges [t0, t1) of 8192-column tiles (one tile holding > kTPartKeys
// keys, or a run of tiles holding <= kTPartKeys), and every part is an
// independent work item taken from a global counter.  The part's products
// are, for each a_ik of the row, the segment [toff[t0][k], toff[t1][k]) of B
// row k (two loads from the TILE-MAJOR offset table, no search).
//
// Parts are processed in the order (dense parts, then hash parts; tile t0
// ascending), so the tile-major offsets of one tile column (4 bytes per B
// row) and the B entries of that tile stay L2-resident while its parts run.
//
// Per part, the row's a_ik are staged kTEnt at a time and split by segment
// length:
//   * long segments (>= kTLongSeg products): warp-sequential rounds, a round
//     = 32 consecutive products of ONE segment (distinct columns, full lanes);
//   * short segments: flattened rounds of 32 consecutive products of the
//     compacted short list (owner entry from a window of segment starts).
// Both lists are cut into contiguous round ranges, one per warp.
// Accumulation (Fig:hash_spgemm numeric; Fig:code_spgemm l.8):
//   * single-tile part: dense smem window of kTileCols fp64 + an occupancy
//     bitmap; emitted in column order (sorted by construction) with the slots
//     reset on the way (the window is zeroed once per block);
//   * multi-tile part: chunked smem hash of 4096 slots + an
//     insertion list; emitted in list order, or sorted by a bitmap rank over
//     the part's span / a bucket sort (a7).
// Output position: C_row_ptr[i] + keys of the row before the part.  No global
// atomics besides the part counter.
// ---------------------------------------------------------------------------
#ifndef SPG_TENT
#define SPG_TENT 1024
#endif
#ifndef SPG_TLONGSEG
#define SPG_TLONGSEG 32
#endif
constexpr int kTEnt = SPG_TENT;             // a_ik staged per chunk
constexpr int kTLongSeg = SPG_TLONGSEG;     // segments of >= this many products run warp-sequential
constexpr int kTPartLogT = 12;
constexpr int kTPartT = 1 << kTPartLogT;      // hash slots of a multi-tile part
static_assert(4 * kTPartKeys <= 3 * kTPartT, "multi-tile part: load <= 3/4");
constexpr int64_t kTRankCols = int64_t(32) * kTileCols;  // sorted emit by bitmap rank up to this span
constexpr size_t kTDenseBytes = size_t(kTileCols) * 8;  // (presence: -0.0 slots)
constexpr size_t kTHashBytes = size_t(kTPartT) * 12 + size_t(kTPartKeys) * 2;
constexpr size_t kTRecDenseBytes = size_t(kTileRec) * 4 + size_t(kTileCols) * 8;  // record + values
constexpr size_t kTUnion0 = kTDenseBytes > kTHashBytes ? kTDenseBytes : kTHashBytes;
constexpr size_t kTUnion =
    (SPG_DENSE_RECORDS && kTRecDenseBytes > kTUnion0) ? kTRecDenseBytes : kTUnion0;
// entry stage (byte offsets): short list es i32 / ea f64 / epre i32[+1];
// long list ls i32 / ll i32 (length) / la f64 / lpre i32[+1] (round prefix)
constexpr size_t kOffEa = 0;
constexpr size_t kOffLa = kOffEa + size_t(kTEnt) * 8;
constexpr size_t kOffEs = kOffLa + size_t(kTEnt) * 8;
constexpr size_t kOffLs = kOffEs + size_t(kTEnt) * 4;
constexpr size_t kOffLl = kOffLs + size_t(kTEnt) * 4;
constexpr size_t kOffEpre = kOffLl + size_t(kTEnt) * 4;
constexpr size_t kOffLpre = kOffEpre + size_t(kTEnt + 4) * 4;
constexpr size_t kTEntBytes = kOffLpre + size_t(kTEnt + 4) * 4;
static_assert(size_t(kTPartKeys) * 12 <= kTEntBytes, "sorted gather");
static_assert(size_t(kTRankCols / 32) * 8 <= kTUnion, "rank bitmap + prefix in the table region");
static_assert(size_t(kPbitsMaxSpan) * kTileRec * 4 + size_t(kTPartKeys) * 12 <= kTUnion,
              "tile records + rank-indexed values in the table region");
static_assert(!SPG_DENSE_RECORDS || size_t(kTileRec) * 4 + size_t(kTileCols) * 8 <= kTUnion,
              "one tile record + a dense part's rank-indexed values");
// Next-part prefetch (cp.async, issued while this part runs): the first
// kTPf entries of the next part -- A.col, A.val, then the two tile offsets of
// every such entry -- so a part's first staging chunk waits on no global load.
constexpr int kTPf = 512;
constexpr size_t kOffPfCol = 0, kOffPfVal = size_t(kTPf) * 4, kOffPfS0 = kOffPfVal + size_t(kTPf) * 8,
                 kOffPfE0 = kOffPfS0 + size_t(kTPf) * 4;
constexpr size_t kTPfBytes = kOffPfE0 + size_t(kTPf) * 4;
constexpr size_t kTPartSmem = kTUnion + kTEntBytes + kTPfBytes;
static_assert(kTEnt <= 32 * 32, "32-ary owner search");

// Asynchronous global -> shared copies (cp.async; Ampere+ LDGSTS, no
// registers held while in flight).
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// last j < n with pre[j] <= x (pre[0] = 0 <= x, pre nondecreasing, n <= 1024):
// a 32-ary search, two ballots over strided then consecutive entries
__device__ __forceinline__ int tpart_find(const int32_t *pre, int n, int x) {
  const int lane = lane_id();
  const int c1 = lane * 32;
  const unsigned b1 = __ballot_sync(kFull, c1 < n && pre[c1] <= x);
  const int blk = 31 - __clz(b1);
  const int c2 = blk * 32 + lane;
  const unsigned b2 = __ballot_sync(kFull, c2 < n && pre[c2] <= x);
  return blk * 32 + 31 - __clz(b2);
}

// Rounds [g0, g1) of 32 consecutive products of the staged SHORT entries (all
// nonempty: products [pre[j], pre[j+1]) (pre[n] = P implied) are the
// segment [es[j], ...) of B, multiplier ea[j], pre strictly increasing).  The owner entry of
// product x is tracked per warp: `cur` owns the round's first product; the
// <= 32 entries that start inside the round are found from a window of the
// next 32 entry starts (one smem load per lane), their start positions
// OR-ed into a 32-bit mask, and lane t's owner = cur + (starts at or before
// t).  Owners and gather addresses of kD rounds first, then the kD gathers,
// then the kD updates f(active, column, a_ik * b_kj).
template <int kD = 2, typename F>
__device__ __forceinline__ void for_tpart_rounds(const DevCSR &B, const int32_t *es,
                                                 const double *ea, const int32_t *pre, int n,
                                                 int P, int g0, int g1, F &&f) {
  if (g0 >= g1) return;
  const int lane = lane_id();
  const unsigned le = lane == 31 ? 0xFFFFFFFFu : ((2u << lane) - 1u);  // lanes <= this one
  int cur = tpart_find(pre, n, g0 * 32);
  for (int g = g0; g < g1; g += kD) {
    uint32_t c[kD];
    double v[kD], a[kD];
    bool act[kD];
    int64_t q[kD];
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      const int x0 = (g + d) * 32, x = x0 + lane;
      act[d] = (g + d < g1) && x < P;
      const int e = cur + 1 + lane;
      const int st = e < n ? pre[e] : INT32_MAX;  // start of entry cur + 1 + lane (> x0)
      const unsigned pos = __reduce_or_sync(kFull, st < x0 + 32 ? (1u << (st - x0)) : 0u);
      const int j = cur + __popc(pos & le);
      cur += __popc(__ballot_sync(kFull, st <= x0 + 32));  // owner of the next round's first product
      q[d] = act[d] ? int64_t(es[j]) + (x - pre[j]) : 0;
      a[d] = act[d] ? ea[j] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < kD; ++d) {
      c[d] = act[d] ? (uint32_t)__ldg(B.col + q[d]) : 0u;
      v[d] = act[d] ? __ldg(B.val + q[d]) : 0.0;
    }
    static_assert(kD == 2, "pairs of rounds");
    f(act[0], c[0], a[0] * v[0], act[1], c[1], a[1] * v[1]);  // a_ik * b_kj (Fig:code_spgemm l.5)
  }
}

// Rounds [g0, g1) of the staged LONG entries: entry j covers rounds
// [lpre[j], lpre[j+1]) = ceil(ll[j] / 32) rounds; round r of entry j is the
// products ls[j] + 32 r + lane of ONE B row segment (distinct columns).  A
// rolling software pipeline of kLD register slots: right after the round in
// slot d is applied, the slot is refilled with the round kLD ahead (the load
// cursor walks the entries), so kLD independent gathers stay in flight
// across entry boundaries.  Inactive lanes hold the column kEmpty.
#ifndef SPG_LONG_DEPTH
#define SPG_LONG_DEPTH 0
#endif
constexpr int kLD = SPG_LONG_DEPTH;
template <typename F>
__device__ __forceinline__ void for_long_rounds_entry(const DevCSR &B, const int32_t *ls,
                                                      const int32_t *ll, const double *la,
                                                      const int32_t *lpre, int n, int R,
                                                      int g0, int g1, F &&f) {
  // (SPG_LONG_DEPTH=0: entry by entry, two rounds per step inside an entry)
  const int lane = lane_id();
  int j = tpart_find(lpre, n, g0);
  int g = g0;
  while (g < g1) {
    const int rb = lpre[j];
    const int re = min(g1, j + 1 < n ? lpre[j + 1] : R);
    const int L = ll[j];
    const double a = la[j];
    const int32_t *pc = B.col + ls[j];
    const double *pv = B.val + ls[j];
    int t = (g - rb) * 32 + lane;
    for (; g + 1 < re; g += 2, t += 64) {
      const bool act0 = t < L, act1 = t + 32 < L;
      const uint32_t c0 = act0 ? (uint32_t)__ldg(pc + t) : 0u;
      const double v0 = act0 ? __ldg(pv + t) : 0.0;
      const uint32_t c1 = act1 ? (uint32_t)__ldg(pc + t + 32) : 0u;
      const double v1 = act1 ? __ldg(pv + t + 32) : 0.0;
      f(act0, c0, a * v0, act1, c1, a * v1);
    }
    if (g < re) {
      const bool act0 = t < L;
      const uint32_t c0 = act0 ? (uint32_t)__ldg(pc + t) : 0u;
      const double v0 = act0 ? __ldg(pv + t) : 0.0;
      f(act0, c0, a * v0, false, 0u, 0.0);
      ++g;
    }
    ++j;
  }
}

template <typename F>
__device__ __forceinline__ void for_long_rounds(const DevCSR &B, const int32_t *ls,
                                                const int32_t *ll, const double *la,
                                                const int32_t *lpre, int n, int R, int g0,
                                                int g1, F &&f) {
  if (g0 >= g1) return;
  if constexpr (kLD == 0) {
    for_long_rounds_entry(B, ls, ll, la, lpre, n, R, g0, g1, f);
    return;
  }
  constexpr int D = kLD > 0 ? kLD : 1;
  const int lane = lane_id();
  int j = tpart_find(lpre, n, g0);  // load cursor: entry j, its rounds [rb, re)
  int rb = lpre[j], re = j + 1 < n ? lpre[j + 1] : R, L = ll[j];
  const int32_t *pc = B.col + ls[j];
  const double *pv = B.val + ls[j];
  int gl = g0;  // next round to load
  uint32_t c[D];
  double v[D];
  int jd[D];  // entry of the slot's round (its a_ik is read from smem when applied)
  auto load = [&](int d) {  // round gl into slot d (gl < g1, warp-uniform)
    while (gl >= re) {
      ++j;
      rb = re;
      re = j + 1 < n ? lpre[j + 1] : R;
      L = ll[j];
      pc = B.col + ls[j];
      pv = B.val + ls[j];
    }
    const int t = (gl - rb) * 32 + lane;
    c[d] = kEmpty;
    v[d] = 0.0;
    if (t < L) {
      c[d] = (uint32_t)__ldg(pc + t);
      v[d] = __ldg(pv + t);
    }
    jd[d] = j;
    ++gl;
  };
#pragma unroll
  for (int d = 0; d < D; ++d) {
    c[d] = kEmpty;
    jd[d] = 0;
    if (gl < g1) load(d);
  }
  for (int g = g0; g < g1; g += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (g + d < g1) {
        f(c[d] != kEmpty, c[d], la[jd[d]] * v[d], false, 0u, 0.0);  // a_ik * b_kj (Fig:code_spgemm l.5)
        if (gl < g1) load(d);
      }
    }
  }
}

// Three exclusive block scans sharing their barriers (s_w: >= 3 * 33 ints).
// No trailing barrier: the caller's next barrier protects s_w.
__device__ __forceinline__ void block_excl_scan3(const int (&v)[3], int (&ex)[3], int (&tot)[3],
                                                 int *s_w) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, NW = blockDim.x >> 5;
  int inc[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    inc[k] = warp_incl_scan(v[k]);
    if (lane == 31) s_w[k * 33 + w] = inc[k];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int x = lane < NW ? s_w[k * 33 + lane] : 0;
      const int xi = warp_incl_scan(x);
      if (lane < NW) s_w[k * 33 + lane] = xi - x;
      if (lane == 31) s_w[k * 33 + 32] = xi;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ex[k] = s_w[k * 33 + w] + inc[k] - v[k];
    tot[k] = s_w[k * 33 + 32];
  }
}

#ifndef SPG_TPART_INSTR
#define SPG_TPART_INSTR 0
#endif
constexpr bool kTpartInstr = SPG_TPART_INSTR != 0;  // per-phase clock counters into dbg[]
template <int THREADS>
__global__ void __launch_bounds__(THREADS, 2) k_num_tpart(
    DevCSR A, DevCSR B, const int64_t *__restrict__ c_rp, int32_t *__restrict__ c_col,
    double *__restrict__ c_val, int sorted, const int4 *__restrict__ parts, int64_t nparts,
    const int32_t *__restrict__ toff, int64_t nB, unsigned long long *counter, int tune,
    unsigned long long *dbg, const uint32_t *__restrict__ pbits,
    const uint16_t *__restrict__ dpfx) {
  extern __shared__ double s_dyn_f64[];
  __shared__ int s_warp[33];
  __shared__ int s_red[66];
  __shared__ int s_cnt;
  // staging reservations, double-buffered by chunk parity: [short, long] =
  // (entries << 32) | (products or rounds)
  __shared__ unsigned long long s_res[2][2];
  __shared__ long long s_rp0;
  __shared__ __align__(16) uint16_t s_dp[kDenseStripes];  // dense part: keys before each warp's stripe
  // part pipeline (thread 0): the part after next is reserved and the next
  // part's records are loaded while this part runs; published at its end
  __shared__ long long s_q;
  __shared__ int4 s_P, s_P1, s_P2, s_Pn[3];
  __shared__ int s_pn_ok;  // the next part exists (its records are in s_Pn once thread 0 waited)
  // the dense window was used by a record / hash part (written by thread 0 at
  // the publish step: a shared flag instead of a register kept across parts)
  __shared__ int s_dirty;
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  char *base = reinterpret_cast<char *>(s_dyn_f64);
  double *dv = reinterpret_cast<double *>(base);                          // dense window
  double *hv = reinterpret_cast<double *>(base);                          // hash table
  uint32_t *hk = reinterpret_cast<uint32_t *>(base + size_t(kTPartT) * 8);
  uint16_t *slot_of = reinterpret_cast<uint16_t *>(base + size_t(kTPartT) * 12);
  char *eb = base + kTUnion;                                              // staged entries
  double *ea = reinterpret_cast<double *>(eb + kOffEa);
  double *la = reinterpret_cast<double *>(eb + kOffLa);
  int32_t *es = reinterpret_cast<int32_t *>(eb + kOffEs);
  int32_t *ls = reinterpret_cast<int32_t *>(eb + kOffLs);
  int32_t *ll = reinterpret_cast<int32_t *>(eb + kOffLl);
  int32_t *epre = reinterpret_cast<int32_t *>(eb + kOffEpre);
  int32_t *lpre = reinterpret_cast<int32_t *>(eb + kOffLpre);
  char *pfb = eb + kTEntBytes;  // next-part prefetch
  int32_t *pf_col = reinterpret_cast<int32_t *>(pfb + kOffPfCol);
  double *pf_val = reinterpret_cast<double *>(pfb + kOffPfVal);
  int32_t *pf_s0 = reinterpret_cast<int32_t *>(pfb + kOffPfS0);
  int32_t *pf_e0 = reinterpret_cast<int32_t *>(pfb + kOffPfE0);
  static_assert(kTPf <= THREADS, "one prefetched entry per thread");
  int pf_n = 0;  // entries of the current part prefetched (block-uniform)
  // the dense window starts clean (every slot -0.0: absent); every dense part
  // resets what it used
  unsigned long long *dvb = reinterpret_cast<unsigned long long *>(dv);
  const uint32_t dv_sa = (uint32_t)__cvta_generic_to_shared(dv);
  for (int s = threadIdx.x; s < kTileCols; s += THREADS) dvb[s] = kNegZeroBits;
  long long q_next = 0;  // (thread 0) reserved part after the current one
  if (threadIdx.x == 0) {
    s_dirty = 0;
    s_res[0][0] = s_res[0][1] = s_res[1][0] = s_res[1][1] = 0ull;
    const long long q = (long long)atomicAdd(counter, 1ull);
    s_q = q;
    if (q < nparts) {
      s_P = parts[3 * q];
      s_P1 = parts[3 * q + 1];
      s_P2 = parts[3 * q + 2];
    }
    q_next = (long long)atomicAdd(counter, 1ull);
  }
  __syncthreads();
  const bool instr = kTpartInstr && threadIdx.x == 0;  // (phase clocks: SPG_TPART_INSTR builds)
  int par = 0;  // staging buffer parity (alternates per chunk)
  while (true) {
    const int64_t q = s_q;
    if (q >= nparts) break;
    const int4 P = s_P, P1 = s_P1, P2 = s_P2;
    // thread 0: async copies (cp.async, no registers held) of the next
    // part's records (q_next was reserved one part ago) and of this part's
    // C row start (used at the emit); reserve the part after next
    long long q_after = 0;
    if (threadIdx.x == 0) {
      cp_async8(&s_rp0, c_rp + P.x);
      if (dpfx != nullptr && P2.z >= 0 && (P.y >> 16) == (P.y & 0xFFFF) + 1) {  // dense part's stripe prefixes
        cp_async16(&s_dp[0], dpfx + int64_t(P2.z) * kDenseStripes);
        cp_async16(&s_dp[8], dpfx + int64_t(P2.z) * kDenseStripes + 8);
      }
      s_pn_ok = q_next < nparts;
      if (q_next < nparts) {
        cp_async16(&s_Pn[0], parts + 3 * q_next);
        cp_async16(&s_Pn[1], parts + 3 * q_next + 1);
        cp_async16(&s_Pn[2], parts + 3 * q_next + 2);
      }
      cp_async_commit();
      q_after = q_next < nparts ? (long long)atomicAdd(counter, 1ull) : q_next;
    }
    const int t0 = P.y & 0xFFFF, t1 = P.y >> 16;
    const int cnt = P.w;
    const bool dense = t1 == t0 + 1;
    const int64_t as = (int64_t)(((unsigned long long)(unsigned)P1.y << 32) | (unsigned)P1.x);
    const int na = P1.z;
    const int64_t lo = int64_t(t0) << kTileLog;
    const long long c0 = instr ? clock64() : 0;
    long long c_stage = 0, c_rounds = 0;
    unsigned long long prods = 0;
    const int logT = dense ? 0 : min(num_log2(cnt), kTPartLogT);
    const int T = 1 << logT;
    // a narrow hash part with its tile records from the symbolic phase (the
    // row's bitmap words + per-word ranks): products index the part's
    // columns by rank (two loads and a popcount, no hashing, no key insert),
    // values accumulate in vals[rank], and the emit walks the bitmap (column
    // order: sorted for free)
    const long long koff = (long long)(((unsigned long long)(unsigned)P2.y << 32) | (unsigned)P2.x);
    const bool known = koff >= 0 && pbits != nullptr;
    uint32_t *rec = reinterpret_cast<uint32_t *>(base);                       // span x kTileRec words
    double *rv = reinterpret_cast<double *>(base + size_t(t1 - t0) * kTileRec * 4);  // [cnt]
    int32_t *rcol = reinterpret_cast<int32_t *>(rv + kTPartKeys);  // [cnt]: column of each rank
    if (known) {
      const int nrec = (t1 - t0) * kTileRec;
      const uint4 *src = reinterpret_cast<const uint4 *>(pbits + koff * kTileRec);
      for (int q = threadIdx.x; q < nrec / 4; q += THREADS) reinterpret_cast<uint4 *>(rec)[q] = ld_once(src + q);
      for (int r = threadIdx.x; r < cnt; r += THREADS) rv[r] = 0.0;
    } else if (!dense) {
      for (int s = threadIdx.x; s < T; s += THREADS) { hk[s] = kEmpty; hv[s] = 0.0; }
    } else if (s_dirty) {  // a dense window after a part that used the region otherwise
      for (int s = threadIdx.x; s < kTileCols; s += THREADS) dvb[s] = kNegZeroBits;
    }
    if (threadIdx.x == 0) s_cnt = 0;
    const int32_t *tk0 = toff + int64_t(t0) * nB, *tk1 = toff + int64_t(t1) * nB;
    const uint32_t lo32 = (uint32_t)lo;
    auto acc_dense = [&](bool a0, uint32_t c0, double v0, bool a1, uint32_t c1, double v1) {
      // c_ij <- c_ij + value (l.8), dense window (presence: the slot left -0.0)
      add2_shared_f64(a0, dv_sa + 8u * dense_slot(c0 - lo32), nz_product(v0), a1,
                      dv_sa + 8u * dense_slot(c1 - lo32), nz_product(v1));
    };
    const uint32_t rv_sa = (uint32_t)__cvta_generic_to_shared(rv);
    auto rank_of = [&](uint32_t c) {  // rank of the column in the part
      const uint32_t off = c - (uint32_t)lo, q = off >> 5;
      const uint32_t *tr = rec + (q >> 8) * kTileRec;
      const uint32_t wd = tr[q & 255u];
      return (int)reinterpret_cast<const uint16_t *>(tr + 256)[q & 255u] + __popc(wd & ((1u << (off & 31u)) - 1u));
    };
    auto acc_known = [&](bool a0, uint32_t c0, double v0, bool a1, uint32_t c1, double v1) {
      const int r0 = a0 ? rank_of(c0) : 0, r1 = a1 ? rank_of(c1) : 0;
      add2_shared_f64(a0, rv_sa + 8u * r0, v0, a1, rv_sa + 8u * r1, v1);  // c_ij <- c_ij + value (l.8)
      if (a0) rcol[r0] = (int32_t)c0;  // (every product of the key stores the same column)
      if (a1) rcol[r1] = (int32_t)c1;
    };
    auto acc_hash1 = [&](bool act, uint32_t c, double v) {
      bool isnew = false;
      uint32_t slot = 0;
      if (act) {
        slot = probe_chunk(hk, c, logT, &isnew);
        atomicAdd(hv + hash_vslot(slot, logT), v);  // c_ij <- c_ij + value (l.8)
      }
      const unsigned m = __ballot_sync(kFull, isnew);
      if (m) {
        const int leader = __ffs(m) - 1;
        int b0 = 0;
        if (lane == leader) b0 = atomicAdd(&s_cnt, __popc(m));
        b0 = __shfl_sync(kFull, b0, leader);
        if (isnew) slot_of[b0 + __popc(m & ((1u << lane) - 1u))] = (uint16_t)slot;
      }
    };
    auto acc_hash = [&](bool a0, uint32_t c0, double v0, bool a1, uint32_t c1, double v1) {
      acc_hash1(a0, c0, v0);
      acc_hash1(a1, c1, v1);
    };
    for (int cb = 0; cb < na; cb += kTEnt) {
      const int n = min(kTEnt, na - cb);
      // the previous chunk's rounds are done with the staged lists (the
      // first chunk follows the publish barrier of the previous part: its
      // emit is done, and the table init is ordered before the rounds by
      // the staging barrier below); the other parity's reservations were
      // last read before the barrier ending the previous chunk's staging
      if (cb > 0) __syncthreads();
      if (threadIdx.x == 0) s_res[par ^ 1][0] = s_res[par ^ 1][1] = 0ull;
      const long long ca = instr ? clock64() : 0;
      // stage: thread owns entries [t*per, t*per + per), per <= 2; entries
      // with a nonempty segment in [t0, t1) go to the short or the long
      // list.  Each warp reserves its slots with one packed (entries,
      // products/rounds) atomic per list, so within a list the products /
      // rounds prefix increases with the slot (round owner searches)
      constexpr int kPer = (kTEnt + THREADS - 1) / THREADS;
      int Ls[kPer], s0s[kPer];
      double avs[kPer];
      unsigned long long vS = 0, vL = 0;  // (entries << 32) | products (short) / rounds (long)
      if (cb == 0 && pf_n > 0) cp_async_wait_all();  // (this thread's own prefetch)
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int j = (int)threadIdx.x + u * THREADS;  // (entries strided over the threads)
        Ls[u] = 0;
        if (j < n) {
          int s0, e0;
          if (cb == 0 && j < pf_n) {  // prefetched while the previous part ran
            s0 = pf_s0[j];
            e0 = pf_e0[j];
            avs[u] = pf_val[j];
          } else {
            const int k = __ldg(A.col + as + cb + j);
            s0 = __ldg(tk0 + k);
            e0 = __ldg(tk1 + k);
            avs[u] = __ldg(A.val + as + cb + j);
          }
          s0s[u] = s0;
          Ls[u] = e0 - s0;
          if (Ls[u] >= kTLongSeg) vL += (1ull << 32) | (unsigned long long)((Ls[u] + 31) >> 5);
          else if (Ls[u] > 0) vS += (1ull << 32) | (unsigned long long)Ls[u];
        }
      }
      unsigned long long iS = vS, iL = vL;  // warp inclusive scans
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long tS = __shfl_up_sync(kFull, iS, o), tL = __shfl_up_sync(kFull, iL, o);
        if (lane >= o) { iS += tS; iL += tL; }
      }
      unsigned long long bS = 0, bL = 0;
      if (lane == 31) {
        if (iS) bS = atomicAdd(&s_res[par][0], iS);
        if (iL) bL = atomicAdd(&s_res[par][1], iL);
      }
      bS = __shfl_sync(kFull, bS, 31) + iS - vS;
      bL = __shfl_sync(kFull, bL, 31) + iL - vL;
      int xs = (int)(bS >> 32), xp = (int)(bS & 0xFFFFFFFFu);
      int xl = (int)(bL >> 32), xr = (int)(bL & 0xFFFFFFFFu);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        if (Ls[u] >= kTLongSeg) {
          ls[xl] = s0s[u];
          ll[xl] = Ls[u];
          la[xl] = avs[u];
          lpre[xl] = xr;
          xr += (Ls[u] + 31) >> 5;
          ++xl;
        } else if (Ls[u] > 0) {
          es[xs] = s0s[u];
          ea[xs] = avs[u];
          epre[xs] = xp;
          xp += Ls[u];
          ++xs;
        }
      }
      if (kTpartInstr) {  // (measurement: products of the long segments)
        unsigned long long lp = 0;
#pragma unroll
        for (int u = 0; u < kPer; ++u) lp += Ls[u] >= kTLongSeg ? (unsigned long long)Ls[u] : 0ull;
        if (lp) atomicAdd(dbg + (dense ? 12 : 13), lp);
      }
      if (cb == 0 && threadIdx.x == 0) cp_async_wait_all();  // (the next part's records: s_Pn)
      __syncthreads();
      if (cb == 0) {
        // prefetch, stage 1: the next part's first kTPf entries (A.col, A.val)
        pf_n = 0;
        if (s_pn_ok) {
          const int4 Qn1 = s_Pn[1];
          const int64_t asn = (int64_t)(((unsigned long long)(unsigned)Qn1.y << 32) | (unsigned)Qn1.x);
          pf_n = min(Qn1.z, kTPf);
          if ((int)threadIdx.x < pf_n) {
            cp_async4(pf_col + threadIdx.x, A.col + asn + threadIdx.x);
            cp_async8(pf_val + threadIdx.x, A.val + asn + threadIdx.x);
            cp_async_commit();
          }
        }
      }
      const unsigned long long tS = s_res[par][0], tL = s_res[par][1];
      par ^= 1;
      const int nS = (int)(tS >> 32), PS = (int)(tS & 0xFFFFFFFFu);
      const int nL = (int)(tL >> 32), RL = (int)(tL & 0xFFFFFFFFu);
      const long long cbk = instr ? clock64() : 0;
      const int RS = (PS + 31) >> 5;
      const int gs0 = (int)((int64_t)RS * w / NW), gs1 = (int)((int64_t)RS * (w + 1) / NW);
      const int gl0 = (int)((int64_t)RL * w / NW), gl1 = (int)((int64_t)RL * (w + 1) / NW);
      if (tune & 32) {  // (measurement only: gathers without accumulation; C left unwritten)
        double sink = 0.0;
        auto acc_none = [&](bool a0, uint32_t c0, double v0, bool a1, uint32_t c1, double v1) {
          sink += (a0 ? v0 + (double)c0 : 0.0) + (a1 ? v1 + (double)c1 : 0.0);
        };
        for_long_rounds(B, ls, ll, la, lpre, nL, RL, gl0, gl1, acc_none);
        for_tpart_rounds<2>(B, es, ea, epre, nS, PS, gs0, gs1, acc_none);
        if (sink == 1.2345e300) dbg[13] = 1;
      } else if (dense && !known) {
        for_long_rounds(B, ls, ll, la, lpre, nL, RL, gl0, gl1, acc_dense);
        for_tpart_rounds<2>(B, es, ea, epre, nS, PS, gs0, gs1, acc_dense);
      } else if (known) {
        for_long_rounds(B, ls, ll, la, lpre, nL, RL, gl0, gl1, acc_known);
        for_tpart_rounds<2>(B, es, ea, epre, nS, PS, gs0, gs1, acc_known);
      } else {
        for_long_rounds(B, ls, ll, la, lpre, nL, RL, gl0, gl1, acc_hash);
        for_tpart_rounds<2>(B, es, ea, epre, nS, PS, gs0, gs1, acc_hash);
      }
      if (instr) {
        c_stage += cbk - ca;
        c_rounds += clock64() - cbk;  // (thread 0's own rounds; the barrier wait lands in the next stage)
        prods += (unsigned long long)PS;
      }
    }
    cp_async_wait_all();  // (thread 0: C row start, stripe prefixes; all: prefetch stage 1)
    __syncthreads();
    const long long ce = instr ? clock64() : 0;
    const int64_t out = s_rp0 + P.z;
    if ((int)threadIdx.x < pf_n) {
      // prefetch, stage 2: the two tile offsets of each prefetched entry
      const int4 Qn = s_Pn[0];
      const int k = pf_col[threadIdx.x];
      cp_async4(pf_s0 + threadIdx.x, toff + int64_t(Qn.y & 0xFFFF) * nB + k);
      cp_async4(pf_e0 + threadIdx.x, toff + int64_t(Qn.y >> 16) * nB + k);
      cp_async_commit();
    }
    if (tune & 48) {  // (measurement only: no emit; the dense window is still reset)
      if (dense && !known)
        for (int s2 = threadIdx.x; s2 < kTileCols; s2 += THREADS) dvb[s2] = kNegZeroBits;
    } else if (dense && !known && dpfx != nullptr && P2.z >= 0) {
      // one pass: warp w owns the 512-column stripe w (32-column groups
      // [GPW w, GPW (w + 1))) and starts at the symbolic's count of the
      // tile's keys before it; present slots (bits != -0.0) are stored in
      // column order (coalesced) and reset to -0.0
      constexpr int GPW = (kTileCols / 32) / NW;
      static_assert(GPW * NW * 32 == kTileCols && NW == kDenseStripes, "one stripe per warp");
      const int64_t ob = out + s_dp[w];
      int32_t *cc = c_col + ob;
      double *cvp = c_val + ob;
      const unsigned below = (1u << lane) - 1u;
      const int32_t cbase = (int32_t)lo + w * GPW * 32 + lane;
      int o = 0;
      // batches of kEB groups: every slot value loaded first (no store
      // between the loads, so they are all in flight at once), the batch's
      // slots reset to -0.0 unconditionally, then ballots and coalesced
      // stores from registers
      constexpr int kEB = 8;
      static_assert(GPW % kEB == 0, "emit batches");
#pragma unroll
      for (int j0 = 0; j0 < GPW; j0 += kEB) {
        unsigned long long bits[kEB];
        uint32_t ds[kEB];
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          ds[u] = dense_slot(uint32_t(w * GPW + j0 + u) * 32u + lane);
          bits[u] = dvb[ds[u]];
        }
#pragma unroll
        for (int u = 0; u < kEB; ++u) dvb[ds[u]] = kNegZeroBits;
#pragma unroll
        for (int u = 0; u < kEB; ++u) {
          const bool pres = bits[u] != kNegZeroBits;
          const unsigned m = __ballot_sync(kFull, pres);
          if (pres) {
            const int p = o + __popc(m & below);
            st_c(cc + p, cbase + (j0 + u) * 32);
            st_c(cvp + p, __longlong_as_double(bits[u]));
          }
          o += __popc(m);
        }
      }
    } else if (dense && !known) {
      // warp w owns the 32-column groups [GPW w, GPW (w + 1)) (ascending
      // columns): one pass of ballots over the present slots (bits != -0.0)
      // counts them, a scan of the NW warp totals gives each warp's output
      // start, a second pass stores the present entries (coalesced, ascending
      // columns) and resets their slots to -0.0
      constexpr int GPW = (kTileCols / 32) / NW;
      static_assert(GPW * NW * 32 == kTileCols, "groups per warp");
      unsigned msk[GPW];
      int tot = 0;
#pragma unroll
      for (int j = 0; j < GPW; ++j) {
        const uint32_t off = uint32_t(w * GPW + j) * 32u + lane;
        msk[j] = __ballot_sync(kFull, dvb[dense_slot(off)] != kNegZeroBits);
        tot += __popc(msk[j]);
      }
      if (lane == 0) s_red[w] = tot;
      __syncthreads();
      int64_t o = out + (int)__reduce_add_sync(kFull, lane < w ? (unsigned)s_red[lane] : 0u);
      const unsigned below = (1u << lane) - 1u;
#pragma unroll
      for (int j = 0; j < GPW; ++j) {
        if ((msk[j] >> lane) & 1u) {
          const uint32_t off = uint32_t(w * GPW + j) * 32u + lane;
          const uint32_t ds = dense_slot(off);
          const int64_t p = o + __popc(msk[j] & below);
          st_c(c_col + p, (int32_t)(lo + off));
          st_c(c_val + p, dv[ds]);
          dvb[ds] = kNegZeroBits;
        }
        o += __popc(msk[j]);
      }
    } else if (known && dense) {  // walk the tile's words, a warp per word: coalesced stores
      for (int q = w; q < 256; q += NW) {
        const uint32_t wd = rec[q];
        if (!wd) continue;  // (warp-uniform)
        if ((wd >> lane) & 1u) {
          const int r = reinterpret_cast<const uint16_t *>(rec + 256)[q] + __popc(wd & ((1u << lane) - 1u));
          st_c(c_col + out + r, (int32_t)(lo + q * 32 + lane));
          st_c(c_val + out + r, rv[r]);
        }
      }
    } else if (known) {
      // every key of the part received at least one product, which stored
      // its column at the key's rank: columns and values (rank order = column
      // order) go out as two coalesced copies, no bitmap walk
      for (int r = threadIdx.x; r < cnt; r += THREADS) {
        st_c(c_col + out + r, rcol[r]);
        st_c(c_val + out + r, rv[r]);
      }
    } else if (!sorted) {
      for (int p = threadIdx.x; p < cnt; p += THREADS) {
        const int s = slot_of[p];
        st_c(c_col + out + p, (int32_t)hk[s]);
        st_c(c_val + out + p, hv[hash_vslot(s, logT)]);
      }
    } else {
      // gather the pairs into the entry stage, sort them with the table
      // region as scratch
      uint32_t *gk = reinterpret_cast<uint32_t *>(eb);
      double *gv = reinterpret_cast<double *>(eb + size_t(kTPartKeys) * 4);
      for (int p = threadIdx.x; p < cnt; p += THREADS) {
        const int s = slot_of[p];
        gk[p] = hk[s];
        gv[p] = hv[hash_vslot(s, logT)];
      }
      __syncthreads();
      const int64_t span = (int64_t(t1 - t0)) << kTileLog;
      if (span <= kTRankCols) {
        // narrow part: rank by a bitmap over its columns [lo, lo + span)
        // (table region as scratch): set bits, prefix popcounts per word,
        // position = prefix + bits below in the word
        uint32_t *rbm = reinterpret_cast<uint32_t *>(base);
        int32_t *rpre = reinterpret_cast<int32_t *>(base + size_t(kTRankCols / 32) * 4);
        const int nw = (int)(span >> 5);
        for (int q2 = threadIdx.x; q2 < nw; q2 += THREADS) rbm[q2] = 0u;
        __syncthreads();
        for (int p = threadIdx.x; p < cnt; p += THREADS) {
          const uint32_t off = gk[p] - (uint32_t)lo;
          atomicOr(rbm + (off >> 5), 1u << (off & 31u));
        }
        __syncthreads();
        const int per = (nw + THREADS - 1) / THREADS;
        const int q0 = min(nw, (int)threadIdx.x * per), q1 = min(nw, q0 + per);
        int mine = 0;
        for (int q2 = q0; q2 < q1; ++q2) mine += __popc(rbm[q2]);
        int totr;
        int exr = block_excl_scan_int(mine, s_warp, &totr);
        for (int q2 = q0; q2 < q1; ++q2) {
          rpre[q2] = exr;
          exr += __popc(rbm[q2]);
        }
        __syncthreads();
        // ranks first (u16 after the gathered pairs), then the pairs placed at
        // their ranks in the table region (rbm / rpre are done), then two
        // coalesced copies out
        uint16_t *rk = reinterpret_cast<uint16_t *>(eb + size_t(kTPartKeys) * 12);
        static_assert(size_t(kTPartKeys) * 14 <= kTEntBytes, "ranks after the gathered pairs");
        for (int p = threadIdx.x; p < cnt; p += THREADS) {
          const uint32_t off = gk[p] - (uint32_t)lo;
          const uint32_t wd = off >> 5;
          rk[p] = (uint16_t)(rpre[wd] + __popc(rbm[wd] & ((1u << (off & 31u)) - 1u)));
        }
        __syncthreads();
        int32_t *scol = reinterpret_cast<int32_t *>(base);
        double *sval = reinterpret_cast<double *>(base + size_t(kTPartKeys) * 4);
        for (int p = threadIdx.x; p < cnt; p += THREADS) {
          scol[rk[p]] = (int32_t)gk[p];
          sval[rk[p]] = gv[p];
        }
        __syncthreads();
        for (int r = threadIdx.x; r < cnt; r += THREADS) {
          st_c(c_col + out + r, scol[r]);
          st_c(c_val + out + r, sval[r]);
        }
      } else {
        int NB = 32;
        while (NB < cnt) NB <<= 1;
        uint32_t *scr = reinterpret_cast<uint32_t *>(base);
        block_bucket_sort_to(gk, gv, cnt, NB, scr, scr + NB, scr + NB + kTPartKeys, out, c_col,
                             c_val, s_red);
      }
    }
    if (threadIdx.x == 0) {  // publish the next part (every thread has read this one)
      s_dirty = known || !dense;  // (a dense part's emit leaves its window clean)
      s_q = q_next;
      s_P = s_Pn[0];
      s_P1 = s_Pn[1];
      s_P2 = s_Pn[2];
      q_next = q_after;
    }
    __syncthreads();
    if (instr) {
      const long long cz = clock64();
      atomicAdd(dbg + 0, 1ull);
      atomicAdd(dbg + 1, (unsigned long long)dense);
      atomicAdd(dbg + (dense ? 2 : 3), (unsigned long long)(cz - c0));
      atomicAdd(dbg + (dense ? 4 : 5), prods);  // (short-segment products; long ones in dbg[12])
      atomicAdd(dbg + 6, (unsigned long long)c_stage);
      atomicAdd(dbg + 7, (unsigned long long)c_rounds);
      atomicAdd(dbg + (dense ? 8 : 11), (unsigned long long)(cz - ce));   // emit
      if (!dense && !known) atomicAdd(dbg + 9, (unsigned long long)(cz - ce));  // emit of the hashing parts
      atomicAdd(dbg + 10, (unsigned long long)cnt);
      if (!dense) atomicAdd(dbg + 14, (unsigned long long)(t1 - t0));  // hash part spans (tiles)
      if (known) atomicAdd(dbg + 15, 1ull);                            // parts indexed by tile records
    }
  }
}

// One-phase compaction: row i of the workspace (at the flop prefix fofs[i],
// nnz(c_i) entries) to C at C_row_ptr[i].  A warp per row, coalesced.
__global__ void __launch_bounds__(256) k_onephase_copy(int64_t m, const int64_t *__restrict__ fofs,
                                                       const int64_t *__restrict__ c_rp,
                                                       const int32_t *__restrict__ t_col,
                                                       const double *__restrict__ t_val,
                                                       int32_t *__restrict__ c_col,
                                                       double *__restrict__ c_val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < m; i += nwarps) {
    const int64_t s = fofs[i], d = c_rp[i], n = c_rp[i + 1] - d;
    for (int64_t q = lane; q < n; q += 32) {
      c_col[d + q] = __ldg(t_col + s + q);
      c_val[d + q] = __ldg(t_val + s + q);
    }
  }
}

}  // namespace spg
