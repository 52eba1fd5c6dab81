// spg_internal.cuh -- shared device helpers of the sm_100a hash SpGEMM library.
// Product code: never includes or links anything under oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spgemm.h"

namespace spg {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;     // P:283 "initialized by storing -1"
constexpr uint32_t kHashMul = 2654435761u;   // odd 32-bit constant (reading R5)
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kMinLogT = 5;                  // GPU tables are at least 32 slots
constexpr int64_t kMaxBRow = int64_t(1) << 26;  // 32 rows * 2^26 < 2^31 per chunk

// ---------------------------------------------------------------- bins
// Symbolic bins by T_s = lowest 2^n > min(flop_i, ncols), raised
// to >= 32 slots on the GPU.  Numeric bins by T_n = lowest 2^n >= 2 nnz(c_i)
// (load <= 1/2, reading R6).
enum SymBin { SB_SKIP = 0, SB_W128, SB_W1024, SB_B2K, SB_B4K, SB_B8K, SB_B16K, SB_B32K,
              SB_G, SB_BM, SB_COUNT };
enum NumBin { NB_SKIP = 0, NB_W256, NB_W1024, NB_B2K, NB_B4K, NB_B8K, NB_B16K, NB_G, NB_COUNT };
constexpr int kMaxBins = 12;

struct DevCSR {
  int64_t nrows, ncols;
  const int64_t *__restrict__ rp;
  const int32_t *__restrict__ col;
  const double *__restrict__ val;
};

// Device-side plan summary (atomics target), mirrored to pinned host memory.
struct PlanInfo {
  unsigned long long flop_total;
  unsigned long long max_flop;
  unsigned long long max_brow;
  unsigned long long nnz_total;
  unsigned long long max_nnz;
  unsigned long long sym_count[kMaxBins];
  unsigned long long num_count[kMaxBins];
  unsigned long long cursor[kMaxBins];
  unsigned long long num_cursor[kMaxBins];
  unsigned long long mask_sum;
  unsigned long long flags;
  unsigned long long max_arow;    // max nnz(a_i)
  unsigned long long b_unsorted;  // nonzero iff some B row is not strictly increasing
  unsigned long long parts_used;  // bump allocator of the parts buffer
  unsigned long long parts_overflow;
  unsigned long long row_counter;   // dynamic work queue of the numeric G tier
  unsigned long long b_end;         // B.row_ptr[B.nrows] (tile offsets are int32 positions)
  unsigned long long b_empty;       // empty rows of B (k_b_rowmask)
  unsigned long long useful;        // a_ik whose B row is nonempty (k_flop_nz)
  unsigned long long a_nnz;         // nnz of A (k_flop_nz)
  unsigned long long mask_ctr[2];   // row queues of the fused mask-and-sum kernels
  double mask_acc;                  // their fp64 sum
  unsigned long long mask_n[2];     // lengths of their row lists (warp tier, block tier)
  unsigned long long mask_isum;     // exact int64 sum of the warp partials (two's complement)
  unsigned long long mask_inexact;  // nonzero: some warp partial was not an integer below 2^53
  unsigned long long pkeys_used;    // tile records wanted by the narrow hash parts (exact count)
  unsigned long long parts_pool;    // parts slots handed out in per-block chunks (>= parts_used; holes have row -1)
  unsigned long long pkeys_pool;    // tile records handed out in per-block chunks
  unsigned long long lists_need;    // keys of the rows that want a sorted column list (exact count)
  unsigned long long lists_pool;    // list entries handed out in per-block chunks
  unsigned long long heap_count[kMaxBins];   // rows of each numeric bin taken by the heap tier
  unsigned long long heap_cursor[kMaxBins];  // (scatter cursors, from the back of the bin)
  unsigned long long dbg[16];       // measurement counters (SPG_TUNE bit 8 instrumentation)
};

__host__ __device__ __forceinline__ int log2_ceil64(uint64_t x) {  // smallest n: 2^n >= x
#ifdef __CUDA_ARCH__
  return x <= 1 ? 0 : 64 - __clzll((long long)(x - 1));
#else
  int n = 0;
  while ((uint64_t(1) << n) < x) ++n;
  return n;
#endif
}

// log2 of the paper's symbolic table size: lowest 2^n STRICTLY greater than
// min(flop, ncols)  (Fig:hash_spgemm l.10-12).
__host__ __device__ __forceinline__ int sym_log2_paper(int64_t flop, int64_t ncols) {
  const int64_t s = flop < ncols ? flop : ncols;
#ifdef __CUDA_ARCH__
  return s <= 0 ? 0 : 64 - __clzll((long long)s);  // bits of s = lowest n: 2^n > s
#else
  int n = 0;
  while ((int64_t(1) << n) <= s) ++n;
  return n;
#endif
}

__device__ __forceinline__ int sym_log2_gpu(int64_t flop, int64_t ncols) {
  int n = sym_log2_paper(flop, ncols);
  return n < kMinLogT ? kMinLogT : n;
}

// Rows whose table would exceed 8192 slots use the smem BITMAP tier when the
// column space fits one (it also cuts the row into column-range parts for the
// numeric phase); otherwise the larger smem hash tables / global hash.
constexpr int64_t kBitmapMaxCols = int64_t(200 * 1024) * 8;  // 200 KB of bits
// Warp tiers probe 4-slot chunks (one LDS.128 per probe; SPG_WARP_CHUNK=0:
// scalar linear probing, the round-1 warp tiers)
#ifndef SPG_WARP_CHUNK
#define SPG_WARP_CHUNK 0
#endif
#ifndef SPG_MED_BM
#define SPG_MED_BM 0
#endif

// Rows with more than kWarpMaxEntries a_ik go to a block tier even when their
// table is small: one warp would walk all their a_ik alone.
constexpr int64_t kWarpMaxEntries = 512;

__device__ __forceinline__ int sym_bin(int64_t flop, int64_t ncols, int64_t na) {
  if (flop == 0) return SB_SKIP;
  int n = sym_log2_gpu(flop, ncols);
  if (na > kWarpMaxEntries && n <= 10) return SB_B2K;
  if (n <= 7) return SB_W128;
  if (n <= 10) return SB_W1024;
  // rows of 1024..8191 products: the bitmap tier when the column space fits
  // (it hands the numeric block tier the row's sorted column list)
  if (n <= 13 && (!SPG_MED_BM || ncols > kBitmapMaxCols)) return SB_B2K + (n - 11);
  if (ncols <= kBitmapMaxCols) return SB_BM;
  if (n <= 15) return SB_B2K + (n - 11);
  return SB_G;
}

// Column tiles of the long-row tier (numeric G tier, B rows sorted): every B
// row is cut at multiples of kTileCols columns (tile offsets built once per
// multiply, k_tile_offsets), and a long row of C is cut into PARTS = runs of
// consecutive tiles holding <= kTPartKeys keys (smem hash table) or one tile
// holding more (dense smem window).  Rows with nnz(c_i) > kPartMinKeys get
// parts (the numeric G bin).
constexpr int kTileLog = 13;
constexpr int kTileCols = 1 << kTileLog;
#ifndef SPG_TPART_KEYS
#define SPG_TPART_KEYS 2048
#endif
constexpr int kTPartKeys = SPG_TPART_KEYS;
constexpr int kPartMinKeys = 8192;
constexpr int kMaxTiles = 256;  // >= kBitmapMaxCols / kTileCols + 1

__device__ __forceinline__ int num_log2(int64_t nnz) {
  int n = log2_ceil64(uint64_t(2 * nnz));
  return n < kMinLogT ? kMinLogT : n;
}

__device__ __forceinline__ int num_bin(int64_t nnz, int64_t na) {
  if (nnz == 0) return NB_SKIP;
  int n = num_log2(nnz);
  if (na > kWarpMaxEntries && n <= 10) return NB_B2K;
  if (n <= 8) return NB_W256;
  if (n <= 10) return NB_W1024;
  if (n <= 14) return NB_B2K + (n - 11);
  return NB_G;
}

// Heap tier (§4.2.3 Heap SpGEMM):
// with sorted output, a warp-tier row whose B rows are sorted, with nnz(a_i)
// <= kHeapMax and flop_i <= kHeapMaxFlop, is computed by a per-thread k-way
// heap merge when the paper's cost model says so (accumulator mode AUTO):
//   T_heap = flop_i * log2 nnz(a_i)                          (Eq:heap_est)
//   T_hash = flop_i * c + nnz(c_i) * log2 nnz(c_i)           (Eq:hash_est)
// with c the collision factor (measured: DESIGN.md §9c) and T_heap scaled by
// h, the cost of one heap step relative to one hash probe on this GPU
// (measured on B200; h = 1 is the paper's unit-cost model).
// Mode HASH never, HEAP always (for the eligible rows).
enum AccumMode { ACC_AUTO = 0, ACC_HASH = 1, ACC_HEAP = 2 };
constexpr int kHeapMax = 16;
constexpr int64_t kHeapMaxFlop = 2048;  // bounds one thread's serial merge

__device__ __forceinline__ bool heap_pick(int bin, int64_t flop, int64_t na, int64_t nnz,
                                          int accum, float cfac, bool b_sorted, float hfac) {
  if (accum == ACC_HASH || !b_sorted || nnz <= 0 || na > kHeapMax || flop > kHeapMaxFlop ||
      (bin != NB_W256 && bin != NB_W1024))
    return false;
  if (accum == ACC_HEAP) return true;
  const float th = hfac * (float)flop * log2f((float)na);
  const float tc = (float)flop * cfac + (float)nnz * log2f((float)nnz);
  return th < tc;
}

// One-phase tables (spg_onephase): T = lowest 2^n >= 2 min(flop_i, ncols)
// -- the flop bound stands in for nnz(c_i) in the numeric rule (load <= 1/2,
// reading R6; the sorted emits use the free upper half as scratch) -- binned
// like the symbolic tiers: W128 / W1024 / B2K..B16K; larger -> SB_G (the
// one-phase path refuses those rows).
__device__ __forceinline__ int onep_log2(int64_t flop, int64_t ncols) {
  const int64_t s = flop < ncols ? flop : ncols;
  const int n = log2_ceil64(uint64_t(2 * s));
  return n < kMinLogT ? kMinLogT : n;
}

__device__ __forceinline__ int onep_bin(int64_t flop, int64_t ncols, int64_t na) {
  if (flop == 0) return SB_SKIP;
  const int n = onep_log2(flop, ncols);
  if (na > kWarpMaxEntries && n <= 10) return SB_B2K;
  if (n <= 7) return SB_W128;
  if (n <= 10) return SB_W1024;
  if (n <= 14) return SB_B2K + (n - 11);
  return SB_G;
}

// Fibonacci hashing: HIGH bits of col*H (reading R5 of DESIGN.md; the paper's
// "multiplied by constant number and divided by hash table size to compute
// the remainder", with the remainder taken on the high bits).
__device__ __forceinline__ uint32_t hash_slot(uint32_t c, int logT) {
  return (c * kHashMul) >> (32 - logT);
}

// ---------------------------------------------------------------------------
// HashVector-style probing of SHARED-memory tables (§4.2.2, P:329-338:
// "the hash indicates the identifier of target chunk in hash table"; compare
// the key against the whole chunk; "new element is pushed ... in order from
// the beginning" of the chunk; "when the chunk is occupied with other keys,
// the next chunk is to be checked in accordance with linear probing").  A
// chunk is kChunk = 4 consecutive 32-bit slots read with one 128-bit shared
// load, so a lane resolves most keys in one step and the warp's divergent
// probe loop is short.
// ---------------------------------------------------------------------------
constexpr int kChunkLog = 2;

__device__ __forceinline__ uint4 lds_volatile_v4(const uint32_t *p) {
  uint4 r;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(a));
  return r;
}

// Find or insert key c in smem table keys[0, 2^logT); returns the slot and
// sets *isnew when this call inserted c.
__device__ __forceinline__ uint32_t probe_chunk(uint32_t *keys, uint32_t c, int logT,
                                                bool *isnew) {
  const uint32_t cmask = (1u << (logT - kChunkLog)) - 1u;
  uint32_t ch = (c * kHashMul) >> (32 - (logT - kChunkLog));
  while (true) {
    const uint32_t b = ch << kChunkLog;
    const uint4 k = lds_volatile_v4(keys + b);
    if (k.x == c) return b;
    if (k.y == c) return b + 1;
    if (k.z == c) return b + 2;
    if (k.w == c) return b + 3;
    const int e = k.x == kEmpty ? 0 : k.y == kEmpty ? 1 : k.z == kEmpty ? 2 : k.w == kEmpty ? 3 : 4;
    if (e < 4) {
      const uint32_t old = atomicCAS(keys + b + e, kEmpty, c);
      if (old == kEmpty) { *isnew = true; return b + e; }
      if (old == c) return b + e;
      continue;  // lost the slot to another key: re-read this chunk
    }
    ch = (ch + 1u) & cmask;  // chunk full: next chunk (linear probing)
  }
}

// Slot of key c, known to be in the (complete) table: chunked probing
// without inserts.
__device__ __forceinline__ uint32_t probe_find(const uint32_t *keys, uint32_t c, int logT) {
  const uint32_t cmask = (1u << (logT - kChunkLog)) - 1u;
  uint32_t ch = (c * kHashMul) >> (32 - (logT - kChunkLog));
  while (true) {
    const uint32_t b = ch << kChunkLog;
    const uint4 k = *reinterpret_cast<const uint4 *>(keys + b);
    if (k.x == c) return b;
    if (k.y == c) return b + 1;
    if (k.z == c) return b + 2;
    if (k.w == c) return b + 3;
    ch = (ch + 1u) & cmask;
  }
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }



template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(kFull, v, o);
    if (l >= o) v += t;
  }
  return v;
}

// Owner lane of flattened product p inside a chunk: number of lanes whose
// inclusive end is <= p (ends are nondecreasing across lanes).
__device__ __forceinline__ int owner_lane(int incl, int p) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    int v = __shfl_sync(kFull, incl, pos + s - 1);
    if (v <= p) pos += s;
  }
  return pos;
}

__device__ __forceinline__ int64_t shfl_i64(int64_t v, int src) {
  return __shfl_sync(kFull, v, src);
}

__device__ __forceinline__ double shfl_f64(double v, int src) {
  return __shfl_sync(kFull, v, src);
}

// fp64 add into shared memory for the (rare) case where several lanes of one
// round share a key: a CAS loop (sm_100a has no native fp64 ATOMS add).
__device__ __forceinline__ void smem_add_f64(double *addr, double v) {
  atomicAdd(addr, v);
}

}  // namespace spg
