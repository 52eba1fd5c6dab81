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

// Warp-private shared-memory table, CAS-first probing (switch
// SPG_SYM_CASFIRST): one ATOMS.CAS per probe decides hit / inserted / occupied
// (no load + compare + conditional CAS), so the divergent probe loop has one
// exit test per step.  Measured on C2 (k_sym_warp<1024>): 0.606 -> 0.565 ms.
#ifndef SPG_SYM_CASFIRST
#define SPG_SYM_CASFIRST 1
#endif
__device__ __forceinline__ int sym_insert_cas(uint32_t *tab, uint32_t c, int logT) {
  const uint32_t mask = (1u << logT) - 1u;
  uint32_t h = hash_slot(c, logT);
  while (true) {
    const uint32_t old = atomicCAS(tab + h, kEmpty, c);
    if (old == kEmpty) return 1;
    if (old == c) return 0;
    h = (h + 1u) & mask;  // linear probing
  }
}

// Block tiers (block-shared tables): CAS-first single-slot probing instead of
// the 4-slot chunks (A/B switch; also the numeric block tier's key probe).
// Measured on C3: numeric block tiers 27.4 -> 26.2 ms, symbolic block tiers
// 11.3 -> 25.0 ms (hits on hot columns become same-word atomics): off.
#ifndef SPG_BLOCK_CASFIRST
#define SPG_BLOCK_CASFIRST 0
#endif

// Same, for a shared-memory table (chunked probing).
__device__ __forceinline__ int sym_insert_smem(uint32_t *tab, uint32_t c, int logT) {
  bool isnew = false;
  probe_chunk(tab, c, logT, &isnew);
  return isnew ? 1 : 0;
}

// Column bitmap of the long-row tiers, laid out per 8192-column tile with the
// bits TRANSPOSED: column offset o in tile t is bit (o >> 8) of word
// 256 t + (o & 255).  The 32 consecutive columns of a sequential round (a
// dense run of one sorted B row, R-MAT hub rows) then hit 32 different words
// in 32 banks instead of ORing one word 32 times (measured: 85% of the
// bitmap's atomic wavefronts were bank conflicts), and each tile still owns
// the same 256 words (the per-tile key counts are unchanged).
__device__ __forceinline__ uint32_t tbm_word(uint32_t c) {
  return ((c >> kTileLog) << (kTileLog - 5)) + (c & 255u);
}
__device__ __forceinline__ uint32_t tbm_bit(uint32_t c) { return 1u << ((c >> 8) & 31u); }

// Tile records of the narrow hash parts (k_sym_bitmap -> k_num_tpart): 256
// bitmap words + 256 u16 ranks per 8192-column tile.
constexpr int kTileRec = 256 + 128;
#ifndef SPG_PBITS_SPAN
#define SPG_PBITS_SPAN 24
#endif
constexpr int kPbitsMaxSpan = SPG_PBITS_SPAN;
constexpr int kDenseStripes = 16;
// The bitmap symbolic hands out parts slots and tile records from per-block
// pools refilled kPoolParts / kPoolRecs at a time (one global atomic per
// refill instead of two round trips per row); unused part slots are marked
// with row -1 and skipped by the parts bucket sort.
constexpr int kPoolParts = 512;
constexpr int kPoolRecs = 2048;
constexpr int kPoolList = 65536;  // sorted column lists of the block-tier rows (entries per pool chunk)  // 512-column stripes of a dense tile (one per numeric warp)  // tiles (the record set must fit the numeric's smem region)

// Which parts get tile records: the narrow multi-tile (hash) parts; with
// SPG_DENSE_RECORDS also the single-tile (dense) ones (A/B, DESIGN.md §9b:
// C3 parts kernel -10 ms sorted but bitmap symbolic +18 ms, not adopted).
#ifndef SPG_DENSE_RECORDS
#define SPG_DENSE_RECORDS 0
#endif
__device__ __forceinline__ bool rec_part(int t0, int t1) {
  return t1 - t0 <= kPbitsMaxSpan && (SPG_DENSE_RECORDS || t1 > t0 + 1);
}

// Bitmap variant for very long rows: column c -> bit c of an ncols-bit set.
__device__ __forceinline__ int sym_bitmap_insert(uint32_t *bm, uint32_t c) {
  const uint32_t bit = 1u << (c & 31u);
  return (atomicOr(bm + (c >> 5), bit) & bit) ? 0 : 1;
}

// ---------------------------------------------------------------------------
// Product enumeration.  The products of a row are cut into ROUNDS of <= 32
// products; f(active, col, a_ik * b_kj) is called by all 32 lanes of a warp
// once per round.
//  - sequential rounds (kSeq): a round is <= 32 consecutive b_kj of ONE B row,
//    so the keys of a round are distinct (CSR rows hold unique columns);
//  - flattened rounds: 32 consecutive products of the row's product list,
//    whatever the B-row lengths (full lanes for short B rows).
// With NW warps per row (B/G tiers) each chunk of 32 a_ik has its rounds cut
// into NW contiguous ranges, one per warp, so a row with few a_ik but long B
// rows still keeps every warp busy; a warp takes two rounds per step (two
// independent gathers in flight).
// `entry(j) -> Entry{bs, len, a}` describes entry j of the row: the B
// segment [bs, bs+len) that its a_ik multiplies.  kVal = false skips values.
// ---------------------------------------------------------------------------
constexpr int kFlatAvgLen = 12;  // kAutoFlat: chunks averaging shorter B rows run flattened

struct Entry {
  int64_t bs;
  int len;
  double a;
};

// Long B rows deferred to a block-wide walk (for_entries, dynamic chunks).
constexpr int kLongLen = 64;
constexpr int kLongCap = 256;
struct DeferList {
  long long bs[kLongCap];
  double a[kLongCap];
  int len[kLongCap];
  int n;
};

template <bool kSeq, bool kVal, int kDepth, bool kAutoFlat = false, typename EF, typename F>
__device__ __forceinline__ void for_entries(const DevCSR &B, int64_t nent, int w, int NW,
                                            EF &&entry, F &&f, int *next = nullptr,
                                            DeferList *dl = nullptr) {
  const int lane = lane_id();
  // Many chunks: each warp owns whole chunks (chunk overhead paid once) --
  // taken from the block's counter `next` when given (chunk costs differ with
  // the B-row lengths), else strided.  Few chunks: every warp walks every
  // chunk and takes a contiguous slice of its rounds (keeps all warps busy on
  // rows with few, long B rows).
  const int64_t nchunks = (nent + 31) >> 5;
  const bool own_chunks = NW == 1 || nchunks >= 2 * int64_t(NW);
  const bool dyn = own_chunks && next != nullptr && NW > 1;
  auto next_chunk = [&](int64_t cur) -> int64_t {
    if (!dyn) return own_chunks ? cur + int64_t(NW) * 32 : cur + 32;
    int v = 0;
    if (lane == 0) v = atomicAdd(next, 32);
    return (int64_t)__shfl_sync(kFull, v, 0);
  };
  int64_t cb0 = own_chunks ? int64_t(w) * 32 : 0;
  if (dyn) cb0 = next_chunk(0);
  // the per-chunk walk (own = this warp owns the chunk; else every warp
  // takes a contiguous slice of the chunk's rounds)
  auto body = [&](Entry en, bool own) {
    // kAutoFlat (f tolerates equal keys inside a round): a chunk of short B
    // rows (average < kFlatAvgLen) runs flattened (full lanes) even in a
    // sequential row
    bool seq = kSeq;
    if (kSeq && kAutoFlat && own) {
      const int sum = (int)__reduce_add_sync(kFull, (unsigned)en.len);
      const int ne = __popc(__ballot_sync(kFull, en.len > 0));
      seq = sum >= kFlatAvgLen * ne;
    }
    if (seq && own && __all_sync(kFull, en.len <= 32)) {
      // this warp owns the chunk and every B row fits one round: one round per
      // nonempty entry.  kDepth <= 2 (warp tiers, occupancy-bound): one round
      // ahead.  Deeper (block / bitmap tiers): rolling software pipeline over
      // kDepth register slots -- slot d holds the gathered (b_kj, a_ik) of a
      // round; right after a round is hashed its slot is refilled with the
      // round kDepth ahead, so kDepth independent gathers stay in flight.
      unsigned pend = __ballot_sync(kFull, en.len > 0);
      if constexpr (kDepth <= 2) {
        // one round ahead: the gathers of the next round are issued before
        // this one is hashed
        if (!pend) return;
        int j = __ffs(pend) - 1;
        pend &= pend - 1;
        int L = __shfl_sync(kFull, en.len, j);
        double aj = kVal ? shfl_f64(en.a, j) : 0.0;
        int64_t jbs = shfl_i64(en.bs, j);
        bool act = lane < L;
        uint32_t c = act ? (uint32_t)__ldg(B.col + jbs + lane) : 0u;
        double bv = (kVal && act) ? __ldg(B.val + jbs + lane) : 0.0;
        while (true) {
          const bool more = pend != 0;
          int nL = 0;
          double na = 0.0;
          uint32_t nc = 0u;
          double nbv = 0.0;
          if (more) {
            const int nj = __ffs(pend) - 1;
            pend &= pend - 1;
            nL = __shfl_sync(kFull, en.len, nj);
            if (kVal) na = shfl_f64(en.a, nj);
            const int64_t nbs = shfl_i64(en.bs, nj);
            if (lane < nL) {
              nc = (uint32_t)__ldg(B.col + nbs + lane);
              if (kVal) nbv = __ldg(B.val + nbs + lane);
            }
          }
          f(act, c, aj * bv);  // value <- a_ik * b_kj (Fig:code_spgemm l.5)
          if (!more) break;
          act = lane < nL;
          c = nc;
          bv = nbv;
          aj = na;
        }
        return;
      }
      int sl[kDepth];
      uint32_t sc[kDepth];
      double sb[kDepth], sa[kDepth];
      auto fill = [&](int d) {
        sl[d] = 0;
        if (pend) {  // warp-uniform
          const int j = __ffs(pend) - 1;
          pend &= pend - 1;
          sl[d] = __shfl_sync(kFull, en.len, j);
          if (kVal) sa[d] = shfl_f64(en.a, j);
          const int64_t bs = shfl_i64(en.bs, j);
          if (lane < sl[d]) {
            sc[d] = (uint32_t)__ldg(B.col + bs + lane);
            if (kVal) sb[d] = __ldg(B.val + bs + lane);
          }
        }
      };
#pragma unroll
      for (int d = 0; d < kDepth; ++d) fill(d);
      bool more = sl[0] > 0;
      while (more) {
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
          if (sl[d] == 0) { more = false; break; }  // rounds are slotted in order
          const bool act = lane < sl[d];
          f(act, act ? sc[d] : 0u, (kVal && act) ? sa[d] * sb[d] : 0.0);  // a_ik * b_kj (l.5)
          fill(d);
        }
      }
      return;
    }
    if ((kDepth <= 2 || !kVal) && seq && own) {
      // warp tiers and the symbolic walks: the nonempty entries directly
      // (measured: the pipelined walker below costs the occupancy-bound warp
      // kernels registers, and the symbolic bitmap tier time)
      unsigned pend = __ballot_sync(kFull, en.len > 0);
      while (pend) {
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        const int64_t jbs = shfl_i64(en.bs, j);
        const int L = __shfl_sync(kFull, en.len, j);
        const double aj = kVal ? shfl_f64(en.a, j) : 0.0;
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
      return;
    }
    if (seq && own) {
      // this warp owns the chunk (some B rows longer than 32): walk its
      // nonempty entries, a round = 32 consecutive b_kj of one B row, with
      // the gathers of the next round issued before this one is applied
      unsigned pend = __ballot_sync(kFull, en.len > 0);
      if (!pend) return;
      int L = 0, t = -32;
      int64_t jbs = 0;
      double aj = 0.0;
      auto next_round = [&]() -> bool {  // warp-uniform
        t += 32;
        if (t < L) return true;
        if (!pend) return false;
        const int j = __ffs(pend) - 1;
        pend &= pend - 1;
        jbs = shfl_i64(en.bs, j);
        L = __shfl_sync(kFull, en.len, j);
        if (kVal) aj = shfl_f64(en.a, j);
        t = 0;
        return true;
      };
      next_round();
      bool act = t + lane < L;
      uint32_t c = act ? (uint32_t)__ldg(B.col + jbs + t + lane) : 0u;
      double bv = (kVal && act) ? __ldg(B.val + jbs + t + lane) : 0.0;
      double a = aj;
      while (true) {
        const bool more = next_round();
        bool nact = false;
        uint32_t nc = 0u;
        double nbv = 0.0;
        if (more) {
          nact = t + lane < L;
          if (nact) {
            nc = (uint32_t)__ldg(B.col + jbs + t + lane);
            if (kVal) nbv = __ldg(B.val + jbs + t + lane);
          }
        }
        f(act, c, a * bv);  // value <- a_ik * b_kj (Fig:code_spgemm l.5)
        if (!more) break;
        act = nact;
        c = nc;
        bv = nbv;
        a = aj;
      }
      return;
    }
    const int r = seq ? ((en.len + 31) >> 5) : en.len;  // rounds (seq) or products
    const int incl = warp_incl_scan(r);
    const int total = __shfl_sync(kFull, incl, 31);
    const int nr = seq ? total : ((total + 31) >> 5);
    const int g0 = own ? 0 : (int)((int64_t)nr * w / NW);
    const int g1 = own ? nr : (int)((int64_t)nr * (w + 1) / NW);
    if (g0 >= g1) return;
    if (seq) {
      // the owner entry of round g advances monotonically along [g0, g1)
      int own = 0, obeg = 0, oend = 0, olen = 0;
      int64_t obs = 0;
      double oa = 0.0;
      auto advance = [&](int g) {
        while (g >= oend) {
          own = owner_lane(incl, g);
          oend = __shfl_sync(kFull, incl, own);
          obeg = oend - __shfl_sync(kFull, r, own);
          obs = shfl_i64(en.bs, own);
          olen = __shfl_sync(kFull, en.len, own);
          if (kVal) oa = shfl_f64(en.a, own);
        }
      };
      for (int g = g0; g < g1; g += 2) {
        advance(g);
        const int t0 = (g - obeg) * 32 + lane;
        const bool act0 = t0 < olen;
        const int64_t q0 = obs + t0;
        const double a0 = oa;
        bool act1 = false;
        int64_t q1 = 0;
        double a1 = 0.0;
        if (g + 1 < g1) {
          advance(g + 1);
          const int t1 = (g + 1 - obeg) * 32 + lane;
          act1 = t1 < olen;
          q1 = obs + t1;
          a1 = oa;
        }
        uint32_t c0 = 0u, c1 = 0u;
        double v0 = 0.0, v1 = 0.0;
        if (act0) c0 = (uint32_t)__ldg(B.col + q0);
        if (act1) c1 = (uint32_t)__ldg(B.col + q1);
        if (kVal) {
          if (act0) v0 = a0 * __ldg(B.val + q0);  // value <- a_ik * b_kj (l.5)
          if (act1) v1 = a1 * __ldg(B.val + q1);
        }
        f(act0, c0, v0);
        f(act1, c1, v1);
      }
    } else {
      for (int g = g0; g < g1; ++g) {
        const int p = g * 32 + lane;
        const int own = owner_lane(incl, p);
        const int oex = __shfl_sync(kFull, incl - r, own);
        const int64_t q = shfl_i64(en.bs, own) + (p - oex);
        const double oa = kVal ? shfl_f64(en.a, own) : 0.0;
        const bool act = p < total;
        uint32_t c = 0u;
        double v = 0.0;
        if (act) {
          c = (uint32_t)__ldg(B.col + q);
          if (kVal) v = oa * __ldg(B.val + q);  // value <- a_ik * b_kj (Fig:code_spgemm l.5)
        }
        f(act, c, v);
      }
    }
  };
  // Deferral of long B rows (block tiers, dynamic chunks): an entry with more
  // than kLongLen products would leave its warp walking it alone while the
  // block waits at the row's barrier (R-MAT hub rows); such entries go to a
  // block-shared list that all warps split by rounds after the chunks.
  const bool defer = dyn && dl != nullptr;
  if (defer) {
    if (threadIdx.x == 0) dl->n = 0;
    __syncthreads();
  }
  for (int64_t cb = cb0; cb < nent; cb = next_chunk(cb)) {
    Entry en{0, 0, 0.0};
    if (cb + lane < nent) en = entry(cb + lane);
    if (defer) {
      const bool lg = en.len > kLongLen;
      const unsigned m = __ballot_sync(kFull, lg);
      if (m) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&dl->n, __popc(m));
        base = __shfl_sync(kFull, base, 0);
        const int idx = base + __popc(m & ((1u << lane) - 1u));
        if (lg && idx < kLongCap) {
          dl->bs[idx] = en.bs;
          dl->len[idx] = en.len;
          if (kVal) dl->a[idx] = en.a;
          en.len = 0;  // walked below by the whole block
        }
      }
    }
    body(en, own_chunks);
  }
  if (defer) {
    __syncthreads();
    const int nl = min(dl->n, kLongCap);
    for (int c0 = 0; c0 < nl; c0 += 32) {
      Entry en{0, 0, 0.0};
      if (c0 + lane < nl) {
        en.bs = dl->bs[c0 + lane];
        en.len = dl->len[c0 + lane];
        en.a = kVal ? dl->a[c0 + lane] : 0.0;
      }
      body(en, false);
    }
  }
}

// All products of row [as, ae) of A.
template <bool kSeq, bool kVal, int kDepth = (kVal ? 4 : 8), bool kAutoFlat = false, typename F>
__device__ __forceinline__ void for_row(const DevCSR &A, const DevCSR &B, int64_t as,
                                        int64_t ae, int w, int NW, F &&f, int *next = nullptr,
                                        DeferList *dl = nullptr) {
  for_entries<kSeq, kVal, kDepth, kAutoFlat>(
      B, ae - as, w, NW,
      [&](int64_t j) {
        const int k = __ldg(A.col + as + j);
        Entry en;
        en.bs = __ldg(B.rp + k);
        en.len = (int)(__ldg(B.rp + k + 1) - en.bs);
        en.a = kVal ? __ldg(A.val + as + j) : 0.0;
        return en;
      },
      f, next, dl);
}

// Rows whose B rows average >= kSeqMinLen entries use the sequential
// enumeration (no owner search, distinct keys per round); shorter ones the
// flattened one (full 32-lane rounds).
#ifndef SPG_SEQ_MIN_LEN
#define SPG_SEQ_MIN_LEN 16
#endif
constexpr int kSeqMinLen = SPG_SEQ_MIN_LEN;
__device__ __forceinline__ bool use_seq(int64_t flop, int64_t nnz_a) {
  return flop >= int64_t(kSeqMinLen) * nnz_a;
}

// ---------------------------------------------------------------------------
// W tier: one warp per row, warp-private table of T <= TMAX slots in smem.
// ---------------------------------------------------------------------------
// HashVector-style warp-bucket insertion (§4.2.2; SURVEY
// §8(f) row 2): the table is cut into 32-slot buckets; the warp takes the
// keys of its lanes one at a time, every lane loads one slot of the key's
// bucket (hash = high bits of key * H over T / 32 buckets), a ballot finds a
// hit or the first empty slot ("pushed ... in order from the beginning" of
// the chunk), a full bucket moves on to the next one (linear probing over
// buckets).  Warp-private table: no atomics.  Returns the new keys (lane 0).
// The A/B variant of the scalar linear probing (SPG_TUNE bit 128).
__device__ __forceinline__ int warp_bucket_insert(uint32_t *tab, int logT, bool act, uint32_t c,
                                                  unsigned long long *probes = nullptr) {
  const int lane = lane_id();
  const uint32_t nbm = (1u << (logT - 5)) - 1u;  // buckets - 1 (logT >= 5)
  int added = 0;
  unsigned pend = __ballot_sync(kFull, act);
  while (pend) {
    const int src = __ffs(pend) - 1;
    pend &= pend - 1;
    const uint32_t key = __shfl_sync(kFull, c, src);
    uint32_t bk = logT > 5 ? (key * kHashMul) >> (32 - (logT - 5)) : 0u;
    while (true) {
      if (probes && lane == 0) ++*probes;
      const uint32_t k = tab[(bk << 5) + lane];
      if (__ballot_sync(kFull, k == key)) break;
      const unsigned emp = __ballot_sync(kFull, k == kEmpty);
      if (emp) {
        if (lane == __ffs(emp) - 1) tab[(bk << 5) + lane] = key;
        ++added;
        break;
      }
      bk = (bk + 1u) & nbm;
    }
    __syncwarp();
  }
  return added;
}

// rounds of one B row in flight per warp in the sequential walk (the gathers
// of the next rounds are issued before the current one is hashed)
#ifndef SPG_SYM_WARP_DEPTH
#define SPG_SYM_WARP_DEPTH 2
#endif
template <int TMAX, int WARPS, bool BUCKET = false>
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
    for (int s = lane * 4; s < T; s += 128)  // T >= 32: 16-byte stores (T % 4 == 0)
      *reinterpret_cast<uint4 *>(tab + s) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    __syncwarp();
    int cnt = 0;
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    auto ins = [&](bool act, uint32_t c, double) {
      if (BUCKET) cnt += warp_bucket_insert(tab, logT, act, c);
      else if (act) cnt += SPG_WARP_CHUNK ? sym_insert_smem(tab, c, logT)
                      : SPG_SYM_CASFIRST ? sym_insert_cas(tab, c, logT) : sym_insert(tab, c, logT);
    };
    if (use_seq(flop[i], ae - as)) for_row<true, false, SPG_SYM_WARP_DEPTH>(A, B, as, ae, 0, 1, ins);
    else for_row<false, false, 2>(A, B, as, ae, 0, 1, ins);
    if (!BUCKET) cnt = warp_sum(cnt);  // (bucket mode: every lane holds the warp's count)
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
  __shared__ int s_cnt, s_next;
  __shared__ DeferList s_dl;  // long B rows walked by the whole block
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = s_dyn_u32;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int logT = sym_log2_gpu(flop[i], B.ncols);
    const int T = 1 << logT;
    for (int s = threadIdx.x; s < T; s += THREADS) tab[s] = kEmpty;
    if (threadIdx.x == 0) { s_cnt = 0; s_next = 0; }
    __syncthreads();
    int cnt = 0;
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    auto ins = [&](bool act, uint32_t c, double) {
      if (act) cnt += SPG_BLOCK_CASFIRST ? sym_insert_cas(tab, c, logT) : sym_insert_smem(tab, c, logT);
    };
    if (use_seq(flop[i], ae - as)) for_row<true, false, 8, true>(A, B, as, ae, w, NW, ins, &s_next, &s_dl);
    else for_row<false, false>(A, B, as, ae, w, NW, ins, &s_next, &s_dl);
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) row_nnz[i] = s_cnt;
  }
}

// Bitmap-tier product walk: the row's a_ik are staged kBmEnt at a time into
// two lists (entries with an empty B row dropped): LONG entries (B row of
// >= 32 entries) at the front of the stage, walked entry by entry in rounds
// of 32 consecutive columns of one B row (two rounds per step, no owner
// search); SHORT ones at the back, cut into FLATTENED rounds of 32
// consecutive products whatever the B-row boundaries (setting a bit twice is
// harmless), the owner entry of each lane's product found from a window of
// the next 32 entry starts.  Each list's rounds are split evenly over the
// warps.  Stage entry: {B row start (int64), length, rounds / products
// before it}.
constexpr int kBmEnt = 1024;  // entries staged per chunk (= block size)
#ifndef SPG_SYM_INSTR
#define SPG_SYM_INSTR 0
#endif
constexpr bool kSymInstr = SPG_SYM_INSTR != 0;
// Bank spreading of the bitmap words: word q is stored at q with its low 5
// bits (the bank) XOR-ed with a multiplicative hash of q >> 5 (a bijection
// inside every 32-word group, so a tile's words stay in the tile's 256).
// R-MAT columns with bits 5-9 clear (a quarter of them) all map to bank 0 of
// their group otherwise.
__device__ __forceinline__ uint32_t bm_phys(uint32_t q) {
  return q ^ (((q >> 5) * 0x9E3779B1u) >> 27);
}
constexpr int kBmD = 4;        // short rounds resolved per batch
#ifndef SPG_BM_LONG
#define SPG_BM_LONG 32
#endif
constexpr int kBmLong = SPG_BM_LONG;  // B rows of >= kBmLong entries walk sequentially
constexpr size_t kBmStageBytes = size_t(kBmEnt) * 16 + 16;

__device__ __forceinline__ void bm_set(uint32_t *bm, uint32_t c) {
  atomicOr(bm + bm_phys(c >> 5), 1u << (c & 31u));  // insert key
}

// last j < n with pre[j] <= x (pre[0] = 0 <= x, nondecreasing, n <= 1024)
__device__ __forceinline__ int bm_find(const int32_t *pre, int n, int x) {
  const int lane = lane_id();
  const int c1 = lane * 32;
  const unsigned b1 = __ballot_sync(kFull, c1 < n && pre[c1] <= x);
  const int blk = 31 - __clz(b1);
  const int c2 = blk * 32 + lane;
  const unsigned b2 = __ballot_sync(kFull, c2 < n && pre[c2] <= x);
  return blk * 32 + 31 - __clz(b2);
}

template <int THREADS>
__device__ __forceinline__ void bm_walk_row(const DevCSR &A, const DevCSR &B, int64_t as,
                                            int64_t ae, uint32_t *bm, int64_t *st_bs,
                                            int32_t *st_len, int32_t *st_pre, int *s_w) {
  static_assert(THREADS == kBmEnt, "one staged entry per thread");
  constexpr int NW = THREADS / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned le = lane == 31 ? kFull : ((2u << lane) - 1u);  // lanes <= this one
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t cb = as; cb < ae; cb += kBmEnt) {
    // stage: thread t holds entry cb + t
    const int64_t e = cb + threadIdx.x;
    int len = 0;
    int64_t bs = 0;
    if (e < ae) {
      const int k = __ldg(A.col + e);
      const int64_t b0 = __ldg(B.rp + k);
      len = (int)(__ldg(B.rp + k + 1) - b0);
      bs = b0;
    }
    const bool lg = len >= kBmLong, sh = len > 0 && !lg;
    const int rl = lg ? (len + 31) >> 5 : 0, ps = sh ? len : 0;
    const unsigned bl = __ballot_sync(kFull, lg), bsh = __ballot_sync(kFull, sh);
    const int irl = warp_incl_scan(rl), ips = warp_incl_scan(ps);
    if (lane == 31) {
      s_w[w] = __popc(bl);
      s_w[32 + w] = irl;
      s_w[64 + w] = __popc(bsh);
      s_w[96 + w] = ips;
    }
    __syncthreads();  // (also: the previous chunk's rounds are done with the stage)
    if (w < 4) {  // four block scans, one per warp
      const int x = lane < NW ? s_w[32 * w + lane] : 0;
      const int xi = warp_incl_scan(x);
      if (lane < NW) s_w[32 * w + lane] = xi - x;
      if (lane == 31) s_w[128 + w] = xi;
    }
    __syncthreads();
    const int nL = s_w[128], RL = s_w[129], nS = s_w[130], PS = s_w[131];
    if (lg) {
      const int x = s_w[w] + __popc(bl & lt);
      st_bs[x] = bs;
      st_len[x] = len;
      st_pre[x] = s_w[32 + w] + irl - rl;
    } else if (sh) {
      const int x = kBmEnt - nS + s_w[64 + w] + __popc(bsh & lt);
      st_bs[x] = bs;
      st_pre[x] = s_w[96 + w] + ips - ps;
    }
    __syncthreads();
    // long entries: rounds [RL w / NW, RL (w + 1) / NW), entry by entry
    {
      const int g0 = (int)((int64_t)RL * w / NW), g1 = (int)((int64_t)RL * (w + 1) / NW);
      if (g0 < g1) {
        int j = bm_find(st_pre, nL, g0);
        int g = g0;
        while (g < g1) {
          const int rb = st_pre[j];
          const int re = min(g1, j + 1 < nL ? st_pre[j + 1] : RL);
          const int L = st_len[j];
          const int32_t *pc = B.col + st_bs[j];
          int t = (g - rb) * 32 + lane;
          // four rounds' column loads in flight per step (the walk waits on
          // these gathers, not on the bitmap ORs)
          for (; g + 7 < re; g += 8, t += 256) {
            uint32_t c[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) c[d] = t + 32 * d < L ? (uint32_t)__ldg(pc + t + 32 * d) : kEmpty;
#pragma unroll
            for (int d = 0; d < 8; ++d)
              if (c[d] != kEmpty) bm_set(bm, c[d]);
          }
          for (; g + 3 < re; g += 4, t += 128) {
            uint32_t c[4];
#pragma unroll
            for (int d = 0; d < 4; ++d) c[d] = t + 32 * d < L ? (uint32_t)__ldg(pc + t + 32 * d) : kEmpty;
#pragma unroll
            for (int d = 0; d < 4; ++d)
              if (c[d] != kEmpty) bm_set(bm, c[d]);
          }
          if (g + 1 < re) {
            const bool a0 = t < L, a1 = t + 32 < L;
            const uint32_t c0 = a0 ? (uint32_t)__ldg(pc + t) : 0u;
            const uint32_t c1 = a1 ? (uint32_t)__ldg(pc + t + 32) : 0u;
            if (a0) bm_set(bm, c0);
            if (a1) bm_set(bm, c1);
            g += 2;
            t += 64;
          }
          if (g < re) {
            if (t < L) bm_set(bm, (uint32_t)__ldg(pc + t));
            ++g;
          }
          ++j;
        }
      }
    }
    // short entries: flattened rounds [R w / NW, R (w + 1) / NW)
    const int64_t *es = st_bs + (kBmEnt - nS);
    const int32_t *epre = st_pre + (kBmEnt - nS);
    const int R = (PS + 31) >> 5;
    const int g0 = (int)((int64_t)R * w / NW), g1 = (int)((int64_t)R * (w + 1) / NW);
    if (g0 < g1) {
      int cur = bm_find(epre, nS, g0 * 32);  // owner of round g0's first product
      for (int g = g0; g < g1; g += kBmD) {
        int64_t q[kBmD];
        bool act[kBmD];
#pragma unroll
        for (int d = 0; d < kBmD; ++d) {
          const int x0 = (g + d) * 32, x = x0 + lane;
          act[d] = (g + d < g1) && x < PS;
          const int ej = cur + 1 + lane;
          const int st = ej < nS ? epre[ej] : INT32_MAX;  // start of entry cur + 1 + lane (> x0)
          const unsigned pos = __reduce_or_sync(kFull, st < x0 + 32 ? (1u << (st - x0)) : 0u);
          const int j = cur + __popc(pos & le);
          cur += __popc(__ballot_sync(kFull, st <= x0 + 32));  // owner of the next round's first product
          q[d] = act[d] ? es[j] + (x - epre[j]) : 0;
        }
        uint32_t c[kBmD];
#pragma unroll
        for (int d = 0; d < kBmD; ++d) c[d] = act[d] ? (uint32_t)__ldg(B.col + q[d]) : 0u;
#pragma unroll
        for (int d = 0; d < kBmD; ++d)
          if (act[d]) bm_set(bm, c[d]);
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// BM tier (bitmap, ncols <= kBitmapMaxCols): the set of distinct columns of
// c_i* is exactly the set bits of an ncols-bit smem bitmap.  When B rows are
// sorted it also cuts rows with nnz > kPartMinKeys into column-tile parts for
// the numeric G tier (spg_internal.cuh): part = three int4 records {row,
// first tile | end tile << 16, keys of the row before the part, keys in the
// part}, {A.row_ptr[row] (lo, hi), nnz(a_row), 0} and {index of the part's
// first tile record in pbits (lo, hi) or -1, 0, 0}.  For the parts spanning
// <= kPbitsMaxSpan tiles the row's bitmap itself is kept: per tile a record
// of kTileRec words = the tile's 256 bitmap words and 256 u16 ranks (keys of
// the PART before each word), so the numeric phase indexes the part's
// columns by rank (no hashing, no occupancy bits).
// ---------------------------------------------------------------------------
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_sym_bitmap(const int32_t *__restrict__ rows,
                                                        int64_t nrows, DevCSR A, DevCSR B,
                                                        const int64_t *__restrict__ flop,
                                                        int64_t *__restrict__ row_nnz,
                                                        PlanInfo *info, int4 *__restrict__ parts,
                                                        int64_t parts_cap,
                                                        uint32_t *__restrict__ pbits,
                                                        int64_t pbits_cap,
                                                        uint16_t *__restrict__ dpfx,
                                                        int64_t *__restrict__ list_off,
                                                        int32_t *__restrict__ lists,
                                                        int64_t lists_cap) {
  extern __shared__ uint32_t s_dyn_u32[];
  __shared__ long long s_lbase, s_lp_cur, s_lp_end;  // this row's sorted column list; the block's list pool
  __shared__ int s_cnt, s_next;
  __shared__ int s_w[132];
  __shared__ int s_dpart[kMaxTiles];  // part index of a dense (single-tile, no record) part at the tile, or -1
  __shared__ long long s_pbase;
  __shared__ long long s_pp_cur, s_pp_end, s_rp_cur, s_rp_end, s_hole_lo, s_hole_hi, s_rbase;
  __shared__ int s_prec[kMaxTiles];  // record tiles of the row's parts before each part
  __shared__ int s_tile[kMaxTiles + 1];  // keys of the row before each column tile
  __shared__ int s_tcnt[kMaxTiles];      // keys of the row in each column tile
  __shared__ int s_cut[kMaxTiles];       // first | (end tile << 16) of each part
  __shared__ int s_nne[kMaxTiles + 1];   // first nonempty tile at or after each tile
  __shared__ long long s_tkoff[kMaxTiles];  // pbits record of a hash part's tile, or -1
  __shared__ int s_tkb[kMaxTiles];          // keys of that part before the tile
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // (words rounded up to whole tiles)
  const int nwords = (int)(((B.ncols + kTileCols - 1) >> kTileLog) << (kTileLog - 5));
  const int ntiles = (int)((B.ncols + kTileCols - 1) >> kTileLog);
  uint32_t *bm = s_dyn_u32;
  int64_t *bm_bs = reinterpret_cast<int64_t *>(s_dyn_u32 + nwords);  // staged entries (bm_walk_row)
  int32_t *bm_len = reinterpret_cast<int32_t *>(bm_bs + kBmEnt);
  int32_t *bm_pre = bm_len + kBmEnt;
  const bool want_parts = parts != nullptr && info->b_unsorted == 0;
  for (int s = threadIdx.x; s < nwords; s += THREADS) bm[s] = 0u;  // (the count pass re-clears)
  if (threadIdx.x == 0) s_pp_cur = s_pp_end = s_rp_cur = s_rp_end = s_lp_cur = s_lp_end = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    const int64_t as = A.rp[i], ae = A.rp[i + 1];
    const long long k0 = kSymInstr ? clock64() : 0;
    // set the bit of every product's column (long / short lists), then count
    // the set bits once
    bm_walk_row<THREADS>(A, B, as, ae, bm, bm_bs, bm_len, bm_pre, s_w);
    const long long k1 = kSymInstr ? clock64() : 0;
    // keys per column tile (a warp per tile); then the exclusive scan over
    // the tiles = keys before each tile, and the row's count
    for (int t = w; t < ntiles; t += NW) {
      const int q0 = t << (kTileLog - 5), q1 = min(nwords, q0 + kTileCols / 32);
      int c = 0;
      for (int q = q0 + lane; q < q1; q += 32) c += __popc(bm[q]);
      c = (int)__reduce_add_sync(kFull, (unsigned)c);
      if (lane == 0) s_tcnt[t] = c;
      if (lane == 0) {
        s_tkoff[t] = -1;
        s_dpart[t] = -1;
      }
    }
    __syncthreads();
    if (w == 0) {
      int carry = 0;
      for (int t0 = 0; t0 < ntiles; t0 += 32) {
        const int v = t0 + lane < ntiles ? s_tcnt[t0 + lane] : 0;
        const int incl = warp_incl_scan(v);
        if (t0 + lane < ntiles) s_tile[t0 + lane] = carry + incl - v;
        carry += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) {
        s_tile[ntiles] = carry;
        s_cnt = carry;
        // a row the numeric BLOCK tier will take (512 < nnz <= 8192: no
        // parts) gets its sorted column list, from the block's list pool
        long long lb = -1;
        if (lists != nullptr && carry > 512 && carry <= kPartMinKeys) {
          atomicAdd(&info->lists_need, (unsigned long long)carry);  // (the host sizes the buffer from it)
          lb = s_lp_cur;
          if (lb + carry > s_lp_end) {
            lb = (long long)atomicAdd(&info->lists_pool, (unsigned long long)kPoolList);
            s_lp_end = lb + kPoolList;
          }
          if (lb + carry > lists_cap) {
            lb = -1;
            s_lp_cur = s_lp_end;
          } else {
            s_lp_cur = lb + carry;
          }
        }
        s_lbase = lb;
        if (list_off != nullptr) list_off[i] = lb;
      }
    }
    __syncthreads();
    const int nnz = s_cnt;
    if (threadIdx.x == 0) row_nnz[i] = nnz;
    const long long k2 = kSymInstr ? clock64() : 0;
    if (want_parts && nnz > kPartMinKeys) {
      // parts: greedy runs of consecutive tiles holding <= kTPartKeys keys; a
      // tile holding more stands alone (dense window in the numeric phase).
      // Runs start at nonempty tiles only.  With the tile prefix P = s_tile:
      //   u(t)   = end of the greedy run starting at t = x - 1 for the first
      //            x >= t + 2 with P(x) > P(t) + kTPartKeys (else ntiles), so a
      //            run of >= 2 tiles never holds more than kTPartKeys keys;
      //   nne(t) = first nonempty tile >= t (first x > t with P(x) > P(t),
      //            minus one; ntiles if none).
      // One thread per tile, then the chain nne(0) -> nne(u(.)) -> ... (one
      // step per part).
      int *s_nxt = s_tcnt;  // (tile counts are consumed)
      for (int t = threadIdx.x; t <= ntiles; t += THREADS) {
        if (t == ntiles) { s_nne[t] = ntiles; continue; }
        const int lim = s_tile[t] + kTPartKeys;
        int lo = t + 2, hi = ntiles + 1;  // first x in [t + 2, ntiles] with P(x) > lim, else ntiles + 1
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (s_tile[m] > lim) hi = m; else lo = m + 1;
        }
        s_nxt[t] = min(lo - 1, ntiles);
        const int p0 = s_tile[t];
        lo = t + 1, hi = ntiles + 1;  // first x in [t + 1, ntiles] with P(x) > P(t)
        while (lo < hi) {
          const int m = (lo + hi) >> 1;
          if (s_tile[m] > p0) hi = m; else lo = m + 1;
        }
        s_nne[t] = lo - 1;  // (ntiles when no key at or after t)
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int np = 0;
        long long htiles = 0;  // tiles of the row's parts spanning <= kPbitsMaxSpan tiles
        for (int t = s_nne[0]; t < ntiles; t = s_nne[s_nxt[t]]) {
          s_prec[np] = (int)htiles;  // record tiles of the parts before this one
          s_cut[np++] = t | (s_nxt[t] << 16);
          if (rec_part(t, s_nxt[t])) htiles += s_nxt[t] - t;
        }
        // part slots from the block's pool (a refill leaves the rest of the
        // old chunk as holes, marked below by the whole block)
        s_hole_lo = s_hole_hi = 0;
        long long base = s_pp_cur;
        if (base + np > s_pp_end) {
          s_hole_lo = s_pp_cur;
          s_hole_hi = s_pp_end;
          const long long chunk = np > kPoolParts ? np : kPoolParts;
          base = (long long)atomicAdd(&info->parts_pool, (unsigned long long)chunk);
          s_pp_end = base + chunk;
          if (s_pp_end > parts_cap) s_pp_end = parts_cap;
        }
        if (base + np > parts_cap) {
          atomicAdd(&info->parts_overflow, 1ull);
          s_cnt = -1;
          s_pp_cur = s_pp_end;
        } else {
          s_pp_cur = base + np;
          s_cnt = np;
          atomicAdd(&info->parts_used, (unsigned long long)np);  // (exact count; result unused)
          // tile records of the hash parts (block pool, in records; without
          // room the parts keep -1 and the numeric hashes their keys)
          long long rbase = -1;
          if (htiles > 0) {
            atomicAdd(&info->pkeys_used, (unsigned long long)htiles);  // (the host sizes the buffer from it)
            if (pbits != nullptr) {
              rbase = s_rp_cur;
              if (rbase + htiles > s_rp_end) {
                const long long chunk = htiles > kPoolRecs ? htiles : kPoolRecs;
                rbase = (long long)atomicAdd(&info->pkeys_pool, (unsigned long long)chunk);
                s_rp_end = rbase + chunk;
              }
              if ((rbase + htiles) * kTileRec > pbits_cap) {
                rbase = -1;
                s_rp_cur = s_rp_end;
              } else {
                s_rp_cur = rbase + htiles;
              }
            }
          }
          s_rbase = rbase;
          s_pbase = base;
        }
      }
      __syncthreads();
      const int np = s_cnt;
      for (long long h = s_hole_lo + threadIdx.x; h < s_hole_hi; h += THREADS)
        parts[3 * h] = make_int4(-1, 0, 0, 0);  // (hole: skipped by the parts bucket sort)
      const long long rbase = s_rbase;
      for (int p = threadIdx.x; p < np; p += THREADS) {  // (a thread per part)
        const int t0 = s_cut[p] & 0xFFFF, t1 = s_cut[p] >> 16;
        const bool dpt = t1 == t0 + 1 && !rec_part(t0, t1) && dpfx != nullptr;
        if (dpt) s_dpart[t0] = (int)(s_pbase + p);
        long long koff = -1;
        if (rec_part(t0, t1) && rbase >= 0) {
          koff = rbase + s_prec[p];
          for (int t = t0; t < t1; ++t) {  // (<= kPbitsMaxSpan tiles)
            s_tkoff[t] = koff + (t - t0);
            s_tkb[t] = s_tile[t] - s_tile[t0];
          }
        }
        parts[3 * (s_pbase + p)] = make_int4(i, s_cut[p], s_tile[t0], s_tile[t1] - s_tile[t0]);
        parts[3 * (s_pbase + p) + 1] =
            make_int4((int)(unsigned)(unsigned long long)as, (int)(unsigned)((unsigned long long)as >> 32),
                      (int)(ae - as), 0);
        parts[3 * (s_pbase + p) + 2] =
            make_int4((int)(unsigned)(unsigned long long)koff, (int)(unsigned)((unsigned long long)koff >> 32),
                      dpt ? (int)(s_pbase + p) : -1, 0);
      }
    }
    __syncthreads();
    const long long k3 = kSymInstr ? clock64() : 0;
    // tile records of the hash parts (a warp per tile: lane l stores words
    // 8 l .. 8 l + 7 and their ranks -- keys of the part before each word --
    // as two 16-byte stores, coalesced), and the clear of every word for the
    // next row
    for (int t = w; t < ntiles; t += NW) {
      const int q0 = t << (kTileLog - 5), q1 = min(nwords, q0 + kTileCols / 32);
      const long long rec = s_tkoff[t];
      if (rec >= 0) {
        const int qa = q0 + 8 * lane;
        uint32_t wv[8];
        int c = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          wv[u] = bm[bm_phys(qa + u)];
          c += __popc(wv[u]);
        }
        const int incl = warp_incl_scan(c);
        int run = s_tkb[t] + incl - c;
        uint32_t rk[4];
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          const int r0 = run;
          run += __popc(wv[u]);
          rk[u >> 1] = (uint32_t)r0 | ((uint32_t)run << 16);
          run += __popc(wv[u + 1]);
        }
        uint32_t *rp = pbits + rec * kTileRec;
        // (evict-first: read once, by the numeric phase)
        __stcs(reinterpret_cast<uint4 *>(rp) + 2 * lane, make_uint4(wv[0], wv[1], wv[2], wv[3]));
        __stcs(reinterpret_cast<uint4 *>(rp) + 2 * lane + 1, make_uint4(wv[4], wv[5], wv[6], wv[7]));
        __stcs(reinterpret_cast<uint4 *>(rp + 256) + lane, make_uint4(rk[0], rk[1], rk[2], rk[3]));
      }
      // dense single-tile part: keys of the tile before each 512-column
      // stripe (the numeric's warp w emits stripe w: no count pass there)
      const int dp = s_dpart[t];
      if (dp >= 0) {
        const int qa = q0 + 8 * lane;  // lane: half a stripe (8 words)
        int c = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) c += __popc(bm[bm_phys(qa + u)]);
        const int ex = warp_incl_scan(c) - c;
        if ((lane & 1) == 0) dpfx[int64_t(dp) * kDenseStripes + (lane >> 1)] = (uint16_t)ex;
      }
      // the row's sorted column list: lane l writes the columns of the
      // tile's words 8 l .. 8 l + 7 in order
      if (s_lbase >= 0 && s_tile[t + 1] > s_tile[t]) {
        const int qa = q0 + 8 * lane;
        uint32_t wv[8];
        int c = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          wv[u] = bm[bm_phys(qa + u)];
          c += __popc(wv[u]);
        }
        int32_t *dst = lists + s_lbase + s_tile[t] + warp_incl_scan(c) - c;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          uint32_t wd = wv[u];
          const int32_t cb = (int32_t)(qa + u) << 5;
          while (wd) {
            *dst++ = cb + __ffs(wd) - 1;
            wd &= wd - 1;
          }
        }
      }
      for (int q = q0 + lane; q < q1; q += 32) bm[q] = 0u;
    }
    __syncthreads();
    if (kSymInstr && threadIdx.x == 0) {  // (phase clocks: SPG_SYM_INSTR builds)
      const long long k4 = clock64();
      atomicAdd(&info->dbg[0], 1ull);
      atomicAdd(&info->dbg[1], (unsigned long long)(k1 - k0));  // walk (staging + rounds)
      atomicAdd(&info->dbg[2], (unsigned long long)(k2 - k1));  // tile counts + scan
      atomicAdd(&info->dbg[3], (unsigned long long)(k3 - k2));  // parts
      atomicAdd(&info->dbg[4], (unsigned long long)(k4 - k3));  // records, stripes, clear
      atomicAdd(&info->dbg[5], (unsigned long long)(ae - as));
    }
  }
  // the rest of the block's last parts chunk: holes
  if (parts != nullptr)
    for (long long h = s_pp_cur + threadIdx.x; h < s_pp_end; h += THREADS) parts[3 * h] = make_int4(-1, 0, 0, 0);
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
  __shared__ int s_cnt, s_next;
  __shared__ DeferList s_dl;  // long B rows walked by the whole block
  constexpr int NW = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *tab = slab + int64_t(blockIdx.x) * slabT;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int i = rows[r];
    const int logT = sym_log2_gpu(flop[i], B.ncols);
    const int64_t T = int64_t(1) << logT;
    for (int64_t s = threadIdx.x; s < T; s += THREADS) tab[s] = kEmpty;
    if (threadIdx.x == 0) { s_cnt = 0; s_next = 0; }
    __syncthreads();
    int cnt = 0;
    {
      const int64_t as = A.rp[i], ae = A.rp[i + 1];
      auto ins = [&](bool act, uint32_t c, double) {
        if (act) cnt += sym_insert(tab, c, logT);
      };
      if (use_seq(flop[i], ae - as)) for_row<true, false, 8, true>(A, B, as, ae, w, NW, ins, &s_next, &s_dl);
      else for_row<false, false>(A, B, as, ae, w, NW, ins, &s_next, &s_dl);
    }
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&s_cnt, cnt);
    __syncthreads();
    if (threadIdx.x == 0) row_nnz[i] = s_cnt;
  }
}

}  // namespace spg
