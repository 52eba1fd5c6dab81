// spgemm.cu -- C ABI (include/spgemm.h) of the sm_100a hash SpGEMM hot path.
// Host orchestration only: every step of the path runs in the kernels of
// plan.cuh / symbolic.cuh / numeric.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "masked.cuh"
#include "numeric.cuh"
#include "plan.cuh"
#include "probestats.cuh"
#include "relabel.cuh"
#include "spg_internal.cuh"
#include "symbolic.cuh"

using namespace spg;

namespace {

constexpr int kSubStreams = 4;
constexpr int kWarps = 8;  // warps per block of the W tier

struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct spg_ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 0;
  spg_alloc_fn alloc = nullptr;
  spg_free_fn free_fn = nullptr;
  void *user = nullptr;
  std::string err;
  Buf flop, rows_sym, rows_num, partial, slab, info, scratch;
  Buf parts, parts2, part_hist, toff, pkeys, dpfx;
  Buf lists, list_off;    // sorted column lists of the block-tier rows (from the bitmap symbolic)
  size_t lists_want = 0;  // (grown at the start of the next symbolic)
  bool plan_lists = false;  // (+ tile records of the narrow hash parts)
  size_t pkeys_want = 0;  // column-tile parts of long rows (BM tier), sorted copy, B tile offsets
  Buf bnz, prune_cnt, prune_rp, prune_col, prune_val, prune_idx;  // B nonempty-row bitmap; pruned A
  Buf trow;                          // row of the first a_ik of every kFlopTile tile of A
  Buf rl_key, rl_rank, rl_tmp, rl_cub;  // degree relabelling (histograms, ranks/buckets, unsorted rows)
  Buf mask_rows;                     // row lists of the mask-and-sum tiers
  Buf useful_bits;                   // useful-entry bitmask of k_flop_nz (pruning), grow-only
  Buf one_fofs, one_col, one_val;    // one-phase: flop prefix, flop-sized row workspace (grow-only)
  bool have_one = false;             // a one-phase result waits in the workspace
  bool one_graph_ok = true;          // SPG_ONEPHASE_GRAPH=0: no graph capture
  cudaGraphExec_t one_exec = nullptr;
  int64_t one_graph_launches = 0;
  int64_t one_m = 0;
  const int64_t *one_rp = nullptr;
  struct OneKeyT {
    const void *arp, *acol, *aval;
    int64_t am, an;
    const void *brp, *bcol, *bval;
    int64_t bm, bn;
    const void *crp;
    int sorted;
    const void *ws;
    unsigned long long cap;
    bool operator==(const OneKeyT &o) const {
      return arp == o.arp && acol == o.acol && aval == o.aval && am == o.am && an == o.an &&
             brp == o.brp && bcol == o.bcol && bval == o.bval && bm == o.bm && bn == o.bn &&
             crp == o.crp && sorted == o.sorted && ws == o.ws && cap == o.cap;
    }
  } one_key{};
  bool pruned = false;               // the plan runs on the pruned A' (mostly-empty B)
  int64_t prune_n = 0;
  spg_csr Ap{};
  bool plan_parts = false;           // parts were produced for the numeric G tier
  PlanInfo *host_info = nullptr;  // pinned
  cudaStream_t sub[kSubStreams] = {};
  cudaEvent_t ev_fork = nullptr;
  cudaEvent_t ev_join[kSubStreams] = {};
  int64_t launches = 0;
  int serial = 0;  // SPG_SERIAL_BINS=1: all bins on the caller's stream (diagnosis)
  int tune = 0;    // SPG_TUNE=<bits>: kernel variant switches for A/B measurements (default 0)
  int accum = ACC_AUTO;   // accumulator choice for sorted output (spg_set_accumulator)
  float cfac = 1.3f;      // collision factor c of Eq:hash_est (measured)
  float hfac = 8.0f;      // heap step cost / hash probe cost on B200 (measured)
  // optional per-launch timing (events on the stream each kernel runs on)
  int profiling = 0;
  struct Rec { const char *name; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // plan of the last symbolic
  bool have_plan = false;
  const int64_t *plan_a_rp = nullptr, *plan_b_rp = nullptr, *plan_c_rp = nullptr;
  const int32_t *plan_a_col = nullptr, *plan_b_col = nullptr;
  int64_t plan_m = 0, plan_ncols = 0;
  PlanInfo plan{};
};

namespace {

spg_status fail(spg_ctx *c, spg_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

spg_status cuda_check(spg_ctx *c, cudaError_t e, const char *where) {
  if (e == cudaSuccess) return SPG_OK;
  return fail(c, SPG_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

cudaEvent_t prof_event(spg_ctx *c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

// Brackets one launch with events when profiling is on.
struct ProfScope {
  spg_ctx *c;
  cudaStream_t s;
  const char *name;
  cudaEvent_t a = nullptr;
  ProfScope(spg_ctx *c_, cudaStream_t s_, const char *n) : c(c_), s(s_), name(n) {
    if (c->profiling && (a = prof_event(c))) cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = prof_event(c);
    if (!b) return;
    cudaEventRecord(b, s);
    c->recs.push_back({name, a, b});
  }
};

#define SPG_CUDA(ctx, expr)                                  \
  do {                                                       \
    spg_status _s = cuda_check((ctx), (expr), #expr);        \
    if (_s != SPG_OK) return _s;                             \
  } while (0)

#define SPG_LAUNCHED(ctx, name)                                                   \
  do {                                                                            \
    (ctx)->launches++;                                                            \
    spg_status _s = cuda_check((ctx), cudaGetLastError(), "launch " name);        \
    if (_s != SPG_OK) return _s;                                                  \
  } while (0)

void buf_release(spg_ctx *c, Buf &b, cudaStream_t s) {
  if (!b.p) return;
  if (c->free_fn) c->free_fn(b.p, s, c->user);
  else cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
}

spg_status buf_ensure(spg_ctx *c, Buf &b, size_t bytes, cudaStream_t s) {
  if (bytes <= b.bytes && b.p) return SPG_OK;
  buf_release(c, b, s);
  size_t want = std::max(bytes, size_t(256));
  void *p = nullptr;
  if (c->alloc) {
    p = c->alloc(want, s, c->user);
  } else if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  if (!p) return fail(c, SPG_ERR_WORKSPACE, "workspace allocation of " + std::to_string(want) + " bytes failed");
  b.p = p;
  b.bytes = want;
  return SPG_OK;
}

DevCSR dev(const spg_csr *M) { return DevCSR{M->nrows, M->ncols, M->row_ptr, M->col_idx, M->val}; }

spg_status check_csr(spg_ctx *c, const spg_csr *M, const char *name, bool need_val) {
  if (!M) return fail(c, SPG_ERR_INVALID_ARG, std::string(name) + " is NULL");
  if (M->nrows < 0 || M->ncols < 0)
    return fail(c, SPG_ERR_INVALID_ARG, std::string(name) + " has negative dimensions");
  if (M->nrows > INT32_MAX - 1 || M->ncols > INT32_MAX)
    return fail(c, SPG_ERR_OVERFLOW, std::string(name) + ": dimensions above 2^31-1");
  if (!M->row_ptr) return fail(c, SPG_ERR_INVALID_ARG, std::string(name) + ".row_ptr is NULL");
  if (need_val && !M->val) return fail(c, SPG_ERR_INVALID_ARG, std::string(name) + ".val is NULL");
  return SPG_OK;
}

// Fork `n` internal streams off `s`; kernels of different bins run concurrently.
spg_status fork(spg_ctx *c, cudaStream_t s) {
  SPG_CUDA(c, cudaEventRecord(c->ev_fork, s));
  for (int k = 0; k < kSubStreams; ++k) SPG_CUDA(c, cudaStreamWaitEvent(c->sub[k], c->ev_fork, 0));
  return SPG_OK;
}

spg_status join(spg_ctx *c, cudaStream_t s) {
  for (int k = 0; k < kSubStreams; ++k) {
    SPG_CUDA(c, cudaEventRecord(c->ev_join[k], c->sub[k]));
    SPG_CUDA(c, cudaStreamWaitEvent(s, c->ev_join[k], 0));
  }
  return SPG_OK;
}

template <typename K>
spg_status set_smem(spg_ctx *c, K kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    SPG_CUDA(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return SPG_OK;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// a1 (+ a2 counts): per-row flop, nonzero-parallel (balanced whatever the row
// lengths), then a per-row pass for bins / totals.
spg_status launch_flop(spg_ctx *c, const spg_csr *A, const spg_csr *B, int count_bins,
                       cudaStream_t s, const uint32_t *bnz = nullptr,
                       unsigned long long *useful_row = nullptr) {
  const int64_t m = A->nrows;
  if (m == 0) return SPG_OK;
  PlanInfo *info = (PlanInfo *)c->info.p;
  int64_t *flop = (int64_t *)c->flop.p;
  DevCSR a = dev(A);
  SPG_CUDA(c, cudaMemsetAsync(flop, 0, size_t(m) * 8, s));
  // tile-row index of A for the nonzero-parallel kernels (capacity m + 1
  // tiles -- nnz(A) is not known on the host; tiles beyond it search)
  spg_status st0;
  if ((st0 = buf_ensure(c, c->trow, size_t(m + 1) * 8, s)) != SPG_OK) return st0;
  {
    ProfScope _ps(c, s, "k_tile_rows");
    k_tile_rows<<<(unsigned)std::min<int64_t>(ceil_div(m + 1, 256), int64_t(c->num_sms) * 8), 256, 0, s>>>(
        a, m, (int64_t *)c->trow.p);
  }
  SPG_LAUNCHED(c, "k_tile_rows");
  {
    ProfScope _ps(c, s, "k_flop_nz");
    // the useful-entry bitmask is written when a previous call sized it (its
    // capacity covers this A: checked again before the pruning scatter uses it)
    uint32_t *bits = useful_row && c->useful_bits.p ? (uint32_t *)c->useful_bits.p : nullptr;
    k_flop_nz<<<(unsigned)(c->num_sms * 8), kFlopThreads, 0, s>>>(
        a, B->row_ptr, B->nrows, bnz, (unsigned long long *)flop, info, useful_row,
        (const int64_t *)c->trow.p, m, bits, bits ? int64_t(c->useful_bits.bytes / 4) : 0);
  }
  SPG_LAUNCHED(c, "k_flop_nz");
  {
    ProfScope _ps(c, s, "k_flop_stats");
    const int64_t grid = std::min<int64_t>(ceil_div(m, 256), int64_t(c->num_sms) * 8);
    k_flop_stats<<<(unsigned)grid, 256, 0, s>>>(a, B->ncols, flop, info, count_bins);
  }
  SPG_LAUNCHED(c, "k_flop_stats");
  return SPG_OK;
}

// scan of data[0..n) in place (int64), numeric-bin counting in the last pass
spg_status launch_scan(spg_ctx *c, int64_t *data, int64_t n, cudaStream_t s,
                       const int64_t *arp = nullptr, const int64_t *flop = nullptr) {
  if (n == 0) return SPG_OK;
  const int64_t nb = ceil_div(n, kScanTile);
  SPG_CUDA(c, cudaGetLastError());
  spg_status st = buf_ensure(c, c->partial, size_t(nb) * 8, s);
  if (st != SPG_OK) return st;
  int64_t *partial = (int64_t *)c->partial.p;
  {
    ProfScope _ps(c, s, "k_scan_reduce");
    k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, s>>>(data, n, partial);
  }
  SPG_LAUNCHED(c, "k_scan_reduce");
  {
    ProfScope _ps(c, s, "k_scan_partials");
    k_scan_partials<<<1, kScanThreads, 0, s>>>(partial, nb);
  }
  SPG_LAUNCHED(c, "k_scan_partials");
  {
    ProfScope _ps(c, s, "k_scan_down");
    k_scan_down<<<(unsigned)nb, kScanThreads, 0, s>>>(data, n, partial, (PlanInfo *)c->info.p, arp,
                                                      flop, c->accum, c->cfac, c->hfac);
  }
  SPG_LAUNCHED(c, "k_scan_down");
  return SPG_OK;
}

spg_status read_info(spg_ctx *c, cudaStream_t s) {
  SPG_CUDA(c, cudaMemcpyAsync(c->host_info, c->info.p, sizeof(PlanInfo), cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  return SPG_OK;
}

// Workspace budget of the global-hash slabs: a quarter of the free device
// memory (plus what the slab buffer already holds), at most 16 GiB.
int64_t slab_budget(spg_ctx *c) {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    free_b = size_t(1) << 32;
  }
  const int64_t b = int64_t(free_b / 4 + c->slab.bytes);
  return std::min<int64_t>(b, int64_t(16) << 30);
}

int64_t bin_offset(const unsigned long long *cnt, int b) {
  int64_t off = 0;
  for (int u = 1; u < b; ++u) off += (int64_t)cnt[u];
  return off;
}


}  // namespace

// paper's symbolic table size per row (debug export; Fig:hash_spgemm P:302-305)
__global__ void k_plan_tsize(const int64_t *f, int64_t m, int64_t ncols, int64_t *o) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) o[i] = int64_t(1) << sym_log2_paper(f[i], ncols);
}

// ============================================================================
extern "C" {

spg_status spg_ctx_create(spg_ctx **out, spg_alloc_fn alloc, spg_free_fn free_fn, void *user) {
  if (!out) return SPG_ERR_INVALID_ARG;
  *out = nullptr;
  if ((alloc == nullptr) != (free_fn == nullptr)) return SPG_ERR_INVALID_ARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return SPG_ERR_CUDA; }
  spg_ctx *c = new spg_ctx();
  c->device = dev;
  c->alloc = alloc;
  c->free_fn = free_fn;
  c->user = user;
  {
    const char *e = getenv("SPG_SERIAL_BINS");
    c->serial = (e && e[0] == '1') ? 1 : 0;
    const char *t = getenv("SPG_TUNE");
    c->tune = t ? atoi(t) : 0;
    const char *og = getenv("SPG_ONEPHASE_GRAPH");
    c->one_graph_ok = !(og && og[0] == '0');
  }
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess) c->num_sms = v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) == cudaSuccess)
    c->smem_optin = (size_t)v;
  bool ok = cudaMallocHost(&c->host_info, sizeof(PlanInfo)) == cudaSuccess;
  for (int k = 0; ok && k < kSubStreams; ++k) {
    ok = cudaStreamCreateWithFlags(&c->sub[k], cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess;
  if (ok) {
    const size_t s_num_w1024 = 4 * 1024 * 16;
    const size_t s_num_b = size_t(16384) * 12;
    ok = set_smem(c, k_num_warp<1024, 4, 0>, s_num_w1024) == SPG_OK &&
         set_smem(c, k_num_warp<1024, 4, 1>, s_num_w1024) == SPG_OK &&
         set_smem(c, k_num_block<128>, size_t(2048) * 12) == SPG_OK &&
         set_smem(c, k_num_block<512>, s_num_b) == SPG_OK &&
         set_smem(c, k_num_block<1024>, s_num_b) == SPG_OK &&
         set_smem(c, k_sym_block<512>, size_t(32768) * 4) == SPG_OK &&
         set_smem(c, k_sym_block<128>, size_t(4096) * 4) == SPG_OK &&
         set_smem(c, k_sym_block<256>, size_t(8192) * 4) == SPG_OK &&
         set_smem(c, k_sym_block<1024>, size_t(32768) * 4) == SPG_OK &&
         set_smem(c, k_sym_bitmap<1024>, size_t(kBitmapMaxCols / 8) + kBmStageBytes) == SPG_OK &&
         set_smem(c, k_num_tpart<512>, kTPartSmem) == SPG_OK &&
         set_smem(c, k_mask_sum_block<1024>, size_t(kBitmapMaxCols / 8)) == SPG_OK &&
         set_smem(c, k_csr_mask_sum_block<1024>, size_t(kBitmapMaxCols / 8)) == SPG_OK &&
         set_smem(c, k_num_global<1024>, kRankSmem) == SPG_OK &&
         set_smem(c, k_num_heap<kHeapThreads>, kHeapSmem) == SPG_OK &&
         set_smem(c, k_num_warp<1024, 4, 0, true>, s_num_w1024) == SPG_OK &&
         set_smem(c, k_num_warp<1024, 4, 1, true>, s_num_w1024) == SPG_OK &&
         set_smem(c, k_num_block<128, true>, size_t(2048) * 12) == SPG_OK &&
         set_smem(c, k_num_block<512, true>, size_t(8192) * 12) == SPG_OK &&
         set_smem(c, k_num_block<1024, true>, size_t(16384) * 12) == SPG_OK &&
         set_smem(c, k_segsort_long<1024>, size_t(kBitmapMaxCols / 8)) == SPG_OK;
  }
  if (!ok) {
    cudaGetLastError();
    spg_ctx_destroy(c);
    return SPG_ERR_CUDA;
  }
  *out = c;
  return SPG_OK;
}

spg_status spg_ctx_destroy(spg_ctx *c) {
  if (!c) return SPG_ERR_INVALID_ARG;
  cudaDeviceSynchronize();
  Buf *bufs[] = {&c->flop,      &c->rows_sym,  &c->rows_num,  &c->partial,   &c->slab,
                 &c->info,      &c->scratch,   &c->parts,     &c->parts2,    &c->part_hist, &c->pkeys,
                 &c->toff,      &c->bnz,       &c->prune_cnt, &c->prune_rp,  &c->prune_col,
                 &c->prune_val, &c->prune_idx, &c->trow,      &c->rl_key,    &c->rl_rank,
                 &c->rl_tmp,    &c->rl_cub,    &c->mask_rows, &c->useful_bits, &c->one_fofs,
                 &c->one_col,   &c->one_val,   &c->dpfx,      &c->lists,     &c->list_off};
  for (Buf *b : bufs) buf_release(c, *b, nullptr);
  if (c->host_info) cudaFreeHost(c->host_info);
  for (int k = 0; k < kSubStreams; ++k) {
    if (c->sub[k]) cudaStreamDestroy(c->sub[k]);
    if (c->ev_join[k]) cudaEventDestroy(c->ev_join[k]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->one_exec) cudaGraphExecDestroy(c->one_exec);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
  return SPG_OK;
}

const char *spg_last_error(const spg_ctx *c) { return c ? c->err.c_str() : "null ctx"; }

int64_t spg_launch_count(const spg_ctx *c) { return c ? c->launches : -1; }

spg_status spg_profile_enable(spg_ctx *c, int enable) {
  if (!c) return SPG_ERR_INVALID_ARG;
  c->profiling = enable ? 1 : 0;
  return SPG_OK;
}

spg_status spg_set_serial_bins(spg_ctx *c, int on) {
  if (!c) return SPG_ERR_INVALID_ARG;
  c->serial = on ? 1 : 0;
  return SPG_OK;
}

spg_status spg_profile_reset(spg_ctx *c) {
  if (!c) return SPG_ERR_INVALID_ARG;
  for (auto &r : c->recs) cudaEventSynchronize(r.b);
  c->recs.clear();
  c->ev_used = 0;
  return SPG_OK;
}

int64_t spg_profile_count(spg_ctx *c) {
  if (!c) return -1;
  for (auto &r : c->recs) cudaEventSynchronize(r.b);
  return (int64_t)c->recs.size();
}

spg_status spg_profile_record(spg_ctx *c, int64_t idx, const char **name, float *ms) {
  if (!c || !name || !ms || idx < 0 || idx >= (int64_t)c->recs.size()) return SPG_ERR_INVALID_ARG;
  const auto &r = c->recs[(size_t)idx];
  SPG_CUDA(c, cudaEventSynchronize(r.b));
  SPG_CUDA(c, cudaEventElapsedTime(ms, r.a, r.b));
  *name = r.name;
  return SPG_OK;
}

spg_status spg_get_info(const spg_ctx *c, spg_info *o) {
  if (!c || !o) return SPG_ERR_INVALID_ARG;
  if (!c->have_plan) return SPG_ERR_STATE;
  std::memset(o, 0, sizeof(*o));
  const PlanInfo &p = c->plan;
  o->nrows = c->plan_m;
  o->flop_total = (int64_t)p.flop_total;
  o->nnz_total = (int64_t)p.nnz_total;
  o->max_row_flop = (int64_t)p.max_flop;
  o->max_row_nnz = (int64_t)p.max_nnz;
  for (int b = 0; b < 12 && b < kMaxBins; ++b) {
    o->sym_bin_rows[b] = (int64_t)p.sym_count[b];
    o->num_bin_rows[b] = (int64_t)p.num_count[b];
  }
  o->heap_rows = (int64_t)(p.heap_count[NB_W256] + p.heap_count[NB_W1024]);
  o->sym_bin_rows[0] = c->plan_m;  // skip bin = the rest
  o->num_bin_rows[0] = c->plan_m;
  for (int b = 1; b < kMaxBins; ++b) {
    o->sym_bin_rows[0] -= o->sym_bin_rows[b];
    o->num_bin_rows[0] -= o->num_bin_rows[b];
  }
  return SPG_OK;
}

spg_status spg_symbolic(spg_ctx *c, const spg_csr *A, const spg_csr *B, int64_t *C_row_ptr,
                        int64_t *nnz_C, int64_t *flop_total, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  c->have_plan = false;
  c->plan_parts = false;
  spg_status st;
  if ((st = check_csr(c, A, "A", false)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows)
    return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows (" + std::to_string(A->ncols) + " vs " +
                                             std::to_string(B->nrows) + ")");
  if (!C_row_ptr || !nnz_C) return fail(c, SPG_ERR_INVALID_ARG, "C_row_ptr / nnz_C is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  const int64_t m = A->nrows;
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->flop, size_t(std::max<int64_t>(m, 1)) * 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->rows_sym, size_t(std::max<int64_t>(m, 1)) * 4, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->rows_num, size_t(std::max<int64_t>(m, 1)) * 4, s)) != SPG_OK) return st;
  if (c->pkeys_want > c->pkeys.bytes) {  // (grown here only: see the end of spg_symbolic)
    size_t free_b = 0, total_b = 0;
    // (the records must leave room for C: at most a quarter of the device,
    // and 8 GiB of what is free right now)
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && c->pkeys_want <= total_b / 4 &&
        c->pkeys_want + (size_t(8) << 30) < free_b + c->pkeys.bytes)
      buf_ensure(c, c->pkeys, c->pkeys_want, s);
    cudaGetLastError();
    c->pkeys_want = 0;
  }
  if (c->lists_want > c->lists.bytes) {  // (grown here only, like the tile records)
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && c->lists_want <= total_b / 8 &&
        c->lists_want + (size_t(8) << 30) < free_b + c->lists.bytes)
      buf_ensure(c, c->lists, c->lists_want, s);
    cudaGetLastError();
    c->lists_want = 0;
  }
  c->plan_lists = false;
  PlanInfo *info = (PlanInfo *)c->info.p;
  SPG_CUDA(c, cudaMemsetAsync(info, 0, sizeof(PlanInfo), s));
  SPG_CUDA(c, cudaMemsetAsync(C_row_ptr, 0, sizeof(int64_t), s));
  if (B->nrows > 0)
    SPG_CUDA(c, cudaMemcpyAsync(&info->b_end, B->row_ptr + B->nrows, 8, cudaMemcpyDeviceToDevice, s));
  int64_t *row_nnz = C_row_ptr + 1;
  int64_t *flop = (int64_t *)c->flop.p;
  c->pruned = false;
  const spg_csr *A0 = A;  // the caller's A (the plan is keyed on it)
  if (m > 0 && B->nrows > 0) {
    // B nonempty-row bitmap: k_flop_nz skips the B.rp gathers of empty rows
    // when most rows are empty (decided on the device)
    const uint32_t *bnz = nullptr;
    {
      const int64_t nw = (B->nrows + 31) / 32;
      if ((st = buf_ensure(c, c->bnz, size_t(nw) * 4, s)) != SPG_OK) return st;
      ProfScope _ps(c, s, "k_b_rowmask");
      k_b_rowmask<<<(unsigned)std::min<int64_t>(ceil_div(nw * 32, 256), int64_t(c->num_sms) * 8), 256, 0, s>>>(
          dev(B), (uint32_t *)c->bnz.p, info);
      bnz = (const uint32_t *)c->bnz.p;
    }
    SPG_LAUNCHED(c, "k_b_rowmask");
    // are B's rows strictly increasing?  (column-tile parts and the heap tier
    // need it; decided on the device, also visible at the first host read)
    {
      ProfScope _ps(c, s, "k_check_sorted");
      const int64_t gridc = std::min<int64_t>(ceil_div(std::max<int64_t>(B->nrows, 1), 256),
                                              int64_t(c->num_sms) * 8);
      k_check_sorted<<<(unsigned)std::max<int64_t>(gridc, 1), 256, 0, s>>>(dev(B), info);
    }
    SPG_LAUNCHED(c, "k_check_sorted");
    // a1 + a2: flop, symbolic bins (+ per-row useful a_ik counts when most B
    // rows are empty, for the pruning below)
    if ((st = buf_ensure(c, c->prune_cnt, size_t(m) * 8, s)) != SPG_OK) return st;
    SPG_CUDA(c, cudaMemsetAsync(c->prune_cnt.p, 0, size_t(m) * 8, s));
    if ((st = launch_flop(c, A, B, 1, s, bnz, (unsigned long long *)c->prune_cnt.p)) != SPG_OK)
      return st;
    {
      ProfScope _ps(c, s, "k_bin_scatter_sym");
      k_bin_scatter<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(m, flop, A->row_ptr, B->ncols, 0, info,
                                                               (int32_t *)c->rows_sym.p, row_nnz);
    }
    SPG_LAUNCHED(c, "k_bin_scatter(sym)");
    if ((st = read_info(c, s)) != SPG_OK) return st;
    PlanInfo h = *c->host_info;
    if (2 * (int64_t)h.b_empty > B->nrows && 4 * (int64_t)h.useful < (int64_t)h.a_nnz &&
        h.a_nnz >= (1ull << 20)) {
      // most a_ik hit empty B rows: run the plan on A' = the useful a_ik of A
      // (same rows, same flop; the walks of the symbolic / numeric tiers no
      // longer visit the dead entries)
      const int64_t nu = (int64_t)h.useful;
      if ((st = buf_ensure(c, c->prune_rp, size_t(m + 1) * 8, s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->prune_col, size_t(std::max<int64_t>(nu, 1)) * 4, s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->prune_val, size_t(std::max<int64_t>(nu, 1)) * 8, s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->prune_idx, size_t(std::max<int64_t>(nu, 1)) * 8, s)) != SPG_OK) return st;
      int64_t *cnt = (int64_t *)c->prune_cnt.p, *rp2 = (int64_t *)c->prune_rp.p;
      DevCSR a = dev(A);
      SPG_CUDA(c, cudaMemsetAsync(rp2, 0, 8, s));
      SPG_CUDA(c, cudaMemcpyAsync(rp2 + 1, cnt, size_t(m) * 8, cudaMemcpyDeviceToDevice, s));
      if ((st = launch_scan(c, rp2 + 1, m, s)) != SPG_OK) return st;
      SPG_CUDA(c, cudaMemsetAsync(cnt, 0, size_t(m) * 8, s));
      const int64_t nwords = ceil_div((int64_t)h.a_nnz, kFlopTile) * (kFlopTile / 32);
      if (c->useful_bits.p && int64_t(c->useful_bits.bytes / 4) >= nwords) {
        // k_flop_nz wrote the useful-entry bitmask of this A: visit only those
        ProfScope _ps(c, s, "k_prune_scatter_bits");
        k_prune_scatter_bits<<<(unsigned)std::min<int64_t>(ceil_div(nwords, 256), c->num_sms * 8),
                               256, 0, s>>>(a, (const uint32_t *)c->useful_bits.p, nwords,
                                            (unsigned long long *)cnt, rp2,
                                            (int32_t *)c->prune_col.p, (int64_t *)c->prune_idx.p,
                                            (const int64_t *)c->trow.p, m);
        SPG_LAUNCHED(c, "k_prune_scatter_bits");
      } else {
        {
          ProfScope _ps(c, s, "k_prune_scatter");
          k_prune_scatter<<<(unsigned)(c->num_sms * 8), kFlopThreads, 0, s>>>(
              a, bnz, (unsigned long long *)cnt, rp2, (int32_t *)c->prune_col.p,
              (int64_t *)c->prune_idx.p, (const int64_t *)c->trow.p, m);
        }
        SPG_LAUNCHED(c, "k_prune_scatter");
        // size the bitmask for the next multiply (grow-only workspace)
        if ((st = buf_ensure(c, c->useful_bits, size_t(nwords) * 4, s)) != SPG_OK) return st;
      }
      c->prune_n = nu;
      c->Ap = spg_csr{m, A->ncols, rp2, (const int32_t *)c->prune_col.p,
                      (const double *)c->prune_val.p};
      c->pruned = true;
      A = &c->Ap;
      // re-bin on A': flop per row is unchanged (no flop pass again), the bins
      // also depend on |a_i|; keep the first pass's B facts, reset the rest
      {
        PlanInfo h2{};
        h2.max_brow = h.max_brow;
        h2.b_end = h.b_end;
        h2.b_empty = h.b_empty;
        h2.useful = h.useful;
        h2.b_unsorted = h.b_unsorted;
        h2.a_nnz = (unsigned long long)nu;
        *c->host_info = h2;  // (pinned; consumed by the copy before the next read_info)
        SPG_CUDA(c, cudaMemcpyAsync(info, c->host_info, sizeof(PlanInfo), cudaMemcpyHostToDevice, s));
      }
      {
        ProfScope _ps(c, s, "k_flop_stats");
        const int64_t grid = std::min<int64_t>(ceil_div(m, 256), int64_t(c->num_sms) * 8);
        k_flop_stats<<<(unsigned)grid, 256, 0, s>>>(dev(A), B->ncols, flop, info, 1);
      }
      SPG_LAUNCHED(c, "k_flop_stats");
      {
        ProfScope _ps(c, s, "k_bin_scatter_sym");
        k_bin_scatter<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(m, flop, A->row_ptr, B->ncols, 0, info,
                                                                 (int32_t *)c->rows_sym.p, row_nnz);
      }
      SPG_LAUNCHED(c, "k_bin_scatter(sym)");
      if ((st = read_info(c, s)) != SPG_OK) return st;
      h = *c->host_info;
    }
    if ((int64_t)h.max_brow > kMaxBRow)
      return fail(c, SPG_ERR_OVERFLOW, "a row of B has more than 2^26 entries");
    // BM tier: is B row-sorted (column-range parts need it)?  parts buffers
    c->plan_parts = false;
    int4 *parts = nullptr;
    int64_t parts_cap = 0;
    if (h.sym_count[SB_BM] && h.b_unsorted == 0) {
      // parts per row <= 2 nnz / kTPartKeys + 1 (consecutive parts hold > kTPartKeys keys)
      parts_cap = (int64_t)(2 * h.flop_total / kTPartKeys) + (int64_t)h.sym_count[SB_BM] + 16;
      const int64_t ntiles = (B->ncols + kTileCols - 1) / kTileCols;
      parts_cap = std::min<int64_t>(parts_cap, (int64_t)h.sym_count[SB_BM] * ntiles + 16);
      parts_cap += int64_t(c->num_sms) * 2 * kPoolParts;  // (per-block pools: at most one partial chunk per block)
      if ((st = buf_ensure(c, c->parts, size_t(parts_cap) * 3 * sizeof(int4), s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->dpfx, size_t(parts_cap) * kDenseStripes * 2, s)) != SPG_OK) return st;
      parts = (int4 *)c->parts.p;
      c->plan_parts = true;
    }
    // a3: symbolic per bin, bins on concurrent internal streams
    if ((st = fork(c, s)) != SPG_OK) return st;
    DevCSR a = dev(A), b = dev(B);
    const int32_t *rows = (const int32_t *)c->rows_sym.p;
    int sidx = 0;
    for (int bin = 1; bin < SB_COUNT; ++bin) {
      const int64_t n = (int64_t)h.sym_count[bin];
      if (n == 0) continue;
      const int32_t *rb = rows + bin_offset(h.sym_count, bin);
      cudaStream_t ss = c->serial ? s : c->sub[sidx++ % kSubStreams];
      if (bin == SB_W128 || bin == SB_W1024) {
        const int64_t grid = std::min<int64_t>(ceil_div(n, kWarps), int64_t(c->num_sms) * 32);
        // SPG_TUNE bit 128: HashVector-style warp-bucket probing (A/B)
        const bool bucket = (c->tune & 128) != 0;
        if (bin == SB_W128)
          {
            ProfScope _ps(c, ss, "k_sym_warp<128>");
            if (bucket)
              k_sym_warp<128, kWarps, true><<<(unsigned)grid, kWarps * 32, kWarps * 128 * 4, ss>>>(rb, n, a, b, flop, row_nnz);
            else
              k_sym_warp<128, kWarps><<<(unsigned)grid, kWarps * 32, kWarps * 128 * 4, ss>>>(rb, n, a, b, flop, row_nnz);
          }
        else
          {
            ProfScope _ps(c, ss, "k_sym_warp<1024>");
            if (bucket)
              k_sym_warp<1024, kWarps, true><<<(unsigned)grid, kWarps * 32, kWarps * 1024 * 4, ss>>>(rb, n, a, b, flop, row_nnz);
            else
              k_sym_warp<1024, kWarps><<<(unsigned)grid, kWarps * 32, kWarps * 1024 * 4, ss>>>(rb, n, a, b, flop, row_nnz);
          }
        SPG_LAUNCHED(c, "k_sym_warp");
      } else if (bin >= SB_B2K && bin <= SB_B32K) {
        const int logT = 11 + (bin - SB_B2K);
        const size_t smem = (size_t(1) << logT) * 4;
        const int64_t grid = std::min<int64_t>(n, int64_t(c->num_sms) * 8);
        if (logT <= 13)
          {
            // small blocks for small tables: a row's few rounds are split
            // over fewer warps, so less of the block idles at the row barrier
            // (measured: 2K/4K slots 128 threads, 8K slots 256)
            if (logT <= 12) {
              ProfScope _ps(c, ss, "k_sym_block<128>");
              k_sym_block<128><<<(unsigned)std::min<int64_t>(n, int64_t(c->num_sms) * 32), 128, smem, ss>>>(
                  rb, n, a, b, flop, row_nnz);
            } else {
              ProfScope _ps(c, ss, "k_sym_block<256>");
              k_sym_block<256><<<(unsigned)std::min<int64_t>(n, int64_t(c->num_sms) * 16), 256, smem, ss>>>(
                  rb, n, a, b, flop, row_nnz);
            }
          }
        else
          {
            ProfScope _ps(c, ss, "k_sym_block<1024>");
            k_sym_block<1024><<<(unsigned)grid, 1024, smem, ss>>>(rb, n, a, b, flop, row_nnz);
          }
        SPG_LAUNCHED(c, "k_sym_block");
      } else if (bin == SB_BM) {
        const size_t nwords = size_t(ceil_div(B->ncols, kTileCols)) * (kTileCols / 32);  // whole tiles (tbm_word)
        const int64_t grid = std::min<int64_t>(n, int64_t(c->num_sms) * 2);
        // sorted column lists for the rows the numeric block tier will take
        // (first call: a guess from the bin's row count; then the need).
        // Off by default (SPG_TUNE bit 65536 turns them on): measured on C3
        // the block tier gains what the bitmap symbolic loses
        if ((c->tune & 65536) && c->lists.bytes == 0) {
          size_t free_b = 0, total_b = 0;
          const size_t guess = size_t(n) * 2048 * 4;
          if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && guess <= total_b / 8 &&
              guess + (size_t(8) << 30) < free_b)
            buf_ensure(c, c->lists, guess, ss);
          cudaGetLastError();
        }
        if ((c->tune & 65536) && c->lists.bytes && buf_ensure(c, c->list_off, size_t(m) * 8, ss) == SPG_OK) {
          SPG_CUDA(c, cudaMemsetAsync(c->list_off.p, 0xFF, size_t(m) * 8, ss));
          c->plan_lists = true;
        }
        {
          ProfScope _ps(c, ss, "k_sym_bitmap<1024>");
          k_sym_bitmap<1024><<<(unsigned)grid, 1024, nwords * 4 + kBmStageBytes, ss>>>(
              rb, n, a, b, flop, row_nnz, info, parts, parts_cap,
              c->pkeys.p ? (uint32_t *)c->pkeys.p : nullptr, int64_t(c->pkeys.bytes / 4),
              parts ? (uint16_t *)c->dpfx.p : nullptr,
              c->plan_lists ? (int64_t *)c->list_off.p : nullptr,
              c->plan_lists ? (int32_t *)c->lists.p : nullptr, int64_t(c->lists.bytes / 4));
        }
        SPG_LAUNCHED(c, "k_sym_bitmap");
      } else {  // SB_G
        {
          int64_t grid = std::min<int64_t>(n, int64_t(c->num_sms) * 2);
          int lg = 0;
          {
            const int64_t mn = std::min<int64_t>((int64_t)h.max_flop, B->ncols);
            while ((int64_t(1) << lg) <= mn) ++lg;
          }
          const int64_t slabT = int64_t(1) << std::max(lg, kMinLogT);
          // one table per block, sized for the largest row: cap the grid so
          // the slabs fit the workspace budget (the kernel's row loop is
          // grid-strided, so fewer blocks only costs time)
          grid = std::max<int64_t>(1, std::min<int64_t>(grid, slab_budget(c) / (slabT * 4)));
          if ((st = buf_ensure(c, c->slab, size_t(grid) * size_t(slabT) * 4, s)) != SPG_OK) return st;
          {
            ProfScope _ps(c, ss, "k_sym_global<1024>");
            k_sym_global<1024><<<(unsigned)grid, 1024, 0, ss>>>(rb, n, a, b, flop, row_nnz,
                                                                 (uint32_t *)c->slab.p, slabT);
          }
          SPG_LAUNCHED(c, "k_sym_global");
        }
      }
    }
    if ((st = join(c, s)) != SPG_OK) return st;
  } else if (m > 0) {
    SPG_CUDA(c, cudaMemsetAsync(row_nnz, 0, size_t(m) * 8, s));
  }
  // a4: C_row_ptr = exclusive scan of row nnz (+ numeric bin counts)
  if ((st = launch_scan(c, row_nnz, m, s, A->row_ptr, (const int64_t *)c->flop.p)) != SPG_OK) return st;
  if (m > 0) {
    {
      ProfScope _ps(c, s, "k_bin_scatter_num");
      k_bin_scatter<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(m, C_row_ptr, A->row_ptr, 0, 1, info,
                                                               (int32_t *)c->rows_num.p, nullptr,
                                                               (const int64_t *)c->flop.p, c->accum,
                                                               c->cfac, c->hfac);
    }
    SPG_LAUNCHED(c, "k_bin_scatter(num)");
  }
  if ((st = read_info(c, s)) != SPG_OK) return st;
  c->plan = *c->host_info;
  // the hash parts' tile records did not all fit: the buffer grows at the START
  // of the next symbolic (never between this plan and its numeric phase,
  // whose parts point into the current buffer); these parts hash their keys
  if (c->plan_lists && size_t(c->plan.lists_need + size_t(c->num_sms) * 2 * kPoolList) * 4 > c->lists.bytes)
    c->lists_want = size_t(c->plan.lists_need + (c->plan.lists_need >> 4) +
                           size_t(c->num_sms) * 2 * kPoolList) * 4;
  if (c->plan.pkeys_used * kTileRec * 4 > c->pkeys.bytes && c->plan_parts)
    c->pkeys_want = std::max<size_t>(
        c->pkeys_want, size_t(c->plan.pkeys_used + (c->plan.pkeys_used >> 4) +
                              size_t(c->num_sms) * 2 * kPoolRecs) * kTileRec * 4);
  *nnz_C = (int64_t)c->plan.nnz_total;
  if (flop_total) *flop_total = (int64_t)c->plan.flop_total;
  c->have_plan = true;
  c->plan_a_rp = A0->row_ptr;
  c->plan_b_rp = B->row_ptr;
  c->plan_c_rp = C_row_ptr;
  c->plan_a_col = A0->col_idx;
  c->plan_b_col = B->col_idx;
  c->plan_m = m;
  c->plan_ncols = B->ncols;
  return SPG_OK;
}

spg_status spg_numeric(spg_ctx *c, const spg_csr *A, const spg_csr *B, const int64_t *C_row_ptr,
                       int32_t *C_col_idx, double *C_val, int sorted, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, A, "A", false)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (sorted != 0 && sorted != 1) return fail(c, SPG_ERR_INVALID_ARG, "sorted must be 0 or 1");
  if (!c->have_plan || c->plan_a_rp != A->row_ptr || c->plan_b_rp != B->row_ptr ||
      c->plan_c_rp != C_row_ptr || c->plan_a_col != A->col_idx || c->plan_b_col != B->col_idx ||
      c->plan_m != A->nrows || c->plan_ncols != B->ncols)
    return fail(c, SPG_ERR_STATE, "spg_numeric without a matching spg_symbolic");
  const PlanInfo &h = c->plan;
  if (h.nnz_total == 0) return SPG_OK;
  if (!C_col_idx || !C_val) return fail(c, SPG_ERR_INVALID_ARG, "C_col_idx / C_val is NULL");
  if (!A->val || !B->val) return fail(c, SPG_ERR_INVALID_ARG, "A.val / B.val is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  if (c->pruned) {
    // the plan runs on the pruned A' (same rows, same products): gather its
    // values from the caller's A now (the symbolic needs none)
    if (c->prune_n > 0) {
      ProfScope _ps(c, s, "k_prune_values");
      k_prune_values<<<(unsigned)std::min<int64_t>(ceil_div(c->prune_n, 256), int64_t(c->num_sms) * 8),
                       256, 0, s>>>(A->val, (const int64_t *)c->prune_idx.p, c->prune_n,
                                    (double *)c->prune_val.p);
    }
    SPG_LAUNCHED(c, "k_prune_values");
    A = &c->Ap;
  }
  DevCSR a = dev(A), b = dev(B);
  const int32_t *rows = (const int32_t *)c->rows_num.p;
  const int64_t *flop = (const int64_t *)c->flop.p;
  // G tier: column-tile parts (B sorted, parts cut by the symbolic) or the
  // global-hash fallback (slab: keys + vals of lowest 2^n >= 2 max nnz(c_i) per block)
  int64_t g_grid = 0, slabT = 0, ntiles = 0;
  // (tile offsets are int32 positions: a B with >= 2^31 entries takes the
  // global-hash tier instead)
  const bool use_parts = c->plan_parts && h.b_unsorted == 0 && h.parts_overflow == 0 &&
                         h.b_end < (unsigned long long)INT32_MAX;
  if (h.num_count[NB_G]) {
    if (use_parts) {
      ntiles = (B->ncols + kTileCols - 1) / kTileCols;
      if ((st = buf_ensure(c, c->toff, size_t(B->nrows) * size_t(ntiles + 1) * 4, s)) != SPG_OK)
        return st;
      if ((st = buf_ensure(c, c->parts2, size_t(h.parts_used) * 3 * sizeof(int4), s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->part_hist, size_t(kPartBuckets) * 4, s)) != SPG_OK) return st;
      PlanInfo *dinfo = (PlanInfo *)c->info.p;
      SPG_CUDA(c, cudaMemsetAsync(&dinfo->row_counter, 0, 8, s));
      SPG_CUDA(c, cudaMemsetAsync(c->part_hist.p, 0, size_t(kPartBuckets) * 4, s));
      {
        ProfScope _ps(c, s, "k_tile_offsets");
        const int64_t grid = std::min<int64_t>(ceil_div(B->nrows, kToffRows), int64_t(c->num_sms) * 8);
        k_tile_offsets<<<(unsigned)std::max<int64_t>(grid, 1), 256, size_t(ntiles + 1) * 33 * 4, s>>>(
            b, (int)ntiles, (int32_t *)c->toff.p);
      }
      SPG_LAUNCHED(c, "k_tile_offsets");
      // parts in processing order (dense first, tile ascending)
      const unsigned pgrid = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>(ceil_div((int64_t)h.parts_pool, 256), int64_t(c->num_sms) * 4));
      {
        ProfScope _ps(c, s, "k_parts_hist");
        k_parts_hist<<<pgrid, 256, 0, s>>>((const int4 *)c->parts.p, dinfo, (unsigned *)c->part_hist.p);
      }
      SPG_LAUNCHED(c, "k_parts_hist");
      {
        ProfScope _ps(c, s, "k_parts_scan");
        k_parts_scan<<<1, kPartBuckets, 0, s>>>((unsigned *)c->part_hist.p);
      }
      SPG_LAUNCHED(c, "k_parts_scan");
      {
        ProfScope _ps(c, s, "k_parts_scatter");
        k_parts_scatter<<<pgrid, 256, 0, s>>>((const int4 *)c->parts.p, dinfo, (unsigned *)c->part_hist.p,
                                              (int4 *)c->parts2.p);
      }
      SPG_LAUNCHED(c, "k_parts_scatter");
    } else {
      g_grid = std::min<int64_t>((int64_t)h.num_count[NB_G], int64_t(c->num_sms));
      int lg = log2_ceil64(2 * h.max_nnz);
      slabT = int64_t(1) << std::max(lg, kMinLogT);
      g_grid = std::max<int64_t>(1, std::min<int64_t>(g_grid, slab_budget(c) / (slabT * 12)));
      if ((st = buf_ensure(c, c->slab, size_t(g_grid) * size_t(slabT) * 12, s)) != SPG_OK) return st;
    }
  }
  if ((st = fork(c, s)) != SPG_OK) return st;
  int sidx = 0;
  // heap tier (sorted output only): the rows heap_pick chose sit at the back
  // of the W256 / W1024 bin segments
  const bool use_heap = sorted && (h.heap_count[NB_W256] + h.heap_count[NB_W1024]) > 0;
  if (use_heap) {
    HeapSegs hs;
    hs.n[0] = (long long)h.heap_count[NB_W256];
    hs.n[1] = (long long)h.heap_count[NB_W1024];
    hs.off[0] = bin_offset(h.num_count, NB_W256) + (long long)h.num_count[NB_W256] - hs.n[0];
    hs.off[1] = bin_offset(h.num_count, NB_W1024) + (long long)h.num_count[NB_W1024] - hs.n[1];
    const int64_t nh = hs.n[0] + hs.n[1];
    cudaStream_t ss = c->serial ? s : c->sub[sidx++ % kSubStreams];
    {
      ProfScope _ps(c, ss, "k_num_heap<64>");
      k_num_heap<kHeapThreads><<<(unsigned)std::min<int64_t>(ceil_div(nh, kHeapThreads), int64_t(c->num_sms) * 5),
                                 kHeapThreads, kHeapSmem, ss>>>(rows, hs, a, b, C_row_ptr, C_col_idx, C_val);
    }
    SPG_LAUNCHED(c, "k_num_heap");
  }
  // largest bins first so the long rows start early
  for (int bin = NB_COUNT - 1; bin >= 1; --bin) {
    const int64_t n = (int64_t)h.num_count[bin] - (use_heap ? (int64_t)h.heap_count[bin] : 0);
    if (n == 0) continue;
    const int32_t *rb = rows + bin_offset(h.num_count, bin);
    cudaStream_t ss = c->serial ? s : c->sub[sidx++ % kSubStreams];
    if (bin == NB_W256) {
      const int64_t grid = std::min<int64_t>(ceil_div(n, kWarps), int64_t(c->num_sms) * 32);
      {
        ProfScope _ps(c, ss, "k_num_warp<256>");
        if (sorted)
          k_num_warp<256, kWarps, 1><<<(unsigned)grid, kWarps * 32, kWarps * 256 * 16, ss>>>(
              rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val);
        else
          k_num_warp<256, kWarps, 0><<<(unsigned)grid, kWarps * 32, kWarps * 256 * 16, ss>>>(
              rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val);
      }
      SPG_LAUNCHED(c, "k_num_warp<256>");
    } else if (bin == NB_W1024) {
      const int64_t grid = std::min<int64_t>(ceil_div(n, 4), int64_t(c->num_sms) * 32);
      {
        ProfScope _ps(c, ss, "k_num_warp<1024>");
        if (sorted)
          k_num_warp<1024, 4, 1><<<(unsigned)grid, 4 * 32, 4 * 1024 * 16, ss>>>(
              rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val);
        else
          k_num_warp<1024, 4, 0><<<(unsigned)grid, 4 * 32, 4 * 1024 * 16, ss>>>(
              rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val);
      }
      SPG_LAUNCHED(c, "k_num_warp<1024>");
    } else if (bin >= NB_B2K && bin <= NB_B16K) {
      const int logT = 11 + (bin - NB_B2K);
      const int tmax = 1 << logT;
      const size_t smem = size_t(tmax) * 12;
      const int64_t grid = std::min<int64_t>(n, int64_t(c->num_sms) * 8);
      // rows with a sorted column list from the bitmap symbolic (SPG_TUNE
      // bit 32768 ignores the lists: A/B)
      const bool use_lists = c->plan_lists && !(c->tune & 32768);
      const int64_t *lo_p = use_lists ? (const int64_t *)c->list_off.p : nullptr;
      const int32_t *li_p = use_lists ? (const int32_t *)c->lists.p : nullptr;
      // block size per table size (measured on C3: 2K slots 128 threads,
      // 4K / 8K 512, 16K 1024 -- smaller blocks idle less at the row
      // barrier, larger ones keep the occupancy of the big tables)
      if (logT <= 11) {
        ProfScope _ps(c, ss, "k_num_block<128>");
        k_num_block<128><<<(unsigned)std::min<int64_t>(n, int64_t(c->num_sms) * 32), 128, smem, ss>>>(
            rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val, sorted, tmax, OnePhase{}, lo_p, li_p);
      } else if (logT <= 13) {
        ProfScope _ps(c, ss, "k_num_block<512>");
        k_num_block<512><<<(unsigned)grid, 512, smem, ss>>>(rb, n, a, b, flop, C_row_ptr, C_col_idx,
                                                           C_val, sorted, tmax, OnePhase{}, lo_p, li_p);
      } else {
        ProfScope _ps(c, ss, "k_num_block<1024>");
        k_num_block<1024><<<(unsigned)grid, 1024, smem, ss>>>(rb, n, a, b, flop, C_row_ptr, C_col_idx,
                                                             C_val, sorted, tmax, OnePhase{}, lo_p, li_p);
      }
      SPG_LAUNCHED(c, "k_num_block");
    } else if (use_parts) {  // NB_G: column-tile parts, independent work items
      {
        ProfScope _ps(c, ss, "k_num_tpart<512>");
        PlanInfo *dinfo = (PlanInfo *)c->info.p;
        k_num_tpart<512><<<(unsigned)(2 * c->num_sms), 512, kTPartSmem, ss>>>(
            a, b, C_row_ptr, C_col_idx, C_val, sorted, (const int4 *)c->parts2.p,
            (int64_t)h.parts_used, (const int32_t *)c->toff.p, B->nrows, &dinfo->row_counter,
            c->tune, dinfo->dbg, (c->tune & 256) ? nullptr : (const uint32_t *)c->pkeys.p,
            (c->tune & 1024) ? nullptr : (const uint16_t *)c->dpfx.p);
      }
      SPG_LAUNCHED(c, "k_num_tpart");
    } else {  // NB_G
      uint32_t *sk = (uint32_t *)c->slab.p;
      double *sv = (double *)((char *)c->slab.p + size_t(g_grid) * size_t(slabT) * 4);
      {
        ProfScope _ps(c, ss, "k_num_global<1024>");
        k_num_global<1024><<<(unsigned)g_grid, 1024, sorted ? kRankSmem : 0, ss>>>(
            rb, n, a, b, flop, C_row_ptr, C_col_idx, C_val, sorted, sk, sv, slabT);
      }
      SPG_LAUNCHED(c, "k_num_global");
    }
  }
  return join(c, s);
}

spg_status spg_set_accumulator(spg_ctx *c, int accum, double collision_factor, double heap_cost) {
  if (!c) return SPG_ERR_INVALID_ARG;
  if (accum < SPG_ACCUM_AUTO || accum > SPG_ACCUM_HEAP)
    return fail(c, SPG_ERR_INVALID_ARG, "accumulator must be SPG_ACCUM_AUTO, _HASH or _HEAP");
  if (!(collision_factor >= 1.0) || collision_factor > 1e6)
    return fail(c, SPG_ERR_INVALID_ARG, "collision factor must be >= 1");
  if (!(heap_cost > 0.0) || heap_cost > 1e6)
    return fail(c, SPG_ERR_INVALID_ARG, "heap cost must be > 0");
  c->accum = accum;
  c->cfac = (float)collision_factor;
  c->hfac = (float)heap_cost;
  return SPG_OK;
}

// One-phase multiply, step 1: see include/spgemm.h.
spg_status spg_onephase(spg_ctx *c, const spg_csr *A, const spg_csr *B, int64_t *C_row_ptr,
                        int64_t *nnz_C, int64_t *flop_total, int sorted, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  c->have_one = false;
  c->have_plan = false;
  spg_status st;
  if ((st = check_csr(c, A, "A", true)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", true)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (!C_row_ptr || !nnz_C) return fail(c, SPG_ERR_INVALID_ARG, "C_row_ptr / nnz_C is NULL");
  if (sorted != 0 && sorted != 1) return fail(c, SPG_ERR_INVALID_ARG, "sorted must be 0 or 1");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  const int64_t m = A->nrows;
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->flop, size_t(std::max<int64_t>(m, 1)) * 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->rows_sym, size_t(std::max<int64_t>(m, 1)) * 4, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->one_fofs, size_t(m + 1) * 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->bnz, size_t((B->nrows + 31) / 32) * 4, s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  int64_t *row_nnz = C_row_ptr + 1;
  int64_t *fofs = (int64_t *)c->one_fofs.p;
  // the launch sequence up to the host read, replayed as a CUDA graph when
  // the inputs, outputs and workspace are the ones it was captured with
  // (SPG_ONEPHASE_GRAPH=0 disables; the launch-bound small configs gain
  // most), else enqueued on `s`
  auto enqueue = [&](unsigned long long cap, cudaStream_t s) -> spg_status {
    spg_status st;
    SPG_CUDA(c, cudaMemsetAsync(info, 0, sizeof(PlanInfo), s));
    SPG_CUDA(c, cudaMemsetAsync(C_row_ptr, 0, size_t(m + 1) * 8, s));
    if (m > 0 && B->nrows > 0) {
      // B nonempty-row bitmap: the flop pass skips the B.row_ptr gathers of
      // empty B rows when most are empty (decided on the device; C4)
      {
        ProfScope _ps(c, s, "k_b_rowmask");
        const int64_t nw = (B->nrows + 31) / 32;
        k_b_rowmask<<<(unsigned)std::min<int64_t>(ceil_div(nw * 32, 256), int64_t(c->num_sms) * 8), 256, 0, s>>>(
            dev(B), (uint32_t *)c->bnz.p, info);
      }
      SPG_LAUNCHED(c, "k_b_rowmask");
      // a1 + a2: flop, one-phase bins (the tables are sized by the flop bound)
      if ((st = launch_flop(c, A, B, 2, s, (const uint32_t *)c->bnz.p)) != SPG_OK) return st;
      {
        ProfScope _ps(c, s, "k_bin_scatter_1p");
        k_bin_scatter<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(m, (const int64_t *)c->flop.p, A->row_ptr,
                                                                 B->ncols, 2, info, (int32_t *)c->rows_sym.p,
                                                                 row_nnz);
      }
      SPG_LAUNCHED(c, "k_bin_scatter(sym)");
      // workspace row offsets: exclusive prefix of flop
      SPG_CUDA(c, cudaMemsetAsync(fofs, 0, 8, s));
      SPG_CUDA(c, cudaMemcpyAsync(fofs + 1, c->flop.p, size_t(m) * 8, cudaMemcpyDeviceToDevice, s));
      if ((st = launch_scan(c, fofs + 1, m, s)) != SPG_OK) return st;
      if (cap > 0) {
        // a6 (+ a7) on the symbolic bins, counts read on the device
        DevCSR a = dev(A), b = dev(B);
        const int32_t *rows = (const int32_t *)c->rows_sym.p;
        const int64_t *flop = (const int64_t *)c->flop.p;
        int32_t *tc = (int32_t *)c->one_col.p;
        double *tv = (double *)c->one_val.p;
        OnePhase op{info, fofs, row_nnz, cap, SB_W128};
        const unsigned gw = (unsigned)(c->num_sms * 16);
        {
          ProfScope _ps(c, s, "k_num_warp<256>(1p)");
          if (sorted)
            k_num_warp<256, kWarps, 1, true><<<gw, kWarps * 32, kWarps * 256 * 16, s>>>(rows, 0, a, b, flop, nullptr, tc, tv, op);
          else
            k_num_warp<256, kWarps, 0, true><<<gw, kWarps * 32, kWarps * 256 * 16, s>>>(rows, 0, a, b, flop, nullptr, tc, tv, op);
        }
        SPG_LAUNCHED(c, "k_num_warp(1p)");
        op.bin = SB_W1024;
        {
          ProfScope _ps(c, s, "k_num_warp<1024>(1p)");
          if (sorted)
            k_num_warp<1024, 4, 1, true><<<gw, 4 * 32, 4 * 1024 * 16, s>>>(rows, 0, a, b, flop, nullptr, tc, tv, op);
          else
            k_num_warp<1024, 4, 0, true><<<gw, 4 * 32, 4 * 1024 * 16, s>>>(rows, 0, a, b, flop, nullptr, tc, tv, op);
        }
        SPG_LAUNCHED(c, "k_num_warp(1p)");
        for (int bin = SB_B2K; bin <= SB_B16K; ++bin) {
          op.bin = bin;
          const int tmax = 2048 << (bin - SB_B2K);
          ProfScope _ps(c, s, "k_num_block(1p)");
          if (tmax == 2048)
            k_num_block<128, true><<<(unsigned)(c->num_sms * 8), 128, size_t(tmax) * 12, s>>>(
                rows, 0, a, b, flop, nullptr, tc, tv, sorted, tmax, op);
          else if (tmax <= 8192)
            k_num_block<512, true><<<(unsigned)(c->num_sms * 4), 512, size_t(tmax) * 12, s>>>(
                rows, 0, a, b, flop, nullptr, tc, tv, sorted, tmax, op);
          else
            k_num_block<1024, true><<<(unsigned)(c->num_sms), 1024, size_t(tmax) * 12, s>>>(
                rows, 0, a, b, flop, nullptr, tc, tv, sorted, tmax, op);
          SPG_LAUNCHED(c, "k_num_block(1p)");
        }
      }
    }
    // a4: C_row_ptr = exclusive scan of nnz(c_i)
    if ((st = launch_scan(c, row_nnz, m, s)) != SPG_OK) return st;
    return SPG_OK;
  };
  for (int attempt = 0; attempt < 2; ++attempt) {
    // workspace: grow-only, sized by the last flop total seen
    const unsigned long long cap = (unsigned long long)(c->one_col.bytes / 4);
    const spg_ctx::OneKeyT key{A->row_ptr, A->col_idx, A->val, A->nrows, A->ncols, B->row_ptr, B->col_idx, B->val,
                     B->nrows, B->ncols, C_row_ptr, sorted, c->one_col.p, cap};
    const bool use_graph = c->one_graph_ok && !c->profiling && m > 0;
    if (use_graph && c->one_exec && key == c->one_key) {
      SPG_CUDA(c, cudaGraphLaunch(c->one_exec, s));
      c->launches += c->one_graph_launches;
    } else if (use_graph) {
      // everything the sequence allocates is sized before the capture
      if ((st = buf_ensure(c, c->trow, size_t(m + 1) * 8, s)) != SPG_OK) return st;
      if ((st = buf_ensure(c, c->partial, size_t(ceil_div(m, kScanTile)) * 8, s)) != SPG_OK) return st;
      if (c->one_exec) { cudaGraphExecDestroy(c->one_exec); c->one_exec = nullptr; }
      cudaGraph_t g = nullptr;
      const int64_t l0 = c->launches;
      // (captured on an internal stream: the caller's may be the legacy
      // default stream, which cannot be captured)
      cudaStream_t cs = c->sub[0];
      SPG_CUDA(c, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      const spg_status st2 = enqueue(cap, cs);
      const cudaError_t e2 = cudaStreamEndCapture(cs, &g);
      if (st2 != SPG_OK) { if (g) cudaGraphDestroy(g); return st2; }
      SPG_CUDA(c, e2);
      cudaGraphExec_t ex = nullptr;
      const cudaError_t e3 = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      SPG_CUDA(c, e3);
      c->one_exec = ex;
      c->one_key = key;
      c->one_graph_launches = c->launches - l0;
      SPG_CUDA(c, cudaGraphLaunch(c->one_exec, s));
    } else {
      if ((st = enqueue(cap, s)) != SPG_OK) return st;
    }
    if ((st = read_info(c, s)) != SPG_OK) return st;  // the one host round trip
    const PlanInfo &h = *c->host_info;
    if (h.sym_count[SB_G])
      return fail(c, SPG_ERR_OVERFLOW,
                  "one-phase: rows need tables beyond 16384 slots (min(flop_i, N_col) > 8192); use "
                  "spg_symbolic + spg_numeric");
    if ((int64_t)h.max_brow > kMaxBRow) return fail(c, SPG_ERR_OVERFLOW, "a row of B has more than 2^26 entries");
    if (h.flop_total <= cap || h.flop_total == 0) {
      *nnz_C = (int64_t)h.nnz_total;
      if (flop_total) *flop_total = (int64_t)h.flop_total;
      c->have_one = true;
      c->one_m = m;
      c->one_rp = C_row_ptr;
      return SPG_OK;
    }
    // the workspace was too small: grow it to this flop total and rerun once
    const size_t want = size_t(h.flop_total) + (size_t(h.flop_total) >> 3);
    if (want > size_t(1) << 40) return fail(c, SPG_ERR_WORKSPACE, "one-phase workspace too large");
    if ((st = buf_ensure(c, c->one_col, want * 4, s)) != SPG_OK) return st;
    if ((st = buf_ensure(c, c->one_val, want * 8, s)) != SPG_OK) return st;
  }
  return fail(c, SPG_ERR_WORKSPACE, "one-phase workspace could not be sized");
}

// One-phase multiply, step 2: compact the rows into the caller's C.
spg_status spg_onephase_emit(spg_ctx *c, int32_t *C_col_idx, double *C_val, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  if (!c->have_one) return fail(c, SPG_ERR_STATE, "spg_onephase_emit without a matching spg_onephase");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  const int64_t m = c->one_m;
  if (m > 0 && (C_col_idx || C_val)) {
    if (!C_col_idx || !C_val) return fail(c, SPG_ERR_INVALID_ARG, "C_col_idx / C_val is NULL");
    ProfScope _ps(c, s, "k_onephase_copy");
    k_onephase_copy<<<(unsigned)std::min<int64_t>(ceil_div(m, 8), int64_t(c->num_sms) * 16), 256, 0, s>>>(
        m, (const int64_t *)c->one_fofs.p, c->one_rp, (const int32_t *)c->one_col.p,
        (const double *)c->one_val.p, C_col_idx, C_val);
    SPG_LAUNCHED(c, "k_onephase_copy");
  }
  c->have_one = false;
  return SPG_OK;
}

spg_status spg_debug_counters(spg_ctx *c, int64_t *out, void *stream) {
  if (!c || !out) return SPG_ERR_INVALID_ARG;
  if (!c->info.p) return fail(c, SPG_ERR_STATE, "no plan");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaMemcpyAsync(out, ((PlanInfo *)c->info.p)->dbg, 16 * 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  return SPG_OK;
}

spg_status spg_plan_export(spg_ctx *c, int64_t *flop_out, int64_t *tsize_out, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  if (!c->have_plan) return fail(c, SPG_ERR_STATE, "no symbolic plan");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t m = c->plan_m;
  if (m == 0) return SPG_OK;
  if (flop_out)
    SPG_CUDA(c, cudaMemcpyAsync(flop_out, c->flop.p, size_t(m) * 8, cudaMemcpyDeviceToDevice, s));
  if (tsize_out) {
    // table size of the paper's rule, computed on the device from the plan
    {
      ProfScope _ps(c, s, "k_plan_tsize");
      k_plan_tsize<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>((const int64_t *)c->flop.p, m,
                                                              c->plan_ncols, tsize_out);
    }
    SPG_LAUNCHED(c, "k_plan_tsize");
  }
  return SPG_OK;
}

spg_status spg_rows_to_parts(spg_ctx *c, const spg_csr *A, const spg_csr *B, int64_t nparts,
                             int64_t *offsets, int64_t *flop_total, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, A, "A", false)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (nparts < 1 || !offsets) return fail(c, SPG_ERR_INVALID_ARG, "nparts < 1 or offsets NULL");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  const int64_t m = A->nrows;
  c->have_plan = false;  // the flop buffer is reused
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->flop, size_t(m + 1) * 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->scratch, size_t(m + 1 + nparts + 1) * 8, s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  int64_t *ps = (int64_t *)c->scratch.p;
  int64_t *doff = ps + (m + 1);
  SPG_CUDA(c, cudaMemsetAsync(info, 0, sizeof(PlanInfo), s));
  SPG_CUDA(c, cudaMemsetAsync(ps, 0, size_t(m + 1) * 8, s));
  if (m > 0 && B->nrows > 0) {
    if ((st = launch_flop(c, A, B, 0, s)) != SPG_OK) return st;
    SPG_CUDA(c, cudaMemcpyAsync(ps + 1, c->flop.p, size_t(m) * 8, cudaMemcpyDeviceToDevice, s));
    if ((st = launch_scan(c, ps + 1, m, s)) != SPG_OK) return st;  // ParallelPrefixSum
  }
  {
    ProfScope _ps(c, s, "k_lowbnd");
    k_lowbnd<<<(unsigned)ceil_div(nparts + 1, 256), 256, 0, s>>>(ps, m, nparts, doff);
  }
  SPG_LAUNCHED(c, "k_lowbnd");
  SPG_CUDA(c, cudaMemcpyAsync(offsets, doff, size_t(nparts + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (flop_total) SPG_CUDA(c, cudaMemcpyAsync(flop_total, ps + m, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  return SPG_OK;
}

spg_status spg_rows_to_parts_bytes(spg_ctx *c, const spg_csr *A, const spg_csr *B,
                                   const int64_t *row_nnz, int64_t nparts, int64_t *offsets,
                                   int64_t *bytes_total, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, A, "A", false)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (nparts < 1 || !offsets) return fail(c, SPG_ERR_INVALID_ARG, "nparts < 1 or offsets NULL");
  const int64_t m = A->nrows;
  if (m > 0 && !row_nnz) return fail(c, SPG_ERR_INVALID_ARG, "row_nnz is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  c->have_plan = false;  // the flop buffer is reused
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->flop, size_t(m + 1) * 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->scratch, size_t(m + 1 + nparts + 1) * 8, s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  int64_t *ps = (int64_t *)c->scratch.p;
  int64_t *doff = ps + (m + 1);
  SPG_CUDA(c, cudaMemsetAsync(info, 0, sizeof(PlanInfo), s));
  SPG_CUDA(c, cudaMemsetAsync(ps, 0, size_t(m + 1) * 8, s));
  if (m > 0) {
    if (B->nrows > 0) {
      if ((st = launch_flop(c, A, B, 0, s)) != SPG_OK) return st;
    } else {
      SPG_CUDA(c, cudaMemsetAsync(c->flop.p, 0, size_t(m) * 8, s));
    }
    {
      ProfScope _ps(c, s, "k_row_bytes");
      k_row_bytes<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), int64_t(c->num_sms) * 8), 256, 0, s>>>(
          A->row_ptr, (const int64_t *)c->flop.p, row_nnz, m, ps + 1);
    }
    SPG_LAUNCHED(c, "k_row_bytes");
    if ((st = launch_scan(c, ps + 1, m, s)) != SPG_OK) return st;
  }
  {
    ProfScope _ps(c, s, "k_lowbnd");
    k_lowbnd<<<(unsigned)ceil_div(nparts + 1, 256), 256, 0, s>>>(ps, m, nparts, doff);
  }
  SPG_LAUNCHED(c, "k_lowbnd");
  SPG_CUDA(c, cudaMemcpyAsync(offsets, doff, size_t(nparts + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (bytes_total) SPG_CUDA(c, cudaMemcpyAsync(bytes_total, ps + m, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  return SPG_OK;
}

spg_status spg_mask_sum(spg_ctx *c, const spg_csr *C, const spg_csr *G, int64_t g_row_begin,
                        int64_t *sum, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, C, "C", true)) != SPG_OK) return st;
  if ((st = check_csr(c, G, "G", false)) != SPG_OK) return st;
  if (!sum || g_row_begin < 0 || g_row_begin + C->nrows > G->nrows)
    return fail(c, SPG_ERR_INVALID_ARG, "bad mask row range or NULL sum");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  // both queues, the fp64 sum, the list lengths, the int64 sum and its flag
  SPG_CUDA(c, cudaMemsetAsync(info->mask_ctr, 0, 7 * 8, s));
  if (C->nrows > 0) {
    if ((st = buf_ensure(c, c->mask_rows, size_t(C->nrows) * 8, s)) != SPG_OK) return st;
    int32_t *list_w = (int32_t *)c->mask_rows.p, *list_b = list_w + C->nrows;
    {
      ProfScope _ps(c, s, "k_mask_rows");
      k_mask_rows<<<(unsigned)std::min<int64_t>(ceil_div(C->nrows, 256), c->num_sms * 8), 256, 0,
                    s>>>(C->row_ptr, C->nrows, dev(G), g_row_begin, list_w, list_b, info->mask_n);
    }
    SPG_LAUNCHED(c, "k_mask_rows");
    {
      ProfScope _ps(c, s, "k_csr_mask_sum_warp<8>");
      k_csr_mask_sum_warp<kWarps><<<(unsigned)(c->num_sms * 8), kWarps * 32, 0, s>>>(
          dev(C), dev(G), g_row_begin, list_w, &info->mask_n[0], &info->mask_ctr[0], info);
    }
    SPG_LAUNCHED(c, "k_csr_mask_sum_warp");
    const int use_bitmap = G->ncols <= kBitmapMaxCols ? 1 : 0;
    const size_t smem = use_bitmap ? size_t((G->ncols + 31) / 32) * 4 : 0;
    {
      ProfScope _ps(c, s, "k_csr_mask_sum_block<1024>");
      k_csr_mask_sum_block<1024><<<(unsigned)c->num_sms, 1024, smem, s>>>(
          dev(C), dev(G), g_row_begin, list_b, &info->mask_n[1], &info->mask_ctr[1], info,
          use_bitmap);
    }
    SPG_LAUNCHED(c, "k_csr_mask_sum_block");
  }
  SPG_CUDA(c, cudaMemcpyAsync(&c->host_info->mask_acc, &info->mask_acc, 5 * 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  // exact int64 reduction for integer-valued C (triangle counts); else the
  // fp64 sum rounded
  *sum = c->host_info->mask_inexact ? (int64_t)llround(c->host_info->mask_acc)
                                    : (int64_t)c->host_info->mask_isum;
  return SPG_OK;
}

static spg_status masked_sum_impl(spg_ctx *c, const spg_csr *A, const spg_csr *B, const spg_csr *G,
                                  int64_t g_row_begin, double *sum, int64_t *isum, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, A, "A", true)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", true)) != SPG_OK) return st;
  if ((st = check_csr(c, G, "G", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (G->ncols != B->ncols) return fail(c, SPG_ERR_DIM_MISMATCH, "G.ncols != B.ncols");
  if ((!sum && !isum) || g_row_begin < 0 || g_row_begin + A->nrows > G->nrows)
    return fail(c, SPG_ERR_INVALID_ARG, "bad mask row range or NULL sum");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  SPG_CUDA(c, cudaMemsetAsync(info->mask_ctr, 0, 7 * 8, s));  // queues, sums, list lengths, flag
  if (A->nrows > 0 && B->nrows > 0) {
    DevCSR a = dev(A), b = dev(B), g = dev(G);
    if ((st = buf_ensure(c, c->mask_rows, size_t(A->nrows) * 8, s)) != SPG_OK) return st;
    int32_t *list_w = (int32_t *)c->mask_rows.p, *list_b = list_w + A->nrows;
    {
      ProfScope _ps(c, s, "k_mask_rows");
      k_mask_rows<<<(unsigned)std::min<int64_t>(ceil_div(A->nrows, 256), c->num_sms * 8), 256, 0,
                    s>>>(A->row_ptr, A->nrows, g, g_row_begin, list_w, list_b, info->mask_n);
    }
    SPG_LAUNCHED(c, "k_mask_rows");
    {
      ProfScope _ps(c, s, "k_mask_sum_warp<8>");
      k_mask_sum_warp<kWarps><<<(unsigned)(c->num_sms * 8), kWarps * 32, 0, s>>>(
          a, b, g, g_row_begin, list_w, &info->mask_n[0], &info->mask_ctr[0], info);
    }
    SPG_LAUNCHED(c, "k_mask_sum_warp");
    const int use_bitmap = B->ncols <= kBitmapMaxCols ? 1 : 0;
    const size_t smem = use_bitmap ? size_t((B->ncols + 31) / 32) * 4 : 0;
    {
      ProfScope _ps(c, s, "k_mask_sum_block<1024>");
      k_mask_sum_block<1024><<<(unsigned)c->num_sms, 1024, smem, s>>>(
          a, b, g, g_row_begin, list_b, &info->mask_n[1], &info->mask_ctr[1], info, use_bitmap);
    }
    SPG_LAUNCHED(c, "k_mask_sum_block");
  }
  SPG_CUDA(c, cudaMemcpyAsync(&c->host_info->mask_acc, &info->mask_acc, 5 * 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  if (sum) *sum = c->host_info->mask_acc;
  if (isum) {
    if (c->host_info->mask_inexact)
      return fail(c, SPG_ERR_OVERFLOW,
                  "masked sum is not an exact integer (non-integer values or a partial >= 2^53)");
    *isum = (int64_t)c->host_info->mask_isum;
  }
  return SPG_OK;
}

spg_status spg_masked_sum(spg_ctx *c, const spg_csr *A, const spg_csr *B, const spg_csr *G,
                          int64_t g_row_begin, double *sum, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  if (!sum) return fail(c, SPG_ERR_INVALID_ARG, "NULL sum");
  return masked_sum_impl(c, A, B, G, g_row_begin, sum, nullptr, stream);
}

spg_status spg_masked_sum_int(spg_ctx *c, const spg_csr *A, const spg_csr *B, const spg_csr *G,
                              int64_t g_row_begin, int64_t *sum, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  if (!sum) return fail(c, SPG_ERR_INVALID_ARG, "NULL sum");
  return masked_sum_impl(c, A, B, G, g_row_begin, nullptr, sum, stream);
}


spg_status spg_degree_relabel(spg_ctx *c, const spg_csr *G, int32_t *perm, int64_t *L_rp,
                              int32_t *L_col, double *L_val, int64_t *U_rp, int32_t *U_col,
                              double *U_val, int64_t *G_rp, int32_t *G_col, double *G_val,
                              void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, G, "G", false)) != SPG_OK) return st;
  if (G->nrows != G->ncols) return fail(c, SPG_ERR_DIM_MISMATCH, "G must be square");
  if ((G->nrows > 0 && !perm) || !L_rp || !U_rp || !G_rp)
    return fail(c, SPG_ERR_INVALID_ARG, "NULL output");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  const int64_t n = G->nrows;
  int64_t nnz = 0;
  if (n > 0) {
    int64_t ends[2];
    SPG_CUDA(c, cudaMemcpyAsync(&ends[0], G->row_ptr, 8, cudaMemcpyDeviceToHost, s));
    SPG_CUDA(c, cudaMemcpyAsync(&ends[1], G->row_ptr + n, 8, cudaMemcpyDeviceToHost, s));
    SPG_CUDA(c, cudaStreamSynchronize(s));
    nnz = ends[1] - ends[0];
  }
  if (nnz % 2 != 0) return fail(c, SPG_ERR_INVALID_ARG, "nnz(G) is odd: G is not a symmetric pattern");
  if (n >= INT32_MAX || nnz >= INT32_MAX)
    return fail(c, SPG_ERR_OVERFLOW, "degree relabel supports n, nnz(G) < 2^31");
  if (nnz > 0 && (!L_col || !U_col || !G_col)) return fail(c, SPG_ERR_INVALID_ARG, "NULL output");
  SPG_CUDA(c, cudaMemsetAsync(L_rp, 0, 8, s));
  SPG_CUDA(c, cudaMemsetAsync(U_rp, 0, 8, s));
  SPG_CUDA(c, cudaMemsetAsync(G_rp, 0, 8, s));
  if (n == 0) return SPG_OK;
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  // rl_key: degree histogram / fill counters (int64[n+1] each), bucket offsets
  // int64[n+2] (degrees 0..n; n only with an invalid diagonal entry);
  // rl_rank: rank int32[n] + degree buckets int32[n] + long-segment list int32[n]
  if ((st = buf_ensure(c, c->rl_key, size_t(n + 1) * 24 + 8, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->rl_rank, size_t(n) * 12, s)) != SPG_OK) return st;
  if ((st = buf_ensure(c, c->rl_tmp, size_t(std::max<int64_t>(nnz, 1)) * 8, s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  unsigned long long *bad = &info->mask_ctr[0];
  unsigned long long *nlong = &info->mask_ctr[1];
  SPG_CUDA(c, cudaMemsetAsync(info->mask_ctr, 0, 16, s));
  unsigned long long *hist = (unsigned long long *)c->rl_key.p, *fill = hist + (n + 1);
  int64_t *dstart = (int64_t *)(fill + (n + 1));
  int32_t *rank = (int32_t *)c->rl_rank.p, *bucket = rank + n, *longs = bucket + n;
  int32_t *Lt = (int32_t *)c->rl_tmp.p, *Ut = Lt + nnz / 2, *Gt = Lt + nnz;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), int64_t(c->num_sms) * 8);
  const unsigned wgrid = (unsigned)std::min<int64_t>(ceil_div(n, 8), int64_t(c->num_sms) * 16);
  const int lwords = (int)std::min<int64_t>((n + 31) / 32, kBitmapMaxCols / 32);
  const size_t lsmem = size_t(lwords) * 4;
  // segmented sort of distinct ids (ascending) of [seg[i], seg[i+1]), i < nseg
  auto segsort = [&](const int32_t *in, int32_t *out, const int64_t *seg, int64_t nseg) -> spg_status {
    if (nseg <= 0) return SPG_OK;
    SPG_CUDA(c, cudaMemsetAsync(nlong, 0, 8, s));
    { ProfScope _ps(c, s, "k_segsort_warp");
    k_segsort_warp<8><<<(unsigned)std::min<int64_t>(ceil_div(nseg, 8), int64_t(c->num_sms) * 8), 256, 0, s>>>(
        in, out, seg, nseg, longs, nlong); }
    SPG_LAUNCHED(c, "k_segsort_warp");
    { ProfScope _ps(c, s, "k_segsort_long");
      k_segsort_long<1024><<<(unsigned)c->num_sms, 1024, lsmem, s>>>(in, out, seg, longs, nlong, n, lwords); }
    SPG_LAUNCHED(c, "k_segsort_long");
    return SPG_OK;
  };
  DevCSR g = dev(G);
  // vertex order (deg(v), v): counting sort by degree, then each degree
  // bucket sorted by id
  SPG_CUDA(c, cudaMemsetAsync(hist, 0, size_t(n + 1) * 16, s));  // hist + fill
  { ProfScope _ps(c, s, "k_rl_deghist"); k_rl_deghist<<<grid, 256, 0, s>>>(g, hist); }
  SPG_LAUNCHED(c, "k_rl_deghist");
  SPG_CUDA(c, cudaMemsetAsync(dstart, 0, 8, s));
  SPG_CUDA(c, cudaMemcpyAsync(dstart + 1, hist, size_t(n + 1) * 8, cudaMemcpyDeviceToDevice, s));
  if ((st = launch_scan(c, dstart + 1, n + 1, s)) != SPG_OK) return st;  // bucket offsets (degrees 0..n)
  { ProfScope _ps(c, s, "k_rl_degscatter"); k_rl_degscatter<<<grid, 256, 0, s>>>(g, dstart, fill, bucket); }
  SPG_LAUNCHED(c, "k_rl_degscatter");
  if ((st = segsort(bucket, rank, dstart, n + 1)) != SPG_OK) return st;  // (rank: the sorted ids, temporarily)
  { ProfScope _ps(c, s, "k_rl_rank"); k_rl_rank<<<grid, 256, 0, s>>>(rank, n, perm, bucket); }  // bucket <- rank[v]
  SPG_LAUNCHED(c, "k_rl_rank");
  int32_t *rk = bucket;
  { ProfScope _ps(c, s, "k_rl_count"); k_rl_count<<<wgrid, 256, 0, s>>>(g, perm, rk, L_rp + 1, U_rp + 1, G_rp + 1, bad); }
  SPG_LAUNCHED(c, "k_rl_count");
  for (int64_t *rp : {L_rp, U_rp, G_rp})
    if ((st = launch_scan(c, rp + 1, n, s)) != SPG_OK) return st;
  int64_t tail[3];
  SPG_CUDA(c, cudaMemcpyAsync(&tail[0], L_rp + n, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaMemcpyAsync(&tail[1], U_rp + n, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaMemcpyAsync(&tail[2], bad, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  if (tail[2] != 0 || tail[0] != nnz / 2 || tail[1] != nnz / 2)
    return fail(c, SPG_ERR_INVALID_ARG,
                "G is not a symmetric pattern without diagonal (lower/upper counts differ or a "
                "diagonal entry is present)");
  if (nnz == 0) return SPG_OK;
  { ProfScope _ps(c, s, "k_rl_fill"); k_rl_fill<<<wgrid, 256, 0, s>>>(g, perm, rk, L_rp, U_rp, G_rp, Lt, Ut, Gt); }
  SPG_LAUNCHED(c, "k_rl_fill");
  if ((st = segsort(Gt, G_col, G_rp, n)) != SPG_OK) return st;
  if ((st = segsort(Lt, L_col, L_rp, n)) != SPG_OK) return st;
  if ((st = segsort(Ut, U_col, U_rp, n)) != SPG_OK) return st;
  const unsigned vgrid = (unsigned)std::min<int64_t>(ceil_div(nnz, 256), int64_t(c->num_sms) * 8);
  if (L_val) { k_fill_f64<<<vgrid, 256, 0, s>>>(L_val, nnz / 2, 1.0); SPG_LAUNCHED(c, "k_fill_f64"); }
  if (U_val) { k_fill_f64<<<vgrid, 256, 0, s>>>(U_val, nnz / 2, 1.0); SPG_LAUNCHED(c, "k_fill_f64"); }
  if (G_val) { k_fill_f64<<<vgrid, 256, 0, s>>>(G_val, nnz, 1.0); SPG_LAUNCHED(c, "k_fill_f64"); }
  return SPG_OK;
}

spg_status spg_probe_stats(spg_ctx *c, const spg_csr *A, const spg_csr *B,
                           const int64_t *C_row_ptr, int64_t *out, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, A, "A", false)) != SPG_OK) return st;
  if ((st = check_csr(c, B, "B", false)) != SPG_OK) return st;
  if (A->ncols != B->nrows) return fail(c, SPG_ERR_DIM_MISMATCH, "A.ncols != B.nrows");
  if (!out || (A->nrows > 0 && !C_row_ptr)) return fail(c, SPG_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  if ((st = buf_ensure(c, c->scratch, 12 * 8, s)) != SPG_OK) return st;
  unsigned long long *d = (unsigned long long *)c->scratch.p;
  SPG_CUDA(c, cudaMemsetAsync(d, 0, 12 * 8, s));
  if (A->nrows > 0) {
    k_probe_stats<kWarps><<<(unsigned)std::min<int64_t>(ceil_div(A->nrows, kWarps), c->num_sms * 16),
                            kWarps * 32, 0, s>>>(dev(A), dev(B), C_row_ptr, d);
    SPG_LAUNCHED(c, "k_probe_stats");
  }
  SPG_CUDA(c, cudaMemcpyAsync(out, d, 12 * 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  return SPG_OK;
}

spg_status spg_validate(spg_ctx *c, const spg_csr *M, int check_sorted, void *stream) {
  if (!c) return SPG_ERR_INVALID_ARG;
  spg_status st;
  if ((st = check_csr(c, M, "M", false)) != SPG_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  SPG_CUDA(c, cudaSetDevice(c->device));
  if ((st = buf_ensure(c, c->info, sizeof(PlanInfo), s)) != SPG_OK) return st;
  PlanInfo *info = (PlanInfo *)c->info.p;
  SPG_CUDA(c, cudaMemsetAsync(&info->flags, 0, 8, s));
  if (M->nrows > 0) {
    const int64_t grid = std::min<int64_t>(ceil_div(M->nrows, 8), int64_t(c->num_sms) * 16);
    {
      ProfScope _ps(c, s, "k_validate");
      k_validate<<<(unsigned)grid, 256, 0, s>>>(dev(M), check_sorted, &info->flags);
    }
    SPG_LAUNCHED(c, "k_validate");
  }
  SPG_CUDA(c, cudaMemcpyAsync(&c->host_info->flags, &info->flags, 8, cudaMemcpyDeviceToHost, s));
  SPG_CUDA(c, cudaStreamSynchronize(s));
  const unsigned long long f = c->host_info->flags;
  if (f & 1) return fail(c, SPG_ERR_INVALID_ARG, "row_ptr is not nondecreasing");
  if (f & 2) return fail(c, SPG_ERR_INDEX_RANGE, "column index outside [0, ncols)");
  if (f & 4) return fail(c, SPG_ERR_INVALID_ARG, "a row is not strictly increasing");
  return SPG_OK;
}

}  // extern "C"

