/*
 * spgemm.h -- C ABI of the B200-native hash SpGEMM hot path.
 *
 * Method: Gustavson's row-wise SpGEMM C = A*B on CSR (§2,
 * Fig:code_spgemm) with a hash-table accumulator in two phases,
 * symbolic then numeric (Fig:hash_spgemm), optional per-row
 * ascending column sort of C.  "P:n" = line n of PAPER.md.
 *
 * Conventions (all entry points):
 *   - Matrix pointers inside spg_csr are DEVICE pointers on the current CUDA
 *     device.  The caller owns every buffer and the stream; the library never
 *     frees caller memory.  Inputs are never written.
 *   - Scalars returned through int64_t* out-parameters are HOST pointers.
 *   - `stream` is a cudaStream_t passed as void*.  Every call enqueues its
 *     work on `stream` (it may fork to internal streams and joins back before
 *     returning or before the stream's next work); NULL = legacy default stream.
 *   - Every call returns spg_status; nothing aborts.  spg_last_error(ctx)
 *     gives a message for the last failing call on that ctx.
 *   - One spg_ctx per concurrent caller (a ctx holds the plan between the two
 *     phases and a grow-only workspace).  A ctx is bound to the device that
 *     was current at spg_ctx_create.
 *   - Types: row_ptr int64, col_idx int32 in [0, ncols) with ncols <= 2^31-1
 *     (0xFFFFFFFF is the hash table's empty key, "initialized by storing
 *     -1"), values fp64.
 *   - No CPU fallback: without a usable CUDA device every call that computes
 *     returns SPG_ERR_CUDA.
 */
#ifndef SPGEMM_H_
#define SPGEMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPG_OK = 0,
    SPG_ERR_INVALID_ARG = 1,  /* NULL pointer, negative size, bad flag          */
    SPG_ERR_DIM_MISMATCH = 2, /* A.ncols != B.nrows (A m x n, B n x k)    */
    SPG_ERR_INDEX_RANGE = 3,  /* column outside [0, ncols) (spg_validate only)   */
    SPG_ERR_OVERFLOW = 4,     /* a B row longer than 2^26, ncols > 2^31-1, ...   */
    SPG_ERR_WORKSPACE = 5,    /* workspace allocation failed                     */
    SPG_ERR_STATE = 6,        /* spg_numeric without a matching spg_symbolic     */
    SPG_ERR_CUDA = 7          /* a CUDA runtime error (message in last_error)    */
} spg_status;

/* A CSR matrix (§2: rpts[n+1], cols[nnz], vals[nnz]).
 * row_ptr[0] MAY be nonzero: a row-range view of a larger matrix is passed as
 * (row_ptr + r0, nrows = r1 - r0) with the SAME col_idx/val base pointers;
 * entries of row i are col_idx[row_ptr[i] .. row_ptr[i+1]-1].  Columns within
 * a row must be unique; their order is arbitrary ("Any" input order,
 * Tab:summary P:155). */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    const int64_t *row_ptr; /* device, [nrows + 1], nondecreasing              */
    const int32_t *col_idx; /* device, indexed by row_ptr                       */
    const double *val;      /* device, indexed by row_ptr; may be NULL for
                               spg_symbolic / spg_validate                      */
} spg_csr;

/* Optional workspace allocator (e.g. the PyTorch caching allocator).  Called
 * only when the ctx workspace must grow; `stream` is the cudaStream_t of the
 * call.  If both are NULL the library uses cudaMalloc/cudaFree. */
typedef void *(*spg_alloc_fn)(size_t bytes, void *stream, void *user);
typedef void (*spg_free_fn)(void *ptr, void *stream, void *user);

typedef struct spg_ctx spg_ctx;

/* Host-visible summary of the last spg_symbolic (for tests and benches). */
typedef struct {
    int64_t nrows;          /* rows of A (= rows of C)                          */
    int64_t flop_total;     /* sum_i flop_i                  */
    int64_t nnz_total;      /* nnz(C) = C_row_ptr[nrows]                        */
    int64_t max_row_flop;   /* max_i flop_i                                     */
    int64_t max_row_nnz;    /* max_i nnz(c_i*)                                  */
    int64_t sym_bin_rows[12]; /* rows per symbolic bin    */
    int64_t num_bin_rows[12]; /* rows per numeric bin                           */
    int64_t heap_rows;      /* rows the heap tier takes when sorted output is
                               requested (spg_set_accumulator)                  */
} spg_info;

spg_status spg_ctx_create(spg_ctx **ctx, spg_alloc_fn alloc, spg_free_fn free_fn,
                          void *user);
spg_status spg_ctx_destroy(spg_ctx *ctx);
const char *spg_last_error(const spg_ctx *ctx);
/* Number of kernels this ctx has launched so far (evidence for benches). */
int64_t spg_launch_count(const spg_ctx *ctx);

/* Per-launch timing (measurement aid; off by default).  With enable != 0
 * every kernel launch of this ctx is bracketed by two CUDA events recorded
 * on the stream that kernel runs on (internal streams included), so a bench
 * can attribute device time to kernels without a profiler.  Records persist
 * until spg_profile_reset.  spg_profile_count synchronizes on the recorded
 * events and returns their number; spg_profile_record returns the kernel
 * name (static string owned by the library) and duration in ms. */
spg_status spg_profile_enable(spg_ctx *ctx, int enable);
/* Bins on one stream (measurement aid; off by default, also set by the
 * environment variable SPG_SERIAL_BINS=1 at ctx creation).  With on != 0 the
 * per-bin kernels of the symbolic and numeric phases run one after another
 * on the caller's stream instead of on concurrent internal streams, so the
 * per-launch records of spg_profile_enable bracket one kernel each.  The
 * results are identical.  Returns SPG_ERR_INVALID_ARG for a NULL ctx. */
spg_status spg_set_serial_bins(spg_ctx *ctx, int on);
spg_status spg_profile_reset(spg_ctx *ctx);
int64_t spg_profile_count(spg_ctx *ctx);
spg_status spg_profile_record(spg_ctx *ctx, int64_t idx, const char **name, float *ms);

/* Measurement aid: 16 int64 kernel counters of the last call (host out),
 * filled only when the environment variable SPG_TUNE has bit 8 set at ctx
 * creation (per-phase clock64 sums of the column-part kernel: [0] parts,
 * [1] init+segment search, [2] scan, [3] accumulate, [4] emit clocks,
 * [5] products, [6] entries).  Zeroed by spg_symbolic.  Synchronizes
 * `stream`. */
spg_status spg_debug_counters(spg_ctx *ctx, int64_t *out, void *stream);

/* Phase 1 -- symbolic (Fig:hash_spgemm l.1-14 and "Symbolic(rpts_C, A, B)",
 * P:292-310; hashing P:283, "In symbolic phase, it is enough to insert keys",
 * P:285).  Steps, all on the GPU: per-row flop (Fig:load_balance l.1-6),
 * row binning by hash table size (lowest 2^n > min(N_col, flop)),
 * per-bin hash symbolic kernels that count nnz(c_i*), exclusive scan into
 * C_row_ptr.
 *   A, B        : device CSR, A.ncols == B.nrows; values unused.
 *   C_row_ptr   : device, caller-allocated int64[A.nrows + 1]; written with
 *                 C's row pointer, C_row_ptr[0] = 0 (C-local even for a
 *                 row-range view of A).
 *   nnz_C       : host out, nnz(C) = C_row_ptr[A.nrows].
 *   flop_total  : host out (may be NULL), sum of per-row flop.
 * Blocks the calling thread for two small device->host reads (bin counts,
 * then nnz and numeric bin counts); one more when most a_ik hit empty rows
 * of B (then the plan runs on A' = the useful a_ik of A, kept in ctx, e.g.
 * a tall-skinny frontier B).  Keeps the plan (flop, bins) in ctx for
 * spg_numeric. */
spg_status spg_symbolic(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                        int64_t *C_row_ptr, int64_t *nnz_C, int64_t *flop_total,
                        void *stream);

/* Phase 2 -- numeric ("Numeric(C, A, B)"; "In numeric phase ... we need
 * to store the resulting value data"; optional ascending sort).
 * Must follow spg_symbolic on the same ctx with the same A, B and C_row_ptr:
 * SPG_ERR_STATE if any of A.row_ptr, A.col_idx, B.row_ptr, B.col_idx,
 * C_row_ptr, A.nrows or B.ncols differs from that call (pointer identity; the
 * CONTENTS of A and B must not change in between -- not checked, since that
 * would cost a device round trip).
 *   C_col_idx, C_val : device, caller-allocated with nnz_C entries.
 *   sorted           : 0 = columns of each C row in unspecified order;
 *                      1 = strictly increasing columns in every row.
 * Asynchronous on `stream`.  Values are fp64 sums of fp64 products (order of
 * accumulation unspecified). */
spg_status spg_numeric(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                       const int64_t *C_row_ptr, int32_t *C_col_idx, double *C_val,
                       int sorted, void *stream);

/* Accumulator of the rows of C when SORTED output is requested (PAPER.md
 * §4.2.3 Heap SpGEMM P:340-352 and the cost model of §4.2.4 P:358-366;
 * SURVEY.md §8(f) row 4).  Takes effect at the next spg_symbolic (the plan
 * records which rows go where).
 *   SPG_ACCUM_AUTO (default): a row of the warp tiers (nnz(c_i) <= 512) with
 *       nnz(a_i) <= 16, flop_i <= 2048 and sorted B rows is merged by a
 *       per-thread heap when T_heap = h flop_i log2 nnz(a_i) (Eq:heap_est) is
 *       below T_hash = flop_i c + nnz(c_i) log2 nnz(c_i) (Eq:hash_est), else
 *       hashed and sorted;
 *   SPG_ACCUM_HASH: every row hashed (the heap tier never runs);
 *   SPG_ACCUM_HEAP: every row eligible as above is merged by the heap.
 *   collision_factor: c of Eq:hash_est, >= 1 (default 1.3, the measured
 *       average probes of the warp-tier tables).
 *   heap_cost: h, the cost of one heap step relative to one hash probe, > 0
 *       (default 8, measured on B200: DESIGN.md §9d; 1 = the paper's
 *       unit-cost model).
 * Unsorted output always uses the hash tiers.  Errors: SPG_ERR_INVALID_ARG. */
#define SPG_ACCUM_AUTO 0
#define SPG_ACCUM_HASH 1
#define SPG_ACCUM_HEAP 2
spg_status spg_set_accumulator(spg_ctx *ctx, int accum, double collision_factor,
                               double heap_cost);

/* One-phase multiply (§2, the
 * one-phase alternative: "allocate large enough memory space for output
 * matrix and compute").  No symbolic pass: every row's hash table is sized
 * by the flop upper bound (lowest 2^n >= 2 min(N_col, flop_i): the numeric
 * rule of reading R6 with flop_i bounding nnz(c_i)), the
 * numeric kernels run on those bins with their row counts read on the device
 * (persistent launches) and write row i into a flop-sized ctx workspace (12
 * bytes per product, grow-only) while counting nnz(c_i); a scan gives
 * C_row_ptr.  Blocks ONCE, for the 8-byte nnz(C) (plus a rerun when the
 * workspace had to grow).  Then the caller allocates C and calls
 * spg_onephase_emit, which compacts the rows into it (async).
 *   A, B        : device CSR with values; A.ncols == B.nrows.
 *   C_row_ptr   : device, caller-allocated int64[A.nrows + 1].
 *   nnz_C       : host out.   flop_total: host out (may be NULL).
 *   sorted      : 0/1 as for spg_numeric.
 * Errors: SPG_ERR_OVERFLOW when a row needs a table beyond 16384 slots
 * (min(flop_i, N_col) > 8192) -- use the two-phase calls for such
 * matrices; SPG_ERR_WORKSPACE when flop * 12 bytes cannot be allocated. */
spg_status spg_onephase(spg_ctx *ctx, const spg_csr *A, const spg_csr *B, int64_t *C_row_ptr,
                        int64_t *nnz_C, int64_t *flop_total, int sorted, void *stream);
/* Copies the rows of the last spg_onephase into C (C_col_idx int32[nnz_C],
 * C_val f64[nnz_C], device, caller-allocated; NULL allowed when nnz_C = 0).
 * Asynchronous on `stream`.  SPG_ERR_STATE without a pending spg_onephase. */
spg_status spg_onephase_emit(spg_ctx *ctx, int32_t *C_col_idx, double *C_val, void *stream);

/* Summary of the last spg_symbolic on this ctx (host struct). */
spg_status spg_get_info(const spg_ctx *ctx, spg_info *info);

/* Debug export of the last symbolic plan (device outputs, int64[A.nrows]):
 *   flop_out : per-row flop (Fig:load_balance l.1-6), may be NULL
 *   tsize_out: per-row symbolic hash table size of Fig:hash_spgemm
 *              (lowest 2^n > min(N_col, flop_i)), may be NULL.
 * Asynchronous on `stream`. */
spg_status spg_plan_export(spg_ctx *ctx, int64_t *flop_out, int64_t *tsize_out,
                           void *stream);

/* RowsToThreads on the GPU (Fig:load_balance): per-row flop of
 * A*B, prefix sum, offset[t] = lowbnd(flop_ps, floor(total*t/nparts)) for
 * t = 1..nparts-1 (lowbnd = first id with flop_ps[id] >= value),
 * offset[0] = 0, offset[nparts] = A.nrows.
 *   offsets    : HOST out, int64[nparts + 1].
 *   flop_total : HOST out (may be NULL).
 * Blocks for the small device->host read. */
spg_status spg_rows_to_parts(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                             int64_t nparts, int64_t *offsets, int64_t *flop_total,
                             void *stream);

/* Bytes-balanced split for the multi-GPU numeric phase (SURVEY.md §8(e):
 * flop balance leaves the minimal-bytes model imbalanced because nnz(C)
 * per rank differs): the RowsToThreads rule (Fig:load_balance, P:251-270;
 * lowbnd P:246) applied to the per-row bytes w_i = 16 + 12 (nnz(a_i) +
 * flop_i + nnz(c_i)) instead of flop_i.
 *   row_nnz     : device int64[A.nrows], nnz(c_i) of every row (e.g. the
 *                 differences of C_row_ptr, gathered from the ranks).
 *   offsets     : HOST out, int64[nparts + 1].  bytes_total: HOST out (may be
 *                 NULL).  Blocks for the small device->host read. */
spg_status spg_rows_to_parts_bytes(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                                   const int64_t *row_nnz, int64_t nparts, int64_t *offsets,
                                   int64_t *bytes_total, void *stream);

/* Masked sum for triangle counting (Sec 5.6; BASELINE config 5):
 * sum over stored C(i,j) with (i,j) in pattern(G) of C(i,j).  Every warp sums
 * its entries in fp64; the warp partials are reduced in int64 (exact) when
 * each is an integer below 2^53 -- integer-valued C such as the wedge counts
 * of L*U -- otherwise *sum is the fp64 total rounded to the nearest int64.  C and G rows may be in any column
 * order (G rows sorted ascending when G.ncols > 1.6M: binary search); row i
 * of C is row g_row_begin + i of G.  G's row is an smem hash set (short rows)
 * or bitmap (long rows) probed by every C entry.  Result to HOST *sum
 * (blocks for 8 bytes). */
spg_status spg_mask_sum(spg_ctx *ctx, const spg_csr *C, const spg_csr *G,
                        int64_t g_row_begin, int64_t *sum, void *stream);

/* Fused mask-and-sum (triangle counting, Sec 5.6 P:602-605;
 * SURVEY.md §8(f) row 1):  *sum = sum over (i, j) in pattern(G) of (A*B)(i, j)
 * for the rows of A, where row i of A is row g_row_begin + i of G -- computed
 * WITHOUT forming C: the columns of G's row i are the keys of the hash set
 * (bitmap for long G rows) that every product of Gustavson's row i probes;
 * matching products are summed in fp64 (exact for integer-valued inputs below
 * 2^53, e.g. the triangle count's L*U with values 1.0: triangles = *sum / 2).
 *   A, B : device CSR, values required; A.ncols == B.nrows; any column order.
 *   G    : device CSR pattern (values unused), G.ncols == B.ncols, rows
 *          strictly increasing when B.ncols > kBitmapMaxCols (binary search).
 *   sum  : host out.  Synchronizes `stream`. */
spg_status spg_masked_sum(spg_ctx *ctx, const spg_csr *A, const spg_csr *B, const spg_csr *G,
                          int64_t g_row_begin, double *sum, void *stream);

/* The same fused masked sum reduced EXACTLY in int64 (SURVEY.md §8(a) a9:
 * triangle counts are integers): every warp's fp64 partial must be an integer
 * below 2^53 (integer-valued A and B, e.g. L and U with values 1.0), and the
 * partials are added as int64.  *sum: host out.  SPG_ERR_OVERFLOW if some
 * partial is not such an integer (non-integer inputs).  Synchronizes
 * `stream`. */
spg_status spg_masked_sum_int(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                              const spg_csr *G, int64_t g_row_begin, int64_t *sum,
                              void *stream);

/* Degree-ascending relabelling for triangle counting (Sec 5.6,
 * "we reorder rows with increasing number of nonzeros.  The algorithm
 * then splits the reordered matrix A as A = L + U").
 * Untimed preprocessing in the paper.
 *   G     : device CSR, n x n pattern of a symmetric adjacency matrix WITHOUT
 *           diagonal (values unused, any column order), n and nnz(G) < 2^31.
 *   perm  : device out int32[n]: perm[r] = old id of new vertex r, the order
 *           of the keys (deg(v), v) ascending (ties by old id: unique).
 *   L_rp, L_col, L_val : device out, int64[n+1], int32[nnz(G)/2], f64[nnz(G)/2]
 *           (L_val may be NULL): L' = strict lower triangle of P G P^T.
 *   U_rp, U_col, U_val : the same for U' = strict upper triangle.
 *   G_rp, G_col, G_val : device out, int64[n+1], int32[nnz(G)], f64[nnz(G)]
 *           (G_val may be NULL): G' = P G P^T (the mask).
 * All rows of L', U', G' have strictly increasing columns; values are 1.0.
 * Buffers are caller-allocated; workspace from the ctx allocator.  Errors:
 * SPG_ERR_INVALID_ARG when nnz(G) is odd, a diagonal entry is present, or the
 * lower and upper counts differ (necessary conditions of symmetry; a
 * non-symmetric G with equal counts is not detected); SPG_ERR_OVERFLOW for
 * n or nnz >= 2^31.  Synchronizes `stream` twice (nnz(G), count check). */
spg_status spg_degree_relabel(spg_ctx *ctx, const spg_csr *G, int32_t *perm, int64_t *L_rp,
                              int32_t *L_col, double *L_val, int64_t *U_rp, int32_t *U_col,
                              double *U_val, int64_t *G_rp, int32_t *G_col, double *G_val,
                              void *stream);

/* Collision factor c of Eq:hash_est ("the average number
 * of probes") of the warp-tier numeric tables, for
 * MEASUREMENT (not on the product path).  For every row i of A with
 * 0 < 2 nnz(c_i) <= 1024, the row's products are inserted (keys only, in the
 * numeric phase's order) into a table of T = lowest 2^n >= 2 nnz(c_i) slots
 * four times: mode 0 linear probing on the high bits of col * H (the build,
 * reading R5), mode 1 linear probing on the low bits (the literal remainder),
 * mode 2 4-slot chunks (HashVector-style; a probe = one chunk),
 * mode 3 32-slot warp buckets (a probe = one bucket read by the warp).
 *   A, B      : device CSR (values unused); C_row_ptr: device int64[A.nrows+1]
 *               from spg_symbolic on the same A, B.
 *   out       : HOST int64[12]: out[3m] = probes, out[3m+1] = products,
 *               out[3m+2] = keys inserted (= sum of nnz(c_i) over those rows).
 * Synchronizes `stream`. */
spg_status spg_probe_stats(spg_ctx *ctx, const spg_csr *A, const spg_csr *B,
                           const int64_t *C_row_ptr, int64_t *out, void *stream);

/* Validation of the CSR invariants (untimed): row_ptr nondecreasing, columns
 * in [0, ncols); with check_sorted != 0 also strictly increasing columns per
 * row (which implies uniqueness).  Returns SPG_OK or SPG_ERR_INDEX_RANGE /
 * SPG_ERR_INVALID_ARG.  Blocks. */
spg_status spg_validate(spg_ctx *ctx, const spg_csr *M, int check_sorted, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SPGEMM_H_ */
