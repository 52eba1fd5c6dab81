/*
 * spa_oracle.c -- TEST INFRASTRUCTURE ONLY.  NOT part of the product path.
 *
 * Plain, slow, obviously-correct CPU reference for the hash-SpGEMM hot path of
 * Nagasaka, Matsuoka, Azad, Buluc, "High-performance sparse matrix-matrix
 * products on Intel KNL and multicore architectures" (arXiv:1804.01698).
 * Citations "P:n" are lines of /root/reference/PAPER.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header,
 * table or constant with paper_1804_01698_b200/ (the CUDA path) and never
 * includes or links it.
 *
 * What it computes (each function cites the passage it follows):
 *   oracle_flop            -- Fig:load_balance l.1-6, flop def P:137
 *   oracle_table_size      -- Fig:hash_spgemm l.5-13
 *   oracle_rows_to_threads -- Fig:load_balance l.7-14, lowbnd P:246
 *   oracle_symbolic        -- row nnz of C = A*B (Fig:code_spgemm P:106-126)
 *   oracle_numeric         -- Gustavson with a dense SPA (Fig:code_spgemm)
 *   oracle_mask_sum        -- sum of C o G over the pattern of G (triangle
 *                             counting, Sec 5.6; the mask/count step
 *                             is BASELINE config 5's statement)
 *
 * Arithmetic: fp64, one rounding per multiply and one per add, canonical order
 * (a_ik in stored order, then b_kj in stored order).  Compile with
 * -ffp-contract=off so no FMA is formed.
 *
 * Threads: rows are independent, so an optional OpenMP loop over rows
 * changes no value.  Each thread owns its SPA (dense value vector + marker +
 * touched list).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* flop[i] = sum over stored a_ik of nnz(b_k*)
 * Returns the total.  flop_out may be NULL. */
int64_t oracle_flop(int64_t m, const int64_t *a_rp, const int32_t *a_col,
                    const int64_t *b_rp, int64_t *flop_out)
{
    int64_t total = 0;
    for (int64_t i = 0; i < m; ++i) {
        int64_t f = 0;
        for (int64_t j = a_rp[i]; j < a_rp[i + 1]; ++j) {
            int64_t k = a_col[j];
            int64_t rnz = b_rp[k + 1] - b_rp[k];
            f += rnz;
        }
        if (flop_out) flop_out[i] = f;
        total += f;
    }
    return total;
}

/* Hash table size of Fig:hash_spgemm:
 *   size <- min(N_col, size);  size <- lowest_p2(size)  with
 *   "Return minimum 2^n so that 2^n > size_t"  (strictly greater). */
int64_t oracle_table_size(int64_t flop, int64_t ncols)
{
    int64_t s = flop < ncols ? flop : ncols;
    int64_t p = 1;
    while (p <= s) p <<= 1;
    return p;
}

/* lowbnd(vec, value): "the minimum id such that vec[id] is larger than or
 * equal to value".  Linear scan: obviously correct, slow. */
static int64_t lowbnd(const int64_t *vec, int64_t len, int64_t value)
{
    for (int64_t id = 0; id < len; ++id)
        if (vec[id] >= value) return id;
    return len;
}

/* RowsToThreads given flop_ps (exclusive prefix, length m+1).
 * offset[0] = 0; offset[tid] = lowbnd(flop_ps, ave_flop * tid); offset[tnum] = m.
 * ave_flop * tid is taken as floor(sum * tid / tnum) in integers (reading R12). */
void oracle_rows_to_threads(int64_t m, const int64_t *flop_ps, int64_t tnum,
                            int64_t *offset)
{
    int64_t sum = flop_ps[m];
    offset[0] = 0;
    for (int64_t tid = 1; tid < tnum; ++tid) {
        /* floor(sum*tid/tnum) without 64-bit overflow for sum < 2^62 */
        int64_t target = (int64_t)(((__int128)sum * tid) / tnum);
        offset[tid] = lowbnd(flop_ps, m + 1, target);
    }
    offset[tnum] = m;
}

typedef struct {
    double  *acc;      /* dense value vector, length ncols         */
    int64_t *mark;     /* mark[j] == i  <=>  j already in row i    */
    int32_t *touched;  /* list of column ids present in current row */
} spa_t;

static int spa_alloc(spa_t *s, int64_t ncols)
{
    size_t n = (size_t)(ncols > 0 ? ncols : 1);
    s->acc = (double *)malloc(n * sizeof(double));
    s->mark = (int64_t *)malloc(n * sizeof(int64_t));
    s->touched = (int32_t *)malloc(n * sizeof(int32_t));
    if (!s->acc || !s->mark || !s->touched) return -1;
    for (size_t j = 0; j < n; ++j) s->mark[j] = -1;
    return 0;
}

static void spa_free(spa_t *s)
{
    free(s->acc); free(s->mark); free(s->touched);
}

static int cmp_i32(const void *x, const void *y)
{
    int32_t a = *(const int32_t *)x, b = *(const int32_t *)y;
    return (a > b) - (a < b);
}

/* Row i of Fig:code_spgemm into the SPA; returns nnz(c_i*).
 * "if c_ij not in c_i*: insert(c_ij <- value) else c_ij <- c_ij + value". */
static int64_t spa_row(spa_t *s, int64_t i, const int64_t *a_rp,
                       const int32_t *a_col, const double *a_val,
                       const int64_t *b_rp, const int32_t *b_col,
                       const double *b_val)
{
    int64_t nt = 0;
    for (int64_t jj = a_rp[i]; jj < a_rp[i + 1]; ++jj) {
        int64_t k = a_col[jj];
        double aik = a_val ? a_val[jj] : 0.0;
        for (int64_t q = b_rp[k]; q < b_rp[k + 1]; ++q) {
            int32_t j = b_col[q];
            if (s->mark[j] != i) {                /* c_ij not in c_i*      */
                s->mark[j] = i;
                s->touched[nt++] = j;
                if (a_val) s->acc[j] = aik * b_val[q];     /* insert      */
            } else if (a_val) {
                double value = aik * b_val[q];
                s->acc[j] = s->acc[j] + value;             /* accumulate  */
            }
        }
    }
    return nt;
}

static int oracle_threads(int nthreads)
{
#ifdef _OPENMP
    return nthreads > 0 ? nthreads : omp_get_max_threads();
#else
    (void)nthreads;
    return 1;
#endif
}

/* Symbolic: row_nnz[i - row_begin] = nnz(c_i*) for i in [row_begin, row_end).
 * Returns 0, or -1 on allocation failure. */
int oracle_symbolic(int64_t ncols_c, const int64_t *a_rp, const int32_t *a_col,
                    const int64_t *b_rp, const int32_t *b_col,
                    int64_t row_begin, int64_t row_end, int64_t *row_nnz,
                    int nthreads)
{
    int err = 0;
    int nt = oracle_threads(nthreads);
#pragma omp parallel num_threads(nt) reduction(| : err)
    {
        spa_t s;
        if (spa_alloc(&s, ncols_c) != 0) {
            err = 1;
        } else {
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = row_begin; i < row_end; ++i)
                row_nnz[i - row_begin] =
                    spa_row(&s, i, a_rp, a_col, NULL, b_rp, b_col, NULL);
        }
        spa_free(&s);
    }
    return err ? -1 : 0;
}

/* Numeric: rows [row_begin, row_end) of C, columns sorted ascending,
 * written at c_rp[i - row_begin] .. c_rp[i - row_begin + 1]  (c_rp is the
 * caller's local row pointer for the block, c_rp[0] may be 0).
 * Returns 0; -1 on allocation failure; -2 if a row's count disagrees with
 * c_rp. */
int oracle_numeric(int64_t ncols_c, const int64_t *a_rp, const int32_t *a_col,
                   const double *a_val, const int64_t *b_rp,
                   const int32_t *b_col, const double *b_val,
                   int64_t row_begin, int64_t row_end, const int64_t *c_rp,
                   int32_t *c_col, double *c_val, int nthreads)
{
    int err = 0;
    int nt = oracle_threads(nthreads);
#pragma omp parallel num_threads(nt) reduction(| : err)
    {
        spa_t s;
        if (spa_alloc(&s, ncols_c) != 0) {
            err |= 1;
        } else {
#pragma omp for schedule(dynamic, 64)
            for (int64_t i = row_begin; i < row_end; ++i) {
                int64_t r = i - row_begin;
                int64_t n = spa_row(&s, i, a_rp, a_col, a_val, b_rp, b_col, b_val);
                if (n != c_rp[r + 1] - c_rp[r]) { err |= 2; continue; }
                qsort(s.touched, (size_t)n, sizeof(int32_t), cmp_i32);
                for (int64_t t = 0; t < n; ++t) {
                    int32_t j = s.touched[t];
                    c_col[c_rp[r] + t] = j;
                    c_val[c_rp[r] + t] = s.acc[j];
                }
            }
        }
        spa_free(&s);
    }
    if (err & 1) return -1;
    if (err & 2) return -2;
    return 0;
}

/* Sum over (i, j) in the pattern of G of C(i, j), for rows [row_begin,
 * row_end) of C (block-local c_rp), each C value converted to int64 (the
 * values are exact integers when L, U are 0/1 matrices).  The triangle count
 * is this sum / 2 (BASELINE config 5).  G columns need not be sorted; C
 * columns must be sorted (as produced by oracle_numeric).  Binary search is a
 * lookup, not arithmetic of the method. */
int64_t oracle_mask_sum(int64_t row_begin, int64_t row_end, const int64_t *c_rp,
                        const int32_t *c_col, const double *c_val,
                        const int64_t *g_rp, const int32_t *g_col)
{
    int64_t sum = 0;
    for (int64_t i = row_begin; i < row_end; ++i) {
        int64_t r = i - row_begin;
        int64_t lo0 = c_rp[r], hi0 = c_rp[r + 1];
        for (int64_t q = g_rp[i]; q < g_rp[i + 1]; ++q) {
            int32_t j = g_col[q];
            int64_t lo = lo0, hi = hi0;
            while (lo < hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (c_col[mid] < j) lo = mid + 1; else hi = mid;
            }
            if (lo < hi0 && c_col[lo] == j) sum += (int64_t)c_val[lo];
        }
    }
    return sum;
}
