/*
 * oracle/auxamg_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded restatement of the reference auxamg setup + solve
 * path (arXiv 1209.5421 auxiliary-grid AMG), used as the parity checker for
 * the CUDA product in paper_1209_5421_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links or calls this file.
 *
 * Pinning: tests/test_oracle.py checks every exported structure and every
 * solve result of this restatement bitwise against oracle/_ref (the reference
 * headers compiled unmodified from /root/reference, see oracle/Makefile) and
 * against the committed golden fixtures in tests/golden/.
 *
 * Every function cites the reference function it restates
 * (/root/reference/proj/include/auxamg/<file>:<lines>).  Floating-point
 * operations are issued in the reference's order; build with -ffp-contract=off
 * so no FMA is formed (the reference's Release build on x86-64 never forms one,
 * CMakeLists.txt:4-10).
 *
 * The C ABI mirrors include/auxamg_b200.h with an orc_ prefix.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/auxamg_b200.h"

/* ------------------------------------------------------------------ errors */

typedef struct {
    jmp_buf jb;
    int code;
    char msg[512];
} Err;

static void fail(Err* e, int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(e->msg, sizeof e->msg, fmt, ap);
    va_end(ap);
    e->code = code;
    longjmp(e->jb, 1);
}

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) abort();
    return p;
}

/* ------------------------------------------------------------------ types */

typedef struct { int n_rows, n_cols; int* row_ptr; int* col_idx; double* values; long nnz; } Csr;
typedef struct { int n_rows, width; int* col; double* val; } Ell;          /* sparse.hpp:25-54 */
typedef struct { int level, n_agg, n; int *agg_of, *member_ptr, *member_idx; } Agg; /* auxgrid.hpp:41-52 */
typedef struct { int n; double* lu; int* perm; } Lu;                        /* dense.hpp:48-68 */

typedef struct {                                                           /* hierarchy.hpp:288-299 */
    int k, structured, n;
    long nnz;
    Csr csr;
    Ell ell;
    int has_map;
    Agg map;
    unsigned char* active;
    int n_items;
    int* item_color;
    int* groups[4];
    int group_len[4];
    Lu* blocks;        /* per aggregate (finest) */
    int* block_size;
    int n_blocks;
} Level;

struct orc_hierarchy {                                                     /* hierarchy.hpp:301-309 */
    double a1, b1, a2, b2;
    int depth;
    int n_levels;
    Level lv[AUX_MAX_LEVELS];
    Lu coarsest;
    aux_locality loc;
    aux_setup_opts opts;
};
typedef struct orc_hierarchy orc_hierarchy;

/* ------------------------------------------------------ parallel.hpp:86-119 */

/* dot: 1024-element sequential blocks + fixed pairwise tree, parallel.hpp:88-112.
 * ORC_BLK != 1024 builds a sensitivity variant (tests only: it measures how
 * far the reference's own results move under a different summation order). */
#ifndef ORC_BLK
#define ORC_BLK 1024
#endif
static double dot(const double* a, const double* b, size_t n) {
    const size_t blk = ORC_BLK;
    size_t nb = (n + blk - 1) / blk;
    if (nb <= 1) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    double* part = (double*)xcalloc(nb, sizeof(double));
    for (size_t k = 0; k < nb; ++k) {
        size_t lo = k * blk, hi = lo + blk < n ? lo + blk : n;
        double s = 0.0;
        for (size_t i = lo; i < hi; ++i) s += a[i] * b[i];
        part[k] = s;
    }
    size_t m = nb;
    while (m > 1) {
        size_t half = m / 2;
        for (size_t i = 0; i < half; ++i) part[i] = part[2 * i] + part[2 * i + 1];
        if (m % 2 == 1) part[half] = part[m - 1];
        m = half + m % 2;
    }
    double r = part[0];
    free(part);
    return r;
}
static double norm2(const double* v, size_t n) { return sqrt(dot(v, v, n)); } /* :114 */
static void axpy(double alpha, const double* x, double* y, size_t n) {      /* :117-119 */
    for (size_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* -------------------------------------------------------- sparse.hpp */

/* validate_csr, sparse.hpp:101-116 (row_ptr length is implied by the view) */
static void validate_csr(Err* e, const Csr* A) {
    if (A->row_ptr[0] != 0 || (long)A->row_ptr[A->n_rows] != A->nnz)
        fail(e, AUX_STRUCTURE_ERROR, "CSR row_ptr endpoints inconsistent with nnz");
    for (int r = 0; r < A->n_rows; ++r) {
        if (A->row_ptr[r] > A->row_ptr[r + 1])
            fail(e, AUX_STRUCTURE_ERROR, "CSR row_ptr not nondecreasing at row %d", r);
        for (int p = A->row_ptr[r]; p < A->row_ptr[r + 1]; ++p) {
            if (A->col_idx[p] < 0 || A->col_idx[p] >= A->n_cols)
                fail(e, AUX_STRUCTURE_ERROR, "CSR column index out of range in row %d", r);
            if (p > A->row_ptr[r] && A->col_idx[p - 1] >= A->col_idx[p])
                fail(e, AUX_STRUCTURE_ERROR, "CSR row %d not sorted by column", r);
        }
    }
}

/* CsrMatrix::at, sparse.hpp:67-73 (lower_bound within the row) */
static double csr_at(const Csr* A, int r, int c) {
    int lo = A->row_ptr[r], hi = A->row_ptr[r + 1];
    while (lo < hi) {
        int mid = lo + (hi - lo) / 2;
        if (A->col_idx[mid] < c) lo = mid + 1; else hi = mid;
    }
    if (lo == A->row_ptr[r + 1] || A->col_idx[lo] != c) return 0.0;
    return A->values[lo];
}

/* symmetry_defect, sparse.hpp:238-260.  Restated without the explicit
 * transpose: every stored (i,j) pairs with (j,i) if present.  The set of
 * |differences| is identical and max is order-free. */
static double symmetry_defect(const Csr* A) {
    if (A->n_rows != A->n_cols) return INFINITY;
    double scale = 1.0, defect = 0.0;
    for (long p = 0; p < A->nnz; ++p) scale = dmax(scale, fabs(A->values[p]));
    for (int i = 0; i < A->n_rows; ++i)
        for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
            int j = A->col_idx[p];
            int lo = A->row_ptr[j], hi = A->row_ptr[j + 1];
            while (lo < hi) {
                int mid = lo + (hi - lo) / 2;
                if (A->col_idx[mid] < i) lo = mid + 1; else hi = mid;
            }
            if (lo < A->row_ptr[j + 1] && A->col_idx[lo] == i)
                defect = dmax(defect, fabs(A->values[p] - A->values[lo]));
            else
                defect = dmax(defect, fabs(A->values[p]));
        }
    return defect / scale;
}

/* csr_spmv, sparse.hpp:141-150 */
static void csr_spmv(const Csr* A, const double* x, double* y) {
    for (int r = 0; r < A->n_rows; ++r) {
        double s = 0.0;
        for (int p = A->row_ptr[r]; p < A->row_ptr[r + 1]; ++p) s += A->values[p] * x[A->col_idx[p]];
        y[r] = s;
    }
}

/* ell_spmv, sparse.hpp:120-132 */
static void ell_spmv(const Ell* A, const double* x, double* y) {
    for (int r = 0; r < A->n_rows; ++r) {
        double s = 0.0;
        for (int t = 0; t < A->width; ++t) {
            int c = A->col[(size_t)t * A->n_rows + r];
            if (c != -1) s += A->val[(size_t)t * A->n_rows + r] * x[c];
        }
        y[r] = s;
    }
}

/* -------------------------------------------------------- dense.hpp */

/* lu_factor, dense.hpp:76-102 (in place on a row-major n x n array) */
static int lu_factor(double* a, int* perm, int n, int* zero_col) {
    for (int i = 0; i < n; ++i) perm[i] = i;
    for (int k = 0; k < n; ++k) {
        int piv = k;
        double best = fabs(a[(size_t)k * n + k]);
        for (int r = k + 1; r < n; ++r) {
            double m = fabs(a[(size_t)r * n + k]);
            if (m > best) { best = m; piv = r; }
        }
        if (best == 0.0) { *zero_col = k; return 0; }
        if (piv != k) {
            for (int c = 0; c < n; ++c) {
                double t = a[(size_t)k * n + c];
                a[(size_t)k * n + c] = a[(size_t)piv * n + c];
                a[(size_t)piv * n + c] = t;
            }
            int t = perm[k]; perm[k] = perm[piv]; perm[piv] = t;
        }
        for (int r = k + 1; r < n; ++r) {
            double m = a[(size_t)r * n + k] / a[(size_t)k * n + k];
            a[(size_t)r * n + k] = m;
            for (int c = k + 1; c < n; ++c) a[(size_t)r * n + c] -= m * a[(size_t)k * n + c];
        }
    }
    return 1;
}

/* LuFactors::solve, dense.hpp:52-67 */
static void lu_solve(const Lu* f, const double* b, double* x) {
    const int n = f->n;
    for (int i = 0; i < n; ++i) x[i] = b[f->perm[i]];
    for (int i = 1; i < n; ++i) {
        double s = x[i];
        for (int j = 0; j < i; ++j) s -= f->lu[(size_t)i * n + j] * x[j];
        x[i] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int j = i + 1; j < n; ++j) s -= f->lu[(size_t)i * n + j] * x[j];
        x[i] = s / f->lu[(size_t)i * n + i];
    }
}

/* -------------------------------------------------------- auxgrid.hpp */

/* choose_depth, auxgrid.hpp:95-104 */
int orc_choose_depth(long n, int* depth) {
    if (n < 4) return AUX_ARGUMENT_ERROR;
    int level = 0;
    long cells = 1;
    while (cells * 4 < n) { cells *= 4; ++level; }
    *depth = level == 0 ? 1 : level;
    return AUX_OK;
}

/* subregion_of_point, auxgrid.hpp:109-121 */
static int subregion(Err* e, double x, double y, const orc_hierarchy* g, int k) {
    if (!isfinite(x) || !isfinite(y) || x < g->a1 || x > g->b1 || y < g->a2 || y > g->b2)
        fail(e, AUX_GEOMETRY_ERROR, "point (%f, %f) outside bounding box", x, y);
    const double w = (double)(1 << k);
    const double below_one = 1.0 - 2.220446049250313e-16 / 2;
    const double sx = dmin((x - g->a1) / (g->b1 - g->a1), below_one);
    const double sy = dmin((y - g->a2) / (g->b2 - g->a2), below_one);
    const int t1 = (int)(sx * w), t2 = (int)(sy * w);
    return t2 * (1 << k) + t1;
}
int orc_subregion_of_point(double x, double y, const double box[4], int k, int* cell) {
    Err e;
    orc_hierarchy g;
    g.a1 = box[0]; g.b1 = box[1]; g.a2 = box[2]; g.b2 = box[3];
    if (setjmp(e.jb)) return e.code;
    *cell = subregion(&e, x, y, &g, k);
    return AUX_OK;
}

/* build_members (counting sort, members ascending), auxgrid.hpp:58-70 */
static void build_members(Agg* m) {
    m->member_ptr = (int*)xcalloc((size_t)m->n_agg + 1, sizeof(int));
    m->member_idx = (int*)xcalloc((size_t)m->n, sizeof(int));
    for (int j = 0; j < m->n; ++j) ++m->member_ptr[m->agg_of[j] + 1];
    for (int i = 0; i < m->n_agg; ++i) m->member_ptr[i + 1] += m->member_ptr[i];
    int* next = (int*)xcalloc((size_t)m->n_agg + 1, sizeof(int));
    memcpy(next, m->member_ptr, sizeof(int) * (size_t)m->n_agg);
    for (int j = 0; j < m->n; ++j) m->member_idx[next[m->agg_of[j]]++] = j;
    free(next);
}

/* bounding_box, auxgrid.hpp:75-91 */
static void bounding_box(Err* e, const double* xy, long n, orc_hierarchy* g) {
    if (n <= 0) fail(e, AUX_ARGUMENT_ERROR, "bounding_box: no points");
    g->a1 = g->b1 = xy[0];
    g->a2 = g->b2 = xy[1];
    for (long i = 0; i < n; ++i) {
        double x = xy[2 * i], y = xy[2 * i + 1];
        if (!isfinite(x) || !isfinite(y)) fail(e, AUX_ARGUMENT_ERROR, "bounding_box: non-finite coordinate");
        g->a1 = dmin(g->a1, x); g->b1 = dmax(g->b1, x);
        g->a2 = dmin(g->a2, y); g->b2 = dmax(g->b2, y);
    }
    if (!(g->b1 > g->a1) || !(g->b2 > g->a2)) fail(e, AUX_GEOMETRY_ERROR, "bounding_box: degenerate point set");
}

/* aggregate_coarse, auxgrid.hpp:138-150 */
static void aggregate_coarse(int k, Agg* m) {
    const int w = 1 << k;
    m->level = k;
    m->n_agg = 1 << (2 * (k - 1));
    m->n = w * w;
    m->agg_of = (int*)xcalloc((size_t)m->n, sizeof(int));
    for (int t2 = 0; t2 < w; ++t2)
        for (int t1 = 0; t1 < w; ++t1) m->agg_of[t2 * w + t1] = (t2 / 2) * (w / 2) + t1 / 2;
    build_members(m);
}

/* color_of, auxgrid.hpp:154-160 */
static int color_of(int i, int k) {
    const int w = 1 << k;
    return (i % w) % 2 + 2 * ((i / w) % 2);
}

/* -------------------------------------------------------- smoother.hpp */

/* make_schedule, smoother.hpp:41-54 */
static void make_schedule(Level* lv, int k, const unsigned char* active) {
    const int n = 1 << (2 * k);
    lv->n_items = n;
    lv->item_color = (int*)xcalloc((size_t)n, sizeof(int));
    for (int c = 0; c < 4; ++c) { lv->groups[c] = (int*)xcalloc((size_t)n, sizeof(int)); lv->group_len[c] = 0; }
    for (int i = 0; i < n; ++i) {
        lv->item_color[i] = -1;
        if (!active[i]) continue;
        int c = color_of(i, k);
        lv->item_color[i] = c;
        lv->groups[c][lv->group_len[c]++] = i;
    }
}

/* point_gs_sweep (ELL), smoother.hpp:68-89 */
static void point_gs_ell(Err* e, const Ell* A, const double* b, double* x, const Level* lv, int dir) {
    for (int c = 0; c < 4; ++c)
        for (int q = 0; q < lv->group_len[c]; ++q) {
            int i = lv->groups[c][q];
            if (A->val[i] == 0.0) fail(e, AUX_SINGULAR_ERROR, "zero diagonal at row %d", i);
        }
    for (int s = 0; s < 4; ++s) {
        const int c = dir == 0 ? s : 3 - s;
        for (int q = 0; q < lv->group_len[c]; ++q) {
            const int i = lv->groups[c][q];
            double sum = b[i];
            for (int t = 1; t < A->width; ++t) {
                int j = A->col[(size_t)t * A->n_rows + i];
                if (j != -1) sum -= A->val[(size_t)t * A->n_rows + i] * x[j];
            }
            x[i] = sum / A->val[i];
        }
    }
}

/* factor_blocks, smoother.hpp:129-156 */
static void factor_blocks(Err* e, const Csr* A, const Agg* agg, Level* lv) {
    lv->n_blocks = agg->n_agg;
    lv->blocks = (Lu*)xcalloc((size_t)agg->n_agg, sizeof(Lu));
    lv->block_size = (int*)xcalloc((size_t)agg->n_agg, sizeof(int));
    for (int g = 0; g < agg->n_agg; ++g) {
        const int* mem = agg->member_idx + agg->member_ptr[g];
        const int s = agg->member_ptr[g + 1] - agg->member_ptr[g];
        lv->block_size[g] = s;
        if (s == 0) continue;
        double* blk = (double*)xcalloc((size_t)s * s, sizeof(double));
        for (int q = 0; q < s; ++q) {
            const int i = mem[q];
            for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
                int lo = 0, hi = s, c = A->col_idx[p];
                while (lo < hi) { int mid = lo + (hi - lo) / 2; if (mem[mid] < c) lo = mid + 1; else hi = mid; }
                if (lo < s && mem[lo] == c) blk[(size_t)q * s + lo] = A->values[p];
            }
        }
        int* perm = (int*)xcalloc((size_t)s, sizeof(int));
        int zc;
        lv->blocks[g].n = s; lv->blocks[g].lu = blk; lv->blocks[g].perm = perm;
        if (!lu_factor(blk, perm, s, &zc))
            fail(e, AUX_DEFINITENESS_ERROR, "aggregate %d has a singular block", g);
    }
}

/* block_gs_sweep, smoother.hpp:162-205 */
static void block_gs(const Level* lv, const double* b, double* x, int dir) {
    const Csr* A = &lv->csr;
    const Agg* agg = &lv->map;
    double* xp = (double*)xcalloc((size_t)A->n_rows, sizeof(double));
    double *r = NULL, *d = NULL;
    int cap = 0;
    for (int s = 0; s < 4; ++s) {
        const int c = dir == 0 ? s : 3 - s;
        if (lv->group_len[c] == 0) continue;
        memcpy(xp, x, sizeof(double) * (size_t)A->n_rows);
        for (int q = 0; q < lv->group_len[c]; ++q) {
            const int g = lv->groups[c][q];
            const int* mem = agg->member_idx + agg->member_ptr[g];
            const int sz = agg->member_ptr[g + 1] - agg->member_ptr[g];
            if (sz == 1) {
                const int i = mem[0];
                double diag = 0.0, sum = b[i];
                for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
                    int j = A->col_idx[p];
                    if (j == i) diag = A->values[p]; else sum -= A->values[p] * xp[j];
                }
                x[i] = sum / diag;
                continue;
            }
            if (sz > cap) { free(r); free(d); cap = sz; r = (double*)xcalloc((size_t)cap, 8); d = (double*)xcalloc((size_t)cap, 8); }
            for (int qq = 0; qq < sz; ++qq) {
                const int i = mem[qq];
                double sum = b[i];
                for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) sum -= A->values[p] * xp[A->col_idx[p]];
                r[qq] = sum;
            }
            lu_solve(&lv->blocks[g], r, d);
            for (int qq = 0; qq < sz; ++qq) x[mem[qq]] = xp[mem[qq]] + d[qq];
        }
    }
    free(xp); free(r); free(d);
}

/* -------------------------------------------------------- hierarchy.hpp */

static const int stencil_off[8][2] = {{1, 0}, {1, 1}, {0, 1}, {-1, 1}, {-1, 0}, {-1, -1}, {0, -1}, {1, -1}};

/* stencil_slot, hierarchy.hpp:53-57 */
static int stencil_slot(int dx, int dy) {
    static const int table[9] = {6, 7, 8, 5, 0, 1, 4, 3, 2};
    if (dx < -1 || dx > 1 || dy < -1 || dy > 1) return -1;
    return table[3 * (dy + 1) + (dx + 1)];
}

/* build_stencil_indices + preset_stencil, hierarchy.hpp:75-91, 121-131 */
static void preset_stencil(Ell* op, int k, const unsigned char* active) {
    const int w = 1 << k, n = w * w;
    op->n_rows = n; op->width = 9;
    op->col = (int*)xcalloc((size_t)n * 9, sizeof(int));
    op->val = (double*)xcalloc((size_t)n * 9, sizeof(double));
    for (size_t i = 0; i < (size_t)n * 9; ++i) op->col[i] = -1;
    for (int i = 0; i < n; ++i) {
        const int t1 = i % w, t2 = i / w;
        op->col[i] = i;
        for (int s = 0; s < 8; ++s) {
            int u1 = t1 + stencil_off[s][0], u2 = t2 + stencil_off[s][1];
            if (u1 < 0 || u1 >= w || u2 < 0 || u2 >= w) continue;
            op->col[(size_t)(s + 1) * n + i] = u2 * w + u1;
        }
    }
    for (int r = 0; r < n; ++r) {
        if (active[r]) continue;
        for (int t = 1; t < 9; ++t) op->col[(size_t)t * n + r] = -1;
        op->val[r] = 1.0;
    }
}

static long ell_nnz(const Ell* op) {
    long c = 0;
    for (size_t i = 0; i < (size_t)op->n_rows * op->width; ++i) c += op->col[i] != -1;
    return c;
}

/* assemble_coarse_finest, hierarchy.hpp:141-192 (+ active_from_members :94-98) */
static void assemble_coarse_finest(Err* e, const Csr* A, const Agg* agg, const aux_setup_opts* o,
                                   Ell* op, unsigned char** active_out, aux_locality* loc) {
    int k = 0;
    while ((1 << (2 * k)) < agg->n_agg) ++k;
    const int w = 1 << k, n = agg->n_agg;
    unsigned char* active = (unsigned char*)xcalloc((size_t)n, 1);
    for (int i = 0; i < n; ++i) active[i] = agg->member_ptr[i + 1] > agg->member_ptr[i];
    preset_stencil(op, k, active);
    long* rd = (long*)xcalloc((size_t)n, sizeof(long));
    double* rm = (double*)xcalloc((size_t)n, sizeof(double));
    const int lump = o->lump_locality && !o->strict_locality;
    for (int r = 0; r < n; ++r) {
        if (!active[r]) continue;
        const int t1 = r % w, t2 = r / w;
        for (int m = agg->member_ptr[r]; m < agg->member_ptr[r + 1]; ++m) {
            const int i = agg->member_idx[m];
            for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p) {
                const double a = A->values[p];
                const int q = agg->agg_of[A->col_idx[p]];
                const int slot = stencil_slot(q % w - t1, q / w - t2);
                if (slot < 0) {
                    if (lump) op->val[r] += a;
                    ++rd[r];
                    rm[r] += fabs(a);
                    continue;
                }
                op->val[(size_t)slot * n + r] += a;
            }
        }
    }
    memset(loc, 0, sizeof *loc);
    for (int r = 0; r < n; ++r) {
        if (rd[r] == 0) continue;
        if (lump) { loc->lumped += rd[r]; loc->lumped_mass += rm[r]; }
        else { loc->dropped += rd[r]; loc->dropped_mass += rm[r]; }
    }
    free(rd); free(rm);
    if (o->strict_locality && loc->dropped > 0)
        fail(e, AUX_STRUCTURE_ERROR, "strict locality: %ld couplings fall outside the 9-point stencil", (long)loc->dropped);
    *active_out = active;
}

/* assemble_coarse_structured + coarsen_active, hierarchy.hpp:198-235, 101-109 */
static void assemble_coarse_structured(Err* e, const Ell* An, const Agg* agg, const unsigned char* act_n,
                                       Ell* op, unsigned char** active_out) {
    int kc = 0;
    while ((1 << (2 * kc)) < agg->n_agg) ++kc;
    const int wc = 1 << kc, nc = agg->n_agg;
    unsigned char* active = (unsigned char*)xcalloc((size_t)nc, 1);
    for (int j = 0; j < agg->n; ++j) if (act_n[j]) active[agg->agg_of[j]] = 1;
    preset_stencil(op, kc, active);
    for (int r = 0; r < nc; ++r) {
        if (!active[r]) continue;
        const int t1 = r % wc, t2 = r / wc;
        for (int m = agg->member_ptr[r]; m < agg->member_ptr[r + 1]; ++m) {
            const int i = agg->member_idx[m];
            if (!act_n[i]) continue;
            for (int t = 0; t < An->width; ++t) {
                const int j = An->col[(size_t)t * An->n_rows + i];
                if (j == -1) continue;
                const int q = agg->agg_of[j];
                const int slot = stencil_slot(q % wc - t1, q / wc - t2);
                if (slot < 0) fail(e, AUX_STRUCTURE_ERROR, "4-child coarsening escaped the 9-point stencil at row %d", r);
                op->val[(size_t)slot * nc + r] += An->val[(size_t)t * An->n_rows + i];
            }
        }
    }
    *active_out = active;
}

static void free_level(Level* lv) {
    free(lv->csr.row_ptr); free(lv->csr.col_idx); free(lv->csr.values);
    free(lv->ell.col); free(lv->ell.val);
    free(lv->map.agg_of); free(lv->map.member_ptr); free(lv->map.member_idx);
    free(lv->active); free(lv->item_color);
    for (int c = 0; c < 4; ++c) free(lv->groups[c]);
    if (lv->blocks) for (int g = 0; g < lv->n_blocks; ++g) { free(lv->blocks[g].lu); free(lv->blocks[g].perm); }
    free(lv->blocks); free(lv->block_size);
}

void orc_destroy(orc_hierarchy* h) {
    if (!h) return;
    for (int i = 0; i < AUX_MAX_LEVELS; ++i) free_level(&h->lv[i]);
    free(h->coarsest.lu); free(h->coarsest.perm);
    free(h);
}

static void dense_lu(Err* e, double* a, int n, Lu* out) {
    out->n = n; out->lu = a; out->perm = (int*)xcalloc((size_t)n, sizeof(int));
    int zc;
    if (!lu_factor(a, out->perm, n, &zc)) fail(e, AUX_SINGULAR_ERROR, "lu_factor: zero pivot at column %d", zc);
}

/* setup_hierarchy, hierarchy.hpp:315-386 */
int orc_setup(const aux_csr_view* Av, const double* xy, int64_t n_points, const aux_setup_opts* opts_in,
              orc_hierarchy** out, char* msg, size_t msg_len) {
    Err e;
    orc_hierarchy* h = (orc_hierarchy*)xcalloc(1, sizeof(orc_hierarchy));
    *out = NULL;
    if (setjmp(e.jb)) {
        if (msg && msg_len) snprintf(msg, msg_len, "%s", e.msg);
        orc_destroy(h);
        return e.code;
    }
    aux_setup_opts opts = *opts_in;
    h->a1 = 0.0; h->b1 = 1.0; h->a2 = 0.0; h->b2 = 1.0; h->depth = 1;   /* AuxGrid defaults, auxgrid.hpp:30-37 */
    Csr A = {Av->n_rows, Av->n_cols, (int*)Av->row_ptr, (int*)Av->col_idx, (double*)Av->values, (long)Av->nnz};
    if (A.n_rows != A.n_cols) fail(&e, AUX_SIZE_ERROR, "setup_hierarchy: matrix not square");
    if (n_points != A.n_rows) fail(&e, AUX_SIZE_ERROR, "setup_hierarchy: coordinate count does not match matrix order");
    validate_csr(&e, &A);
    for (int r = 0; r < A.n_rows; ++r)
        if (csr_at(&A, r, r) <= 0.0) fail(&e, AUX_DEFINITENESS_ERROR, "nonpositive diagonal at row %d", r);
    if (symmetry_defect(&A) > opts.symmetry_tol) fail(&e, AUX_STRUCTURE_ERROR, "matrix is not symmetric to tolerance");
    if (opts.coarsest_size < 4) opts.coarsest_size = 4;
    h->opts = opts;
    const int n = A.n_rows;

    Level* fine = &h->lv[0];
    fine->structured = 0;
    fine->n = n;
    fine->csr = A;
    fine->csr.row_ptr = (int*)xcalloc((size_t)n + 1, sizeof(int));
    fine->csr.col_idx = (int*)xcalloc((size_t)A.nnz, sizeof(int));
    fine->csr.values = (double*)xcalloc((size_t)A.nnz, sizeof(double));
    memcpy(fine->csr.row_ptr, A.row_ptr, sizeof(int) * ((size_t)n + 1));
    memcpy(fine->csr.col_idx, A.col_idx, sizeof(int) * (size_t)A.nnz);
    memcpy(fine->csr.values, A.values, sizeof(double) * (size_t)A.nnz);
    fine->nnz = A.nnz;
    fine->active = (unsigned char*)xcalloc((size_t)n, 1);
    memset(fine->active, 1, (size_t)n);
    h->n_levels = 1;

    if (n <= opts.coarsest_size) {                                 /* :339-344 */
        fine->k = 0;
        double* d = (double*)xcalloc((size_t)n * n, sizeof(double));
        for (int r = 0; r < n; ++r)
            for (int p = A.row_ptr[r]; p < A.row_ptr[r + 1]; ++p) d[(size_t)r * n + A.col_idx[p]] = A.values[p];
        dense_lu(&e, d, n, &h->coarsest);
        *out = h;
        return AUX_OK;
    }

    bounding_box(&e, xy, n, h);                                    /* :346-347 */
    int depth;
    if (orc_choose_depth(n, &depth) != AUX_OK) fail(&e, AUX_ARGUMENT_ERROR, "choose_depth: need at least 4 DoFs");
    h->depth = depth;
    fine->k = depth + 1;
    fine->has_map = 1;                                             /* aggregate_finest, auxgrid.hpp:124-133 */
    fine->map.level = depth;
    fine->map.n_agg = 1 << (2 * depth);
    fine->map.n = n;
    fine->map.agg_of = (int*)xcalloc((size_t)n, sizeof(int));
    for (int j = 0; j < n; ++j) fine->map.agg_of[j] = subregion(&e, xy[2 * j], xy[2 * j + 1], h, depth);
    build_members(&fine->map);
    factor_blocks(&e, &A, &fine->map, fine);

    Level* cur = &h->lv[1];
    unsigned char* top_active;
    assemble_coarse_finest(&e, &A, &fine->map, &opts, &cur->ell, &top_active, &h->loc);
    make_schedule(fine, depth, top_active);
    cur->k = depth;
    cur->structured = 1;
    cur->n = 1 << (2 * depth);
    cur->active = top_active;
    make_schedule(cur, depth, cur->active);
    h->n_levels = 2;

    while (cur->k > 0 && cur->n > opts.coarsest_size) {            /* :366-381 */
        const int k = cur->k;
        cur->has_map = 1;
        aggregate_coarse(k, &cur->map);
        if (h->n_levels >= AUX_MAX_LEVELS) fail(&e, AUX_INTERNAL_ERROR, "too many levels");
        Level* nx = &h->lv[h->n_levels];
        assemble_coarse_structured(&e, &cur->ell, &cur->map, cur->active, &nx->ell, &nx->active);
        cur->nnz = ell_nnz(&cur->ell);
        nx->k = k - 1;
        nx->structured = 1;
        nx->n = 1 << (2 * (k - 1));
        make_schedule(nx, k - 1, nx->active);
        h->n_levels++;
        cur = nx;
    }
    cur->nnz = ell_nnz(&cur->ell);
    {                                                              /* dense_from_ell + lu_factor :383 */
        const int nc = cur->n;
        double* d = (double*)xcalloc((size_t)nc * nc, sizeof(double));
        for (int r = 0; r < nc; ++r)
            for (int t = 0; t < 9; ++t) {
                int c = cur->ell.col[(size_t)t * nc + r];
                if (c != -1) d[(size_t)r * nc + c] = cur->ell.val[(size_t)t * nc + r];
            }
        dense_lu(&e, d, nc, &h->coarsest);
    }
    *out = h;
    return AUX_OK;
}

/* -------------------------------------------------------- cycle.hpp */

typedef struct {                 /* DirectionWindow, cycle.hpp:60-76 */
    double** p;
    double** ap;
    double* energy;
    int size, cap_alloc, capacity;
} Dirs;

static void dirs_free(Dirs* d) {
    for (int i = 0; i < d->size; ++i) { free(d->p[i]); free(d->ap[i]); }
    free(d->p); free(d->ap); free(d->energy);
    memset(d, 0, sizeof *d);
}

/* next_direction, cycle.hpp:84-97; takes ownership of z, az */
static double next_direction(Dirs* d, double* z, double* az, size_t m) {
    for (int j = 0; j < d->size; ++j) {
        const double beta = -dot(z, d->ap[j], m) / d->energy[j];
        axpy(beta, d->p[j], z, m);
        axpy(beta, d->ap[j], az, m);
    }
    const double energy = dot(z, az, m);
    if (!(energy > 1e-300)) { free(z); free(az); return 0.0; }
    if (d->size == d->cap_alloc) {
        d->cap_alloc = d->cap_alloc ? 2 * d->cap_alloc : 8;
        d->p = (double**)realloc(d->p, sizeof(double*) * (size_t)d->cap_alloc);
        d->ap = (double**)realloc(d->ap, sizeof(double*) * (size_t)d->cap_alloc);
        d->energy = (double*)realloc(d->energy, sizeof(double) * (size_t)d->cap_alloc);
    }
    d->p[d->size] = z; d->ap[d->size] = az; d->energy[d->size] = energy; d->size++;
    if (d->capacity > 0 && d->size > d->capacity) {
        free(d->p[0]); free(d->ap[0]);
        memmove(d->p, d->p + 1, sizeof(double*) * (size_t)(d->size - 1));
        memmove(d->ap, d->ap + 1, sizeof(double*) * (size_t)(d->size - 1));
        memmove(d->energy, d->energy + 1, sizeof(double) * (size_t)(d->size - 1));
        d->size--;
    }
    return energy;
}

static void apply_level(const Level* lv, const double* x, double* y) {     /* cycle.hpp:132-137 */
    if (lv->structured) ell_spmv(&lv->ell, x, y); else csr_spmv(&lv->csr, x, y);
}

static void smooth_level(Err* e, const Level* lv, const double* b, double* x, int sweeps, int dir) { /* :139-147 */
    for (int s = 0; s < sweeps; ++s) {
        if (lv->structured) point_gs_ell(e, &lv->ell, b, x, lv, dir);
        else block_gs(lv, b, x, dir);
    }
}

static void amli_cycle(Err* e, const orc_hierarchy* h, int l, const double* f, double* u, const aux_cycle_opts* o);

/* nonlinear_pcg, cycle.hpp:106-128, with apply = level l, precond = amli_cycle(l) */
static void nonlinear_pcg(Err* e, const orc_hierarchy* h, int l, const double* f, int nsteps, double* u,
                          const aux_cycle_opts* o) {
    const size_t m = (size_t)h->lv[l].n;
    memset(u, 0, sizeof(double) * m);
    double* r = (double*)xcalloc(m, sizeof(double));
    memcpy(r, f, sizeof(double) * m);
    Dirs d;
    memset(&d, 0, sizeof d);
    for (int i = 0; i < nsteps; ++i) {
        double* z = (double*)xcalloc(m, sizeof(double));
        double* az = (double*)xcalloc(m, sizeof(double));
        amli_cycle(e, h, l, r, z, o);
        apply_level(&h->lv[l], z, az);
        const double energy = next_direction(&d, z, az, m);
        if (energy == 0.0) break;
        const double* p = d.p[d.size - 1];
        const double* ap = d.ap[d.size - 1];
        const double alpha = dot(r, p, m) / energy;
        axpy(alpha, p, u, m);
        axpy(-alpha, ap, r, m);
    }
    dirs_free(&d);
    free(r);
}

/* amli_cycle, cycle.hpp:161-197 */
static void amli_cycle(Err* e, const orc_hierarchy* h, int l, const double* f, double* u, const aux_cycle_opts* o) {
    const Level* lv = &h->lv[l];
    if (l == h->n_levels - 1) { lu_solve(&h->coarsest, f, u); return; }
    const size_t n = (size_t)lv->n;
    memset(u, 0, sizeof(double) * n);
    smooth_level(e, lv, f, u, o->pre_sweeps, 0);
    double* au = (double*)xcalloc(n, sizeof(double));
    apply_level(lv, u, au);
    double* r = (double*)xcalloc(n, sizeof(double));
    for (size_t i = 0; i < n; ++i) r[i] = f[i] - au[i];
    const Agg* agg = &lv->map;                                             /* restrict, hierarchy.hpp:267-277 */
    double* rc = (double*)xcalloc((size_t)agg->n_agg, sizeof(double));
    for (int i = 0; i < agg->n_agg; ++i) {
        double s = 0.0;
        for (int m = agg->member_ptr[i]; m < agg->member_ptr[i + 1]; ++m) s += r[agg->member_idx[m]];
        rc[i] = s;
    }
    double* ec = (double*)xcalloc((size_t)agg->n_agg, sizeof(double));
    nonlinear_pcg(e, h, l + 1, rc, o->n_inner, ec, o);
    for (size_t i = 0; i < n; ++i)                                         /* prolongate + masked add :191-194 */
        if (lv->active[i]) u[i] += ec[agg->agg_of[i]];
    smooth_level(e, lv, f, u, o->post_sweeps, 1);
    free(au); free(r); free(rc); free(ec);
}

/* solve, cycle.hpp:202-247 */
int orc_solve(orc_hierarchy* h, const aux_csr_view* Av, const double* b, int64_t n_b, const aux_cycle_opts* o,
              aux_solve_result* res, char* msg, size_t msg_len) {
    Err e;
    double *r = NULL, *u = NULL;
    Dirs d;
    memset(&d, 0, sizeof d);
    if (setjmp(e.jb)) {
        if (msg && msg_len) snprintf(msg, msg_len, "%s", e.msg);
        free(r); free(u); dirs_free(&d);
        return e.code;
    }
    if (o->n_inner < 1 || o->pre_sweeps < 1 || o->post_sweeps < 1 || o->max_outer < 1)
        fail(&e, AUX_ARGUMENT_ERROR, "cycle options must be positive");
    if (!(o->rtol > 0.0) || !(o->rtol < 1.0)) fail(&e, AUX_ARGUMENT_ERROR, "rtol must lie in (0,1)");
    if (o->max_directions < 0) fail(&e, AUX_ARGUMENT_ERROR, "max_directions must be >= 0");
    Csr A = h->lv[0].csr;
    if (Av) { A.n_rows = Av->n_rows; A.n_cols = Av->n_cols; A.row_ptr = (int*)Av->row_ptr; A.col_idx = (int*)Av->col_idx; A.values = (double*)Av->values; A.nnz = (long)Av->nnz; }
    if (n_b != A.n_rows) fail(&e, AUX_SIZE_ERROR, "solve: right-hand side does not match matrix");
    if (h->n_levels < 1 || h->lv[0].n != A.n_rows) fail(&e, AUX_SIZE_ERROR, "solve: hierarchy was built for a different order");
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const size_t n = (size_t)A.n_rows;
    u = (double*)xcalloc(n, sizeof(double));
    res->iterations = 0; res->converged = 0; res->history_len = 0;
    const double norm_b = norm2(b, n);
#define PUSH_HIST(v) do { if (res->history_len < res->history_capacity) res->residual_history[res->history_len] = (v); res->history_len++; } while (0)
    PUSH_HIST(norm_b);
    if (norm_b != 0.0) {
        r = (double*)xcalloc(n, sizeof(double));
        memcpy(r, b, sizeof(double) * n);
        d.capacity = o->max_directions;
        while (res->iterations < o->max_outer) {
            double* z = (double*)xcalloc(n, sizeof(double));
            double* az = (double*)xcalloc(n, sizeof(double));
            amli_cycle(&e, h, 0, r, z, o);
            csr_spmv(&A, z, az);
            const double energy = next_direction(&d, z, az, n);
            if (energy == 0.0) break;
            const double* p = d.p[d.size - 1];
            const double* ap = d.ap[d.size - 1];
            const double alpha = dot(r, p, n) / energy;
            axpy(alpha, p, u, n);
            axpy(-alpha, ap, r, n);
            res->iterations++;
            const double rn = norm2(r, n);
            PUSH_HIST(rn);
            if (rn <= o->rtol * norm_b) { res->converged = 1; break; }
        }
    } else {
        res->converged = 1;
    }
#undef PUSH_HIST
    clock_gettime(CLOCK_MONOTONIC, &t1);
    res->solve_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    res->total_seconds = res->solve_seconds;
    res->setup_seconds = 0.0;
    if (res->u) memcpy(res->u, u, sizeof(double) * n);
    free(r); free(u); dirs_free(&d);
    return AUX_OK;
}

/* -------------------------------------------------------- exports */

int orc_n_levels(const orc_hierarchy* h) { return h->n_levels; }

int orc_grid(const orc_hierarchy* h, double box[4], int32_t* depth) {
    box[0] = h->a1; box[1] = h->b1; box[2] = h->a2; box[3] = h->b2;
    *depth = h->depth;
    return AUX_OK;
}

int orc_locality(const orc_hierarchy* h, aux_locality* out) { *out = h->loc; return AUX_OK; }

/* stats, hierarchy.hpp:395-406 */
int orc_stats(const orc_hierarchy* h, aux_stats_out* s) {
    long total = 0;
    s->levels = h->n_levels;
    for (int i = 0; i < h->n_levels; ++i) {
        s->sizes[i] = h->lv[i].n;
        s->nnz[i] = h->lv[i].nnz;
        total += h->lv[i].nnz;
    }
    s->operator_complexity = (double)total / (double)h->lv[0].nnz;
    return AUX_OK;
}

int orc_level_info_get(const orc_hierarchy* h, int32_t l, aux_level_info* o) {
    if (l < 0 || l >= h->n_levels) return AUX_ARGUMENT_ERROR;
    const Level* lv = &h->lv[l];
    memset(o, 0, sizeof *o);
    o->k = lv->k; o->structured = lv->structured; o->n = lv->n; o->nnz = lv->nnz;
    o->has_map = lv->has_map; o->map_level = lv->map.level; o->n_aggregates = lv->map.n_agg;
    o->n_items = lv->n_items;
    long pool = 0;
    for (int g = 0; g < lv->n_blocks; ++g) pool += (long)lv->block_size[g] * lv->block_size[g];
    o->block_pool = pool;
    return AUX_OK;
}

int orc_export_level(const orc_hierarchy* h, int32_t l, aux_level_export* x) {
    if (l < 0 || l >= h->n_levels) return AUX_ARGUMENT_ERROR;
    const Level* lv = &h->lv[l];
    const size_t n = (size_t)lv->n;
    if (lv->has_map) {
        if (x->agg_of) memcpy(x->agg_of, lv->map.agg_of, 4 * n);
        if (x->member_ptr) memcpy(x->member_ptr, lv->map.member_ptr, 4 * ((size_t)lv->map.n_agg + 1));
        if (x->member_idx) memcpy(x->member_idx, lv->map.member_idx, 4 * n);
    }
    if (x->active) memcpy(x->active, lv->active, n);
    if (x->item_color && lv->n_items) memcpy(x->item_color, lv->item_color, 4 * (size_t)lv->n_items);
    if (lv->structured) {
        if (x->ell_col) memcpy(x->ell_col, lv->ell.col, 4 * 9 * n);
        if (x->ell_val) memcpy(x->ell_val, lv->ell.val, 8 * 9 * n);
    }
    if (lv->blocks) {
        long off = 0, poff = 0;
        for (int g = 0; g < lv->n_blocks; ++g) {
            const int s = lv->block_size[g];
            if (x->block_size) x->block_size[g] = s;
            if (x->block_offset) x->block_offset[g] = off;
            if (s && x->block_lu) memcpy(x->block_lu + off, lv->blocks[g].lu, 8 * (size_t)s * s);
            if (s && x->block_perm) memcpy(x->block_perm + poff, lv->blocks[g].perm, 4 * (size_t)s);
            off += (long)s * s;
            poff += s;
        }
        if (x->block_offset) x->block_offset[lv->n_blocks] = off;
    }
    return AUX_OK;
}

int orc_export_coarsest(const orc_hierarchy* h, int32_t* n, double* lu, int32_t* perm) {
    *n = h->coarsest.n;
    if (lu) memcpy(lu, h->coarsest.lu, 8 * (size_t)h->coarsest.n * h->coarsest.n);
    if (perm) memcpy(perm, h->coarsest.perm, 4 * (size_t)h->coarsest.n);
    return AUX_OK;
}

/* ------------------------------------------------- kernel-level hooks (KATs) */

/* One point_gs_sweep on a 9-wide column-major ELL (smoother.hpp:68-89), all
 * rows active, schedule from color_of on level k. */
int orc_point_gs_sweep_ell(int k, const int* col, const double* val, const double* b, double* x, int dir,
                           char* msg, size_t msg_len) {
    Err e;
    Level lv;
    memset(&lv, 0, sizeof lv);
    unsigned char* act = (unsigned char*)xcalloc((size_t)1 << (2 * k), 1);
    memset(act, 1, (size_t)1 << (2 * k));
    make_schedule(&lv, k, act);
    Ell A = {1 << (2 * k), 9, (int*)col, (double*)val};
    if (setjmp(e.jb)) {
        if (msg && msg_len) snprintf(msg, msg_len, "%s", e.msg);
        free(act); free(lv.item_color); for (int c = 0; c < 4; ++c) free(lv.groups[c]);
        return e.code;
    }
    point_gs_ell(&e, &A, b, x, &lv, dir);
    free(act); free(lv.item_color); for (int c = 0; c < 4; ++c) free(lv.groups[c]);
    return AUX_OK;
}

double orc_dot(const double* a, const double* b, int64_t n) { return dot(a, b, (size_t)n); }

/* galerkin_dense (hierarchy.hpp:239-247): C(agg(i), agg(j)) += a_ij over rows
 * i ascending, then the row's entries in storage order, into a zeroed
 * n_agg x n_agg row-major matrix.  Returns AUX_SIZE_ERROR when the map does
 * not match the matrix (hierarchy.hpp:240-241). */
int orc_galerkin_dense(const aux_csr_view* A, const int32_t* agg_of, int64_t n_agg_of, int32_t n_agg, double* C) {
    if (n_agg_of != A->n_rows) return AUX_SIZE_ERROR;
    memset(C, 0, sizeof(double) * (size_t)n_agg * (size_t)n_agg);
    for (int i = 0; i < A->n_rows; ++i)
        for (int p = A->row_ptr[i]; p < A->row_ptr[i + 1]; ++p)
            C[(size_t)agg_of[i] * n_agg + agg_of[A->col_idx[p]]] += A->values[p];
    return AUX_OK;
}
