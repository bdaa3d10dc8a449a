/*
 * lcsgrid_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's Lu-Liu grid-graph LCS hot path
 * (leaf tables -> recursive min-combine -> cross-vertex recovery -> assembly).
 * It exists so that tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs have a checker that travels to the GPU
 * box (where /root/reference does not exist).  Nothing in the product
 * (paper_2309_09072_b200/) links, loads or calls this file.
 *
 * Parity pin: tests/test_oracle.py checks every function below against
 *   - the SPEC known-answer examples (tests/golden/spec_examples.json),
 *   - the paper-grid golden of SURVEY.md Appendix D (tests/golden/paper_grid.npz),
 *   - whole-tree reach/trace dumps and lcs() outputs of the real reference
 *     (tests/golden/ref_trees.npz, ref_lcs.json) produced by
 *     tests/golden/make_golden.py from /root/reference,
 * and, when oracle/_ref (the reference built from /root/reference) is present,
 * against the reference itself on fresh random instances.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/lcsgrid/).
 */
#include "lcsgrid_oracle.h"

#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* seqcore.py:37-39 -- unreachable sentinel, strictly above every column index */
int32_t orc_inf_value(int32_t n) { return n + 2; }

/* breakout.py:37-55 -- base_case_row: entry i (0-based r = i-1) is
 * (min match position p >= i, 1-based) + 1, or n+2 when no such p.
 * Computed as the reference does: scatter match positions, then a reversed
 * running minimum (suffix-min); "no match" n+1 plus one lands on INF. */
void orc_base_case_row(const uint8_t *cols, int32_t n, uint8_t sym, int32_t *out) {
    int32_t nxt = n + 1;
    for (int32_t r = n - 1; r >= 0; --r) {
        if (cols[r] == sym) nxt = r + 1;
        out[r] = nxt + 1;
    }
}

/* _kernel.pyx:14-25 -- cell_value: compose "weight k above, j-k below". */
static inline int32_t cell_value(const int32_t *U, int32_t wu1, const int32_t *L, int32_t wl1,
                                 int64_t i, int32_t k, int32_t j, int32_t inf, int32_t wl) {
    (void)wl1;
    if (k > j) return inf;
    int32_t x = U[i * (int64_t)wu1 + k];
    if (x >= inf) return inf;
    if (j - k > wl) return inf;
    return L[(int64_t)(x - 1) * wl1 + (j - k)];
}

/* _kernel.pyx:28-60 -- col_mins: Alg. 1 bisection with first-wins (strict <)
 * column scan; an INF middle column fills its right part with (INF, top) and
 * recurses left with the full row range. */
static void col_mins(const int32_t *U, int32_t wu1, const int32_t *L, int32_t wl1, int64_t i,
                     int32_t left, int32_t right, int32_t top, int32_t bottom,
                     int32_t *out_reach, int32_t *out_trace, int32_t w1, int with_trace,
                     int32_t inf, int32_t wl, uint64_t *ncell, uint64_t *ngather) {
    while (right >= left) {
        int32_t mid = (left + right + 1) / 2;
        int32_t best = cell_value(U, wu1, L, wl1, i, top, mid, inf, wl);
        int32_t best_k = top;
        for (int32_t k = top + 1; k <= bottom; ++k) {
            int32_t v = cell_value(U, wu1, L, wl1, i, k, mid, inf, wl);
            if (v < best) { best = v; best_k = k; }
        }
        if (ncell) {
            *ncell += (uint64_t)(bottom - top + 1);
            /* gathers: cells that reach the L lookup (_kernel.pyx:25) */
            for (int32_t k = top; k <= bottom; ++k)
                if (k <= mid && U[i * (int64_t)wu1 + k] < inf && mid - k <= wl) ++*ngather;
        }
        out_reach[i * (int64_t)w1 + mid] = best;
        if (with_trace) out_trace[i * (int64_t)w1 + mid] = best_k;
        if (best != inf) {
            col_mins(U, wu1, L, wl1, i, left, mid - 1, top, best_k, out_reach, out_trace, w1,
                     with_trace, inf, wl, ncell, ngather);
            /* tail-call of the right half (mid+1, right, best_k, bottom) */
            left = mid + 1;
            top = best_k;
        } else {
            for (int32_t c = mid + 1; c <= right; ++c) {
                out_reach[i * (int64_t)w1 + c] = inf;
                if (with_trace) out_trace[i * (int64_t)w1 + c] = top;
            }
            right = mid - 1; /* recurse left with the full row range */
        }
    }
}

/* _kernel.pyx:63-82 -- combine_level over start columns [i_lo, i_hi). */
void orc_combine_level(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                       const int32_t *lower_reach, int32_t wl1, int32_t lower_wstar,
                       int32_t *out_reach, int32_t *out_trace, int32_t w1, int with_trace,
                       int32_t inf, int64_t i_lo, int64_t i_hi, int threads,
                       uint64_t *ncell_out, uint64_t *ngather_out) {
    const int32_t w = w1 - 1;
    const int32_t wl = wl1 - 1;
    uint64_t total = 0, gtotal = 0;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads) reduction(+ : total, gtotal)
#endif
    for (int64_t i = i_lo; i < i_hi; ++i) {
        int32_t bottom = upper_kmax[i];
        int32_t colhi = bottom + lower_wstar;
        if (colhi > w) colhi = w;
        uint64_t cnt = 0, gcnt = 0;
        col_mins(upper_reach, wu1, lower_reach, wl1, i, 0, colhi, 0, bottom, out_reach,
                 out_trace, w1, with_trace, inf, wl, ncell_out ? &cnt : NULL, &gcnt);
        total += cnt;
        gtotal += gcnt;
        for (int32_t c = colhi + 1; c <= w; ++c) {
            out_reach[i * (int64_t)w1 + c] = inf;
            if (with_trace) out_trace[i * (int64_t)w1 + c] = 0;
        }
    }
    (void)threads;
    if (ncell_out) *ncell_out += total;
    if (ngather_out) *ngather_out += gtotal;
}

/* solver.py:84-88 / :104-108 -- kmax = (reach < inf).sum(1) - 1, wstar = max. */
static int32_t fill_kmax(const int32_t *reach, int64_t n1, int32_t w1, int32_t inf, int32_t *kmax) {
    int32_t wstar = -1;
    for (int64_t i = 0; i < n1; ++i) {
        int32_t cnt = 0;
        for (int32_t j = 0; j < w1; ++j) cnt += reach[i * (int64_t)w1 + j] < inf;
        kmax[i] = cnt - 1;
        if (kmax[i] > wstar) wstar = kmax[i];
    }
    return wstar;
}

typedef struct {
    const uint8_t *rows, *cols;
    int32_t n, inf;
    int with_trace, threads, count;
    orc_tree *t;
} build_ctx;

static int32_t new_node(orc_tree *t) {
    if (t->nnodes == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 64;
        t->nodes = (orc_node *)realloc(t->nodes, (size_t)t->cap * sizeof(orc_node));
    }
    memset(&t->nodes[t->nnodes], 0, sizeof(orc_node));
    return t->nnodes++;
}

/* solver.py:72-88 -- _base_table for string row h (1-based, slab-relative
 * row index is h - row_offset). */
static int32_t base_table(build_ctx *c, int32_t h) {
    orc_tree *t = c->t;
    int32_t id = new_node(t);
    orc_node *nd = &t->nodes[id];
    const int32_t n = c->n;
    const int32_t w = n < 1 ? n : 1;
    nd->top_row = h;
    nd->bottom_row = h + 1;
    nd->w1 = w + 1;
    nd->upper = nd->lower = -1;
    nd->reach = (int32_t *)malloc((size_t)(n + 1) * (size_t)(w + 1) * sizeof(int32_t));
    nd->kmax = (int32_t *)malloc((size_t)(n + 1) * sizeof(int32_t));
    nd->trace = NULL;
    for (int32_t r = 0; r <= n; ++r) nd->reach[(int64_t)r * (w + 1)] = r + 1;
    if (w == 1) {
        int32_t *first = (int32_t *)malloc((size_t)n * sizeof(int32_t));
        orc_base_case_row(c->cols, n, c->rows[h - t->row_offset - 1], first);
        for (int32_t r = 0; r < n; ++r) nd->reach[(int64_t)r * 2 + 1] = first[r];
        nd->reach[(int64_t)n * 2 + 1] = c->inf;
        free(first);
    }
    nd->wstar = fill_kmax(nd->reach, n + 1, w + 1, c->inf, nd->kmax);
    return id;
}

/* solver.py:91-110 -- _combine_tables */
static int32_t combine_tables(build_ctx *c, int32_t up, int32_t lo) {
    orc_tree *t = c->t;
    const int32_t n = c->n;
    int32_t top = t->nodes[up].top_row, bottom = t->nodes[lo].bottom_row;
    int32_t w = bottom - top;
    if (w > n) w = n;
    int32_t id = new_node(t);
    orc_node *nd = &t->nodes[id];
    orc_node *U = &t->nodes[up], *L = &t->nodes[lo];
    nd->top_row = top;
    nd->bottom_row = bottom;
    nd->w1 = w + 1;
    nd->upper = up;
    nd->lower = lo;
    nd->reach = (int32_t *)malloc((size_t)(n + 1) * (size_t)(w + 1) * sizeof(int32_t));
    nd->trace = c->with_trace
                    ? (int32_t *)malloc((size_t)(n + 1) * (size_t)(w + 1) * sizeof(int32_t))
                    : NULL;
    nd->kmax = (int32_t *)malloc((size_t)(n + 1) * sizeof(int32_t));
    orc_combine_level(U->reach, U->w1, U->kmax, L->reach, L->w1, L->wstar, nd->reach, nd->trace,
                      nd->w1, c->with_trace, c->inf, 0, n + 1, c->threads,
                      c->count ? &t->ncell : NULL, &t->ngather);
    t->ncombine_out += (uint64_t)(n + 1) * (uint64_t)(w + 1);
    t->ncombine_in += (uint64_t)(n + 1) * (uint64_t)(U->w1 + L->w1);
    nd->wstar = fill_kmax(nd->reach, n + 1, w + 1, c->inf, nd->kmax);
    return id;
}

/* solver.py:113-119 -- _build: mid split on 1-based vertex rows. */
static int32_t build_rec(build_ctx *c, int32_t top, int32_t bottom) {
    if (bottom == top + 1) return base_table(c, top);
    int32_t mid = (top + bottom) / 2;
    int32_t up = build_rec(c, top, mid);
    int32_t lo = build_rec(c, mid, bottom);
    return combine_tables(c, up, lo);
}

/* solver.py:122-139 -- build_cost_table(g, top_row, bottom_row).
 * `rows` is the FULL row string of the grid (length m); the slab covers
 * vertex rows [top_row, bottom_row]. */
int orc_build(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n, int32_t top_row,
              int32_t bottom_row, int with_trace, int threads, orc_tree **out) {
    if (!(1 <= top_row && top_row < bottom_row && bottom_row <= m + 1)) return -1;
    orc_tree *t = (orc_tree *)calloc(1, sizeof(orc_tree));
    t->m = m;
    t->n = n;
    t->inf = orc_inf_value(n);
    t->row_offset = 0;
    t->with_trace = with_trace;
    build_ctx c = {rows, cols, n, t->inf, with_trace & 1, threads, (with_trace & 2) != 0, t};
    t->with_trace = with_trace & 1;
    t->root = build_rec(&c, top_row, bottom_row);
    *out = t;
    return 0;
}

void orc_free(orc_tree *t) {
    if (!t) return;
    for (int32_t i = 0; i < t->nnodes; ++i) {
        free(t->nodes[i].reach);
        free(t->nodes[i].trace);
        free(t->nodes[i].kmax);
    }
    free(t->nodes);
    free(t);
}

int32_t orc_num_nodes(const orc_tree *t) { return t->nnodes; }
int32_t orc_root(const orc_tree *t) { return t->root; }
const orc_node *orc_node_at(const orc_tree *t, int32_t i) { return &t->nodes[i]; }
void orc_counters(const orc_tree *t, uint64_t *ncell, uint64_t *ngather, uint64_t *nout,
                  uint64_t *nin) {
    *ncell = t->ncell;
    *ngather = t->ngather;
    *nout = t->ncombine_out;
    *nin = t->ncombine_in;
}

/* monotone.py:46-63 -- compose_cell on one upper row. */
static int32_t compose_cell(const int32_t *urow, int32_t wu1, const int32_t *L, int32_t wl1,
                            int32_t k, int32_t j, int32_t inf) {
    int32_t x = k < wu1 ? urow[k] : inf;
    if (x >= inf) return inf;
    int32_t d = j - k;
    if (d >= wl1) return inf;
    return L[(int64_t)(x - 1) * wl1 + d];
}

/* solver.py:165-177 -- _retrace: brute-force first-wins split. */
static int32_t retrace(const orc_tree *t, const orc_node *nd, int32_t i, int32_t j) {
    const orc_node *U = &t->nodes[nd->upper], *L = &t->nodes[nd->lower];
    const int32_t *urow = U->reach + (int64_t)(i - 1) * U->w1;
    int32_t hi = U->kmax[i - 1];
    if (j < hi) hi = j;
    int32_t best = t->inf, best_k = 0;
    for (int32_t k = 0; k <= hi; ++k) {
        int32_t v = compose_cell(urow, U->w1, L->reach, L->w1, k, j, t->inf);
        if (v < best) { best = v; best_k = k; }
    }
    return best_k;
}

/* solver.py:180-207 -- recover_cross_vertices (walk). */
static void walk(const orc_tree *t, int32_t id, int32_t i, int32_t jj, int32_t *cols) {
    for (;;) {
        const orc_node *nd = &t->nodes[id];
        if (nd->bottom_row == nd->top_row + 1) {
            cols[nd->top_row - 1] = i;
            return;
        }
        int32_t k = nd->trace ? nd->trace[(int64_t)(i - 1) * nd->w1 + jj] : retrace(t, nd, i, jj);
        const orc_node *U = &t->nodes[nd->upper];
        int32_t x = U->reach[(int64_t)(i - 1) * U->w1 + k];
        walk(t, nd->upper, i, k, cols);
        id = nd->lower;
        i = x;
        jj = jj - k;
    }
}

int orc_recover(const orc_tree *t, int32_t j, int32_t *cols_out) {
    const orc_node *root = &t->nodes[t->root];
    if (!(root->top_row == 1 && root->bottom_row == t->m + 1)) return -1;
    if (j > root->kmax[0]) return -2;
    walk(t, t->root, 1, j, cols_out);
    cols_out[t->m] = root->reach[j];
    return 0;
}

/* solver.py:210-234 -- assemble_lcs: mark rows entering the next grid row
 * strictly to the right through a matching diagonal, then compact. */
int32_t orc_assemble(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n,
                     const int32_t *path, uint8_t *subseq, int32_t *row_pos, int32_t *col_pos) {
    if (m == 0 || n == 0) return 0;
    int32_t len = 0;
    for (int32_t r = 0; r < m; ++r) {
        int64_t prev = path[r], cur = path[r + 1];
        int64_t land = cur - 2;
        if (land < 0) land = 0;
        if (land > n - 1) land = n - 1;
        if (cur > prev && rows[r] == cols[land]) {
            subseq[len] = rows[r];
            row_pos[len] = r + 1;
            col_pos[len] = (int32_t)(cur - 1);
            ++len;
        }
    }
    return len;
}

/* solver.py:237-273 -- lcs(a, b): orientation swap (rows = shorter, tie keeps
 * a as rows), build, length, recover, assemble, un-swap.  Output buffers must
 * hold min(la, lb) entries. */
int32_t orc_lcs(const uint8_t *a, int32_t la, const uint8_t *b, int32_t lb, int low_memory,
                int threads, uint8_t *subseq, int32_t *pos_a, int32_t *pos_b) {
    if (la == 0 || lb == 0) return 0;
    int swapped = la > lb;
    const uint8_t *rows = swapped ? b : a, *cols = swapped ? a : b;
    int32_t m = swapped ? lb : la, n = swapped ? la : lb;
    orc_tree *t = NULL;
    if (orc_build(rows, m, cols, n, 1, m + 1, !low_memory, threads, &t) != 0) return -1;
    int32_t length = t->nodes[t->root].kmax[0];
    int32_t *path = (int32_t *)malloc((size_t)(m + 1) * sizeof(int32_t));
    orc_recover(t, length, path);
    int32_t *rp = swapped ? pos_b : pos_a, *cp = swapped ? pos_a : pos_b;
    int32_t len = orc_assemble(rows, m, cols, n, path, subseq, rp, cp);
    free(path);
    orc_free(t);
    return len;
}
