/* lcsgrid_oracle.h -- TEST INFRASTRUCTURE ONLY (see lcsgrid_oracle.c header).
 * CPU restatement of the reference lcsgrid hot path, used as the parity
 * checker for the CUDA product; never linked into the product. */
#ifndef LCSGRID_ORACLE_H
#define LCSGRID_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One CostTable of the reference recursion tree (solver.py:32-62). */
typedef struct {
    int32_t top_row, bottom_row; /* 1-based vertex rows of the slab */
    int32_t w1;                  /* table width = min(slab rows, n) + 1 */
    int32_t wstar;               /* max(kmax) */
    int32_t upper, lower;        /* child node ids, -1 for a leaf */
    int32_t *reach;              /* (n+1) x w1, row-major */
    int32_t *trace;              /* (n+1) x w1 or NULL (leaf / low-memory) */
    int32_t *kmax;               /* n+1 */
} orc_node;

typedef struct {
    int32_t m, n, inf, row_offset, with_trace;
    int32_t nnodes, cap, root;
    orc_node *nodes;
    uint64_t ncell;        /* Alg. 1 cell evaluations (reference counter) */
    uint64_t ngather;      /* evaluations that gather an L value */
    uint64_t ncombine_out; /* sum of combine output cells */
    uint64_t ncombine_in;  /* sum of (|U| + |L|) cells per combine */
} orc_tree;

int32_t orc_inf_value(int32_t n);
void orc_base_case_row(const uint8_t *cols, int32_t n, uint8_t sym, int32_t *out);
void orc_combine_level(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                       const int32_t *lower_reach, int32_t wl1, int32_t lower_wstar,
                       int32_t *out_reach, int32_t *out_trace, int32_t w1, int with_trace,
                       int32_t inf, int64_t i_lo, int64_t i_hi, int threads,
                       uint64_t *ncell_out, uint64_t *ngather_out);
/* with_trace bit 0: keep traces; bit 1: count Alg. 1 cells (C) and gathers (G) */
int orc_build(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n, int32_t top_row,
              int32_t bottom_row, int with_trace, int threads, orc_tree **out);
void orc_free(orc_tree *t);
int32_t orc_num_nodes(const orc_tree *t);
int32_t orc_root(const orc_tree *t);
const orc_node *orc_node_at(const orc_tree *t, int32_t i);
void orc_counters(const orc_tree *t, uint64_t *ncell, uint64_t *ngather, uint64_t *nout,
                  uint64_t *nin);
int orc_recover(const orc_tree *t, int32_t j, int32_t *cols_out);
int32_t orc_assemble(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n,
                     const int32_t *path, uint8_t *subseq, int32_t *row_pos, int32_t *col_pos);
int32_t orc_lcs(const uint8_t *a, int32_t la, const uint8_t *b, int32_t lb, int low_memory,
                int threads, uint8_t *subseq, int32_t *pos_a, int32_t *pos_b);

#ifdef __cplusplus
}
#endif
#endif
