/*
 * lcsgrid_b200.h -- C-ABI of the B200-native Lu-Liu grid-graph LCS hot path.
 *
 * Plain pointers and sizes only (no torch / numpy types).  Every entry point
 * replaces one interface of the reference Python package `lcsgrid`
 * (/root/reference/pkg/src/lcsgrid/, cited as file:line below); the Python
 * mirror in paper_2309_09072_b200/ binds these with ctypes exactly as
 * INTEGRATION.md shows.  All calls return LCSG_OK (0) or a negative status;
 * lcsg_last_error() then describes the failure (thread-local).
 *
 * Threading: every call is re-entrant for distinct handles; ctypes releases
 * the GIL around each call (the reference released it in _kernel.pyx:71).
 */
#ifndef LCSGRID_B200_H
#define LCSGRID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCSG_OK 0
#define LCSG_EINVAL (-1)   /* precondition violated (reference: AssertionError/ValueError) */
#define LCSG_ECUDA (-2)    /* CUDA runtime / launch failure */
#define LCSG_ENOMEM (-3)   /* device allocation failed */
#define LCSG_ENODEV (-4)   /* no CUDA device */
#define LCSG_ERANGE (-5)   /* recovery weight exceeds the LCS length (solver.py:192-193) */

/* build flags */
#define LCSG_WITH_TRACE 1u /* store split weights (solver.py:94-96, with_trace=True) */

typedef struct lcsg_tree_s *lcsg_handle;

/* Last error message of the calling thread ("" if none). */
const char *lcsg_last_error(void);
/* ABI version (major*100 + minor). */
int lcsg_abi_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int lcsg_device_count(void);

/*
 * Build the whole reach-table tree of the slab of vertex rows
 * [top_row, bottom_row] of the grid (rows[0..m), cols[0..n)), on `device`.
 * Replaces solver.build_cost_table (solver.py:122-139) together with the
 * recursion (_build :113-119), the leaf (_base_table :72-88, base_case_row
 * breakout.py:37-55) and every combine (_combine_tables :91-110 ->
 * backend.combine_level, _kernel.pyx:63-82).  Inputs are HOST buffers; the
 * solve is enqueued on `stream` (cudaStream_t, NULL = the library's own
 * stream) and the call returns once it is enqueued.
 * Preconditions (AssertionError in the reference, solver.py:137):
 *   1 <= top_row < bottom_row <= m + 1.
 */
int lcsg_build(const uint8_t *rows, int64_t m, const uint8_t *cols, int64_t n, int32_t top_row,
               int32_t bottom_row, uint32_t flags, int device, void *stream, lcsg_handle *out);

/* Same with DEVICE-resident row/column strings (no host copy). */
int lcsg_build_device(const uint8_t *rows_dev, int64_t m, const uint8_t *cols_dev, int64_t n,
                      int32_t top_row, int32_t bottom_row, uint32_t flags, int device,
                      void *stream, lcsg_handle *out);

/* Release every device buffer of the tree (back to the library's private
 * stream-ordered pool, which keeps them for the next solve). */
int lcsg_free(lcsg_handle h);
/* Return the unused blocks of the library's memory pool on `device` to the
 * driver (after lcsg_free of the trees; no reference counterpart -- the
 * reference frees numpy arrays with the CostTable, solver.py:52-53). */
int lcsg_trim(int device);
/* Grow the library's pool on `device` by `bytes` now (physical memory mapped
 * at start-up rather than inside the first large solve, whose arena would
 * otherwise pay for it -- ~0.2 s for a 16384^2 solve's 34 GB). */
int lcsg_reserve(int device, int64_t bytes);
/* Wait for all work enqueued on the handle's stream. */
int lcsg_sync(lcsg_handle h);

/* ---- CostTable access (solver.py:32-62) ---------------------------------- */
int32_t lcsg_num_nodes(lcsg_handle h);
int32_t lcsg_root(lcsg_handle h);
/* info[0..7] = top_row, bottom_row, w1 (table width), upper, lower (-1 for a
 * leaf), has_trace, n, inf */
int lcsg_node_info(lcsg_handle h, int32_t node, int32_t *info);
/* wstar of the node (solver.py:88,108) */
int lcsg_node_wstar(lcsg_handle h, int32_t node, int32_t *wstar);
/* Copy the (n+1) x w1 int32 reach table / int32 trace table / (n+1) kmax of a
 * node to HOST memory (row-major, byte-identical to the reference arrays). */
int lcsg_node_reach(lcsg_handle h, int32_t node, int32_t *host_out);
int lcsg_node_trace(lcsg_handle h, int32_t node, int32_t *host_out);
int lcsg_node_kmax(lcsg_handle h, int32_t node, int32_t *host_out);
/* Device pointer of a node's reach table (materialises leaves on demand). */
int lcsg_node_reach_device(lcsg_handle h, int32_t node, void **dev_ptr);

/* ---- extraction (solver.py:160-234) ------------------------------------- */
/* lcs_length (solver.py:160-162): kmax[0] of the root table. */
int lcsg_length(lcsg_handle h, int32_t *length);
/* recover_cross_vertices (solver.py:180-207): device walk of the tree for
 * weight j from start column 1; writes m+1 int32 to HOST memory.
 * LCSG_EINVAL unless the handle holds the full grid (:190-191),
 * LCSG_ERANGE if j > length (:192-193). */
int lcsg_recover(lcsg_handle h, int32_t j, int32_t *cols_out);
/* recover + assemble_lcs (solver.py:210-234) on the device for weight j.
 * Outputs (HOST): *length, subseq[len], row_pos[len], col_pos[len]; buffers
 * must hold min(m, n) entries.  Positions are 1-based in rows / cols. */
int lcsg_extract(lcsg_handle h, int32_t j, int32_t *length, uint8_t *subseq, int32_t *row_pos,
                 int32_t *col_pos);

/* assemble_lcs (solver.py:210-234) for a caller-supplied path (HOST m+1). */
int lcsg_assemble(const uint8_t *rows, int64_t m, const uint8_t *cols, int64_t n,
                  const int32_t *path, int device, int32_t *length, uint8_t *subseq,
                  int32_t *row_pos, int32_t *col_pos);

/* One-shot lcs(a, b) (solver.py:237-273): orientation swap, build, length,
 * recover, assemble, un-swap.  HOST in/out; pos_a / pos_b index a and b
 * (1-based).  Buffers must hold min(la, lb) entries. */
int lcsg_lcs(const uint8_t *a, int64_t la, const uint8_t *b, int64_t lb, uint32_t flags,
             int device, void *stream, int32_t *length, uint8_t *subseq, int32_t *pos_a,
             int32_t *pos_b);

/* Same with DEVICE-resident a / b; results still land in HOST buffers. */
int lcsg_lcs_device(const uint8_t *a_dev, int64_t la, const uint8_t *b_dev, int64_t lb,
                    uint32_t flags, int device, void *stream, int32_t *length, uint8_t *subseq,
                    int32_t *pos_a, int32_t *pos_b);

/* Batched lcs() of `npairs` pairs of EQUAL shape (many
 * small pairs, e.g. cfg4's planted queries): a / b hold the pairs back to back
 * (la / lb bytes each, HOST; _device: DEVICE).  All pairs' recursion trees are
 * built together -- one launch per tree height for the whole batch -- then one
 * walk and one assembly.  Pair p's results: lengths[p], subseq / pos_a / pos_b
 * + p * min(la, lb) (buffers hold npairs * min(la, lb) entries).  Each pair's
 * result is exactly lcs(a_p, b_p) (solver.py:237-273). */
int lcsg_lcs_batch(const uint8_t *a, int64_t la, const uint8_t *b, int64_t lb, int32_t npairs,
                   uint32_t flags, int device, void *stream, int32_t *lengths, uint8_t *subseq,
                   int32_t *pos_a, int32_t *pos_b);
int lcsg_lcs_batch_device(const uint8_t *a_dev, int64_t la, const uint8_t *b_dev, int64_t lb,
                          int32_t npairs, uint32_t flags, int device, void *stream,
                          int32_t *lengths, uint8_t *subseq, int32_t *pos_a, int32_t *pos_b);

/* ---- kernel-level mirrors, for fixture parity ---------------------------- */
/* combine_level (_kernel.pyx:63-82) on DEVICE buffers: start columns
 * [i_lo, i_hi) of one slab pair; tables row-major with widths wu1/wl1/w1 and
 * n1 rows. */
int lcsg_combine_level(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                       const int32_t *lower_reach, int32_t wl1, int32_t lower_wstar,
                       int32_t *out_reach, int32_t *out_trace, int32_t w1, int with_trace,
                       int32_t inf, int64_t n1, int64_t i_lo, int64_t i_hi, void *stream);
/* base_case_row (breakout.py:37-55) on DEVICE buffers: out[0..n). */
int lcsg_base_case_row(const uint8_t *cols_dev, int64_t n, uint8_t sym, int32_t *out_dev,
                       void *stream);

/* ---- multi-GPU building blocks -------------------------- */
/* Rows [i_lo, i_hi) of one combine (_combine_tables, solver.py:91-110) with the
 * fast exact kernels, on DEVICE tables of n1 rows: U/L reach (+kmax) in,
 * reach/trace/kmax rows [i_lo, i_hi) out; *out_wstar (device int32, caller
 * zero-initialises) is atomicMax'ed with the window's kmax.  Lets ranks shard
 * an upper-level combine over start columns.  Asynchronous on `stream`. */
int lcsg_combine_rows(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                      const int32_t *lower_reach, int32_t wl1, const int32_t *lower_kmax,
                      int32_t lower_wstar, int32_t *out_reach, int32_t *out_trace,
                      int32_t *out_kmax, int32_t *out_wstar, int32_t w1, int32_t inf, int64_t n1,
                      int64_t i_lo, int64_t i_hi, void *stream);
/* The recovery walk (solver.py:180-207) of a handle's slab from start column
 * i_start (1-based) for weight j: writes the slab's m_slab+1 cross-vertex
 * columns to HOST memory (a band sub-tree's share of the full-grid path). */
int lcsg_recover_from(lcsg_handle h, int32_t i_start, int32_t j, int32_t *cols_out);

/* ---- instrumentation ----------------------------------------------------- */
/* Number of kernels the library launched on this handle (for bench
 * gpu_launches); time (ms, CUDA events on the handle stream) spent in the
 * combine kernels / leaf step if the handle was built with LCSG_TIMING;
 * host<->device bytes the handle copied (inputs + plan metadata / results). */
#define LCSG_TIMING 2u
int lcsg_stats(lcsg_handle h, int64_t *launches, double *combine_ms, double *leaf_ms,
               double *total_ms, int64_t *h2d_bytes, int64_t *d2h_bytes);

/* Measured INT32 min issue rate of `device` (R_INT32 of the combine
 * roofline): independent IMNMX.U32 chains on every SM, best
 * of 5 timed launches.  *mins_per_s = 32-bit min operations per second. */
int lcsg_probe_int32_rate(int device, double *mins_per_s, int32_t *sm_count, double *ms);

/* Consistency violations counted by the row-sweep kernels on `device`
 * (lcsg_sweep.cu: every generated row is checked against the structural
 * invariants it relies on; non-zero means a result may be wrong).  `reset`
 * non-zero clears the counter after reading. */
int lcsg_sweep_errors(int device, int32_t *count, int reset);
/* Path counters of the row-sweep kernels on `device` since the last reset:
 * blocks of rows redone by the generic kernel after the register-resident
 * kernel flagged them, and blocks swept with the row state kept in the output
 * rows (finite prefix wider than the shared-memory capacity). */
int lcsg_sweep_paths(int device, int64_t *redone_blocks, int64_t *global_state_blocks, int reset);

#ifdef __cplusplus
}
#endif
#endif
