// lcsg_internal.cuh -- device-side data layout shared by the kernels and the
// host scheduler of the B200 Lu-Liu LCS path.  See DESIGN.md "Data layout".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lcsg {

// A reach table of one slab in HBM (solver.py:32-62 CostTable.reach/kmax):
// (n+1) x w1 int32, row r = start column r+1, column d = weight d.  Leaves
// (single string row, solver.py:72-88) are never materialised on the hot
// path: their weight-1 column is the next-occurrence row NX[sym] (built once
// per solve by the leaf kernel) and their weight-0 column is r+1.
//
// A VIRTUAL height-1 node (a 2-row slab whose parent is a narrow combine, n
// >= 2) is never materialised either: its (n+1) x 3 table is a closed form
// of its two leaves' NX rows (virtual_get below), read wherever the table
// would have been read -- the leaf-pair level costs no launch and no HBM
// round trip.
struct TabDev {
    const int32_t *reach;  // nullptr for a leaf / virtual node
    const int32_t *kmax;   // nullptr for a leaf / virtual node
    const int32_t *wstar;  // device scalar (node_wstar[node])
    int32_t w1;            // table width = min(slab rows, n) + 1
    int32_t leaf_row;      // leaf: 0-based index into the slab's row string; virtual
                           // node: its upper leaf's row; else -1
    int32_t leaf2;         // virtual node: its lower leaf's row + 1; else 0
    int32_t pair;          // batched solves: the pair whose NX block a leaf reads (0 otherwise)
};

// Per-solve constants, passed by value to every kernel.
struct Ctx {
    const uint8_t *rows;  // slab row string (device; batched: the pairs' slabs back to back)
    const int32_t *nx;    // 256 x (n+1): NX[s][r] = (first q >= r with cols[q]==s) + 2, else n+2
                          // (batched: one such block per pair, nx_stride ints apart)
    int64_t nx_stride;    // 256 * (n+1)
    int32_t n;
    int32_t inf;  // n + 2 (seqcore.py:37-39)
};

// One combine of the recursion (solver.py:91-110): U = upper slab, L = lower.
struct CombineDesc {
    TabDev U, L;
    int32_t *out_reach;  // (n+1) x w1
    int32_t *out_trace;  // (n+1) x w1 or nullptr (with_trace=False)
    int32_t *out_kmax;   // n+1
    int32_t *out_wstar;  // scalar, zero-initialised, atomicMax'ed
    int32_t w1;
    int32_t node;
    // row-sweep kernels (lcsg_sweep.cu): per-row insertion ranks ("events") of
    // the upper child and of this combine's own table -- ev[c] = first k with
    // reach[c+1][k] != reach[c][k+1]; U_ev_make: U's events are not a sweep
    // by-product and must be derived from its table first
    int32_t *U_ev;
    int32_t *out_ev;
    int32_t U_ev_make;
    int32_t pad_;
    int32_t *blk_flags;  // per block of rows: 1 = redo with the generic sweep kernel (zeroed per solve)
};

// Resolved accessor of a table inside a kernel.
struct TabAcc {
    const int32_t *reach;
    const int32_t *kmax;
    const int32_t *nx;   // leaf, or a virtual node's upper leaf
    const int32_t *nx2;  // virtual node's lower leaf (nullptr otherwise)
    int32_t w1;
    int32_t inf;
};

__device__ __forceinline__ TabAcc resolve(const TabDev &t, const Ctx &c) {
    TabAcc a;
    a.reach = t.reach;
    a.kmax = t.kmax;
    a.w1 = t.w1;
    a.inf = c.inf;
    const int32_t *nxp = c.nx + (size_t)t.pair * (size_t)c.nx_stride;
    a.nx = t.leaf_row >= 0 ? nxp + (size_t)c.rows[t.leaf_row] * (size_t)(c.n + 1) : nullptr;
    a.nx2 = t.leaf2 > 0 ? nxp + (size_t)c.rows[t.leaf2 - 1] * (size_t)(c.n + 1) : nullptr;
    return a;
}

// Row r of a virtual height-1 node = combine of leaf a (upper) and leaf b
// (lower) (solver.py:91-110 on two _base_table leaves): U = (r+1, A), A =
// NX_a[r]; L row x-1 = (x, NX_b[x-1]).  Weight 0: r+1.  Weight 1: min over
// k = 0 (L[r][1] = NX_b[r]) and k = 1 (L[A-1][0] = A).  Weight 2: only k = 1
// (L[A-1][1] = NX_b[A-1]).
__device__ __forceinline__ int32_t virtual_get(const TabAcc &t, int64_t r, int32_t d) {
    if (d == 0) return (int32_t)(r + 1);
    const int32_t xa = __ldg(t.nx + r);
    if (d == 1) return min(__ldg(t.nx2 + r), xa);
    return xa < t.inf ? __ldg(t.nx2 + (xa - 1)) : t.inf;
}

// Entry (r, d) of a table, d <= w1-1 (breakout.py:37-55 for leaves).
__device__ __forceinline__ int32_t tab_get(const TabAcc &t, int64_t r, int32_t d) {
    if (t.nx2) return virtual_get(t, r, d);
    if (t.nx) return d == 0 ? (int32_t)(r + 1) : __ldg(t.nx + r);
    return __ldg(t.reach + r * (int64_t)t.w1 + d);
}

// kmax of row r (solver.py:84,104: (reach < inf).sum - 1).
__device__ __forceinline__ int32_t tab_kmax(const TabAcc &t, int64_t r, int32_t inf) {
    if (t.nx2) {
        const int32_t xa = __ldg(t.nx + r);
        if (xa < inf && __ldg(t.nx2 + (xa - 1)) < inf) return 2;
        return min(__ldg(t.nx2 + r), xa) < inf ? 1 : 0;
    }
    if (t.nx) return (t.w1 == 2 && __ldg(t.nx + r) < inf) ? 1 : 0;
    return __ldg(t.kmax + r);
}

// Division by a launch-constant divisor without a divide sequence: q = n / d
// for 0 <= n < 2^31 as one 64-bit multiply and a shift (M = floor(2^(32+l)/d)
// + 1, l = ceil(log2 d); exact because (M d - 2^(32+l)) n < 2^(32+l)).
struct FastDiv {
    uint64_t M;
    int32_t d, l;
};
inline FastDiv make_fastdiv(int32_t d) {
    FastDiv f;
    f.d = d;
    f.l = 0;
    while ((1LL << f.l) < d) ++f.l;
    f.M = (uint64_t)((((unsigned __int128)1) << (32 + f.l)) / (unsigned)d) + 1;
    return f;
}
__device__ __forceinline__ int32_t fdiv(int32_t n, const FastDiv &f) {
    return (int32_t)(((uint64_t)(uint32_t)n * f.M) >> (32 + f.l));
}

// Recovery walk node (solver.py:180-207).
struct WalkNode {
    int32_t top_row, bottom_row;  // absolute 1-based vertex rows
    int32_t upper, lower;         // child ids (-1 for a leaf)
    int32_t w1;                   // this node's table width
    int32_t is_leaf;
    const int32_t *trace;         // this node's trace (nullptr: retrace)
    TabDev U, L;                  // children tables (for x = U.reach[i-1,k], retrace)
};

}  // namespace lcsg

// ---- launchers implemented in lcsg_kernels.cu ------------------------------
namespace lcsg {
// NX of `npairs` column strings of length n (back to back) -> npairs blocks
int launch_nx(const uint8_t *cols, int32_t n, int32_t npairs, int32_t *nx, int32_t *sym_wstar,
              cudaStream_t s);
// leaf_rows are rows of the concatenated slabs (pair = row / pair_rows)
int launch_leaf_wstar(const uint8_t *rows, const int32_t *leaf_nodes, const int32_t *leaf_rows,
                      int32_t nleaves, int32_t pair_rows, const int32_t *sym_wstar,
                      int32_t *node_wstar, cudaStream_t s);
// wstar of the virtual height-1 nodes: vnodes[4t..4t+3] = (node, upper leaf
// row, lower leaf row, pair)
int launch_virtual_wstar(Ctx c, const int32_t *vnodes, int32_t nvirt, int32_t *node_wstar,
                         cudaStream_t s);
int launch_leaf_table(Ctx c, int32_t leaf_row, int32_t w1, int32_t *reach, int32_t *kmax,
                      cudaStream_t s);
int launch_base_case_row(const uint8_t *cols, int32_t n, uint8_t sym, int32_t *out,
                         cudaStream_t s);
// kind: 0 = thread-per-row bisection, 1 = warp-per-row bisection; stride > 1
// restricts the launch to the skeleton rows 0, S, 2S, ..., n
int launch_combine(int kind, const CombineDesc *descs, int32_t ndesc, Ctx c, int key_shift,
                   bool key64, cudaStream_t s, int32_t stride = 1);
// thread-per-row bisection for tables of width <= 33 with coalesced
// (shared-memory staged) row writes
int launch_combine_staged(const CombineDesc *descs, int32_t ndesc, Ctx c, int key_shift,
                          bool key64, cudaStream_t s);
// narrow combines (every U and L weight <= P, P in 1,2,4,8,16; lcsg_narrow.cu):
// staged brute-force first-wins minimum, all rows
int narrow_bucket(int32_t max_weight);  // P, or -1 when too wide
// height-1 combines (both children leaves): direct NX reads, no staging
int launch_narrow_leafpair(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                           cudaStream_t s);
int launch_narrow(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t P, cudaStream_t s, bool full_width = false);
// skeleton rows 0, S, 2S, ..., n by exact Alg. 1 (one CTA per row)
int launch_skeleton(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                    int32_t stride, cudaStream_t s);
// skeleton rows, one warp per row (batched DFS; slab children, w1 <= 257)
int launch_skeleton_warp(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                         int32_t stride, cudaStream_t s);
// refinement pass: rows (2t+1)*delta from rows (2t)*delta and (2t+2)*delta
int launch_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t delta, cudaStream_t s);
int refine_rows(int64_t n1, int32_t delta);
// column refinement stage (lcsg_tile.cu): blocks of S local rows at row step
// rs; rows at multiples of S*rs (and the last row) must already be known
int launch_block_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                        int32_t S, int32_t rs, int32_t maxw1, cudaStream_t s);
// INF suffix + kmax/wstar of the interior rows after the tiled refinement
int launch_finalize_rows(const CombineDesc *descs, int32_t ndesc, Ctx c, int32_t S,
                         cudaStream_t s, int32_t maxw1, bool pre = false);
// row-sweep path (lcsg_sweep.cu): events of the upper children that need them,
// then the interior rows of blocks of S rows below each skeleton row
int launch_table_events(const CombineDesc *descs, int32_t ndesc, Ctx c, cudaStream_t s);
int launch_sweep(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64, int32_t S,
                 int32_t maxw1, cudaStream_t s);
int sweep_error_count(int32_t *count, bool reset);
int sweep_launch_count(int shift, bool key64, int32_t S, int32_t maxw1);
int sweep_pick_block(int32_t S, int32_t maxw1, int32_t count, int32_t n, int shift, bool key64,
                     int sm_count);
int launch_walk_level(const WalkNode *nodes, const int32_t *ids, int32_t count, Ctx c,
                      int32_t *wi, int32_t *wj, int32_t *cols_out, bool retrace, int key_shift,
                      bool key64, cudaStream_t s);
// Batched walks: pair p's root is root + p * pair_nodes, its table is
// root_tab with table pointers advanced by p * tab_stride ints (a leaf root:
// leaf_row advanced by p * pair_rows), its path lands at cols_out + p * (m+1).
struct RootBatch {
    int32_t npairs = 1, pair_nodes = 0, pair_rows = 0;
    int64_t tab_stride = 0;
};
int launch_walk_root(const WalkNode *nodes, int32_t root, Ctx c, TabDev root_tab, int32_t j,
                     int32_t i_start, int32_t *wi, int32_t *wj, int32_t *cols_out, RootBatch rb,
                     cudaStream_t s);
int launch_walk_final(Ctx c, TabDev root_tab, int32_t i_start, int32_t m, int32_t root,
                      const int32_t *wj, int32_t *cols_out, RootBatch rb, cudaStream_t s);
// assemble_lcs of `npairs` pairs: pair p reads rows + p*m, cols + p*n, path +
// p*(m+1) and writes out_len[p * out_stride], row_pos / col_pos + p * out_stride,
// subseq + p * sub_stride
int launch_assemble(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n,
                    const int32_t *path, int32_t *out_len, int32_t *row_pos, int32_t *col_pos,
                    uint8_t *subseq, cudaStream_t s, int32_t npairs = 1, int64_t out_stride = 0,
                    int64_t sub_stride = 0);
}  // namespace lcsg
