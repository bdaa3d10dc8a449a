// lcsg_kernels.cu -- sm_100a kernels of the Lu-Liu grid-graph LCS hot path.
//
//   nx_kernel            leaf step (breakout.py:37-55): per-symbol next-match
//                        suffix-min with warp shuffles; leaves are read from it
//   combine_*            recursive combine (_kernel.pyx:14-82): exact emulation
//                        of the Alg. 1 bisection with packed first-wins keys
//   walk_* / assemble    extraction (solver.py:160-234)
//
// All arithmetic is int32 compare/min; nothing here is GEMM-shaped, so no
// tensor cores are involved.
#include <cub/block/block_scan.cuh>

#include "lcsg_internal.cuh"

namespace lcsg {

#define LCSG_LAUNCH_CHECK()                         \
    do {                                            \
        cudaError_t e__ = cudaGetLastError();       \
        if (e__ != cudaSuccess) return (int)e__;    \
    } while (0)

// ---------------------------------------------------------------------------
// Leaf step: NX[s][r] = (min{q >= r : cols[q] == s}) + 2, INF = n + 2 if none,
// NX[s][n] = INF.  Entry r is the reference's base_case_row value for start
// column r+1 (breakout.py:51-55: suffix-min of scattered match positions, +1).
// One CTA per symbol walks the string right-to-left in 4096-column chunks;
// inside a chunk each thread takes 4 columns, then a warp-shuffle suffix-min
// and a cross-warp suffix-min over shared memory build the chunk suffix.
// ---------------------------------------------------------------------------
constexpr int NX_THREADS = 1024;
constexpr int NX_PER_THREAD = 4;
constexpr int NX_CHUNK = NX_THREADS * NX_PER_THREAD;

__global__ void __launch_bounds__(NX_THREADS) nx_kernel(const uint8_t *__restrict__ cols_all,
                                                        int32_t n, int32_t *__restrict__ nx,
                                                        int32_t *__restrict__ sym_wstar_all) {
    const int s = blockIdx.x;
    const int32_t pair = blockIdx.y;  // batched solves: one NX block per pair
    const uint8_t *__restrict__ cols = cols_all + (size_t)pair * (size_t)n;
    int32_t *sym_wstar = sym_wstar_all + 256 * pair;
    const int32_t inf = n + 2;
    int32_t *row = nx + ((size_t)pair * 256 + s) * (size_t)(n + 1);
    __shared__ int32_t warp_min[NX_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t carry = inf;  // min over everything right of the current chunk
    if (threadIdx.x == 0) row[n] = inf;
    for (int64_t base = ((int64_t)(n > 0 ? n - 1 : 0) / NX_CHUNK) * NX_CHUNK; n > 0 && base >= 0;
         base -= NX_CHUNK) {
        const int64_t q0 = base + (int64_t)threadIdx.x * NX_PER_THREAD;
        int32_t v[NX_PER_THREAD];
#pragma unroll
        for (int t = NX_PER_THREAD - 1; t >= 0; --t) {
            const int64_t q = q0 + t;
            int32_t x = (q < n && cols[q] == (uint8_t)s) ? (int32_t)q + 2 : inf;
            v[t] = (t == NX_PER_THREAD - 1) ? x : min(x, v[t + 1]);  // thread-local suffix
        }
        // warp suffix-min of the thread aggregates (v[0]) via shuffles
        int32_t agg = v[0];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t o = __shfl_down_sync(0xffffffffu, agg, d);
            if (lane + d < 32) agg = min(agg, o);
        }
        // agg = min over lanes [lane, 31]; exclusive = over lanes (lane, 31]
        int32_t excl = __shfl_down_sync(0xffffffffu, agg, 1);
        if (lane == 31) excl = inf;
        if (lane == 0) warp_min[wid] = agg;
        __syncthreads();
        int32_t right_warps = inf;  // min over warps > wid
        for (int w = wid + 1; w < NX_THREADS / 32; ++w) right_warps = min(right_warps, warp_min[w]);
        const int32_t right = min(min(excl, right_warps), carry);
#pragma unroll
        for (int t = 0; t < NX_PER_THREAD; ++t) {
            const int64_t q = q0 + t;
            if (q < n) row[q] = min(v[t], right);
        }
        int32_t chunk_min = inf;
        for (int w = 0; w < NX_THREADS / 32; ++w) chunk_min = min(chunk_min, warp_min[w]);
        carry = min(carry, chunk_min);
        __syncthreads();
    }
    if (threadIdx.x == 0) sym_wstar[s] = (n >= 1 && carry < inf) ? 1 : 0;
}

int launch_nx(const uint8_t *cols, int32_t n, int32_t npairs, int32_t *nx, int32_t *sym_wstar,
              cudaStream_t s) {
    nx_kernel<<<dim3(256, npairs), NX_THREADS, 0, s>>>(cols, n, nx, sym_wstar);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// wstar of every leaf (solver.py:88): 1 iff its symbol occurs in cols.
__global__ void leaf_wstar_kernel(const uint8_t *__restrict__ rows,
                                  const int32_t *__restrict__ leaf_nodes,
                                  const int32_t *__restrict__ leaf_rows, int32_t nleaves,
                                  int32_t pair_rows, const int32_t *__restrict__ sym_wstar,
                                  int32_t *__restrict__ node_wstar) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nleaves) {
        const int32_t r = leaf_rows[t];
        node_wstar[leaf_nodes[t]] = sym_wstar[256 * (r / pair_rows) + rows[r]];
    }
}

int launch_leaf_wstar(const uint8_t *rows, const int32_t *leaf_nodes, const int32_t *leaf_rows,
                      int32_t nleaves, int32_t pair_rows, const int32_t *sym_wstar,
                      int32_t *node_wstar, cudaStream_t s) {
    if (nleaves <= 0) return 0;
    leaf_wstar_kernel<<<(nleaves + 255) / 256, 256, 0, s>>>(rows, leaf_nodes, leaf_rows, nleaves,
                                                            pair_rows, sym_wstar, node_wstar);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// wstar of the virtual height-1 nodes (solver.py:108, max over rows of kmax):
// kmax of row r is 2 iff a occurs at some q >= r and b after it, 1 iff a or b
// occurs at or after r -- both are largest at r = 0.
__global__ void virtual_wstar_kernel(Ctx c, const int32_t *__restrict__ vnodes, int32_t nvirt,
                                     int32_t *__restrict__ node_wstar) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nvirt) return;
    TabDev d;
    d.reach = nullptr;
    d.kmax = nullptr;
    d.wstar = nullptr;
    d.w1 = 3;
    d.leaf_row = vnodes[4 * t + 1];
    d.leaf2 = vnodes[4 * t + 2] + 1;
    d.pair = vnodes[4 * t + 3];
    node_wstar[vnodes[4 * t]] = tab_kmax(resolve(d, c), 0, c.inf);
}

int launch_virtual_wstar(Ctx c, const int32_t *vnodes, int32_t nvirt, int32_t *node_wstar,
                         cudaStream_t s) {
    if (nvirt <= 0) return 0;
    virtual_wstar_kernel<<<(nvirt + 255) / 256, 256, 0, s>>>(c, vnodes, nvirt, node_wstar);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// Materialise one leaf table (solver.py:72-88) -- only for API copy-out.
__global__ void leaf_table_kernel(Ctx c, int32_t leaf_row, int32_t w1, int32_t *reach,
                                  int32_t *kmax) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r > c.n) return;
    const int32_t *nx = c.nx + (size_t)c.rows[leaf_row] * (size_t)(c.n + 1);  // single solves
    reach[r * w1] = (int32_t)r + 1;
    int32_t k = 0;
    if (w1 == 2) {
        int32_t v = nx[r];
        reach[r * w1 + 1] = v;
        k = v < c.inf ? 1 : 0;
    }
    kmax[r] = k;
}

int launch_leaf_table(Ctx c, int32_t leaf_row, int32_t w1, int32_t *reach, int32_t *kmax,
                      cudaStream_t s) {
    int64_t n1 = (int64_t)c.n + 1;
    leaf_table_kernel<<<(unsigned)((n1 + 255) / 256), 256, 0, s>>>(c, leaf_row, w1, reach, kmax);
    LCSG_LAUNCH_CHECK();
    return 0;
}

__global__ void base_case_row_kernel(const uint8_t *cols, int32_t n, uint8_t sym, int32_t *out) {
    // single-symbol variant of nx_kernel, used by the lcsg_base_case_row mirror
    __shared__ int32_t warp_min[NX_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int32_t inf = n + 2;
    int32_t carry = inf;
    for (int64_t base = ((int64_t)(n > 0 ? n - 1 : 0) / NX_CHUNK) * NX_CHUNK; n > 0 && base >= 0;
         base -= NX_CHUNK) {
        const int64_t q0 = base + (int64_t)threadIdx.x * NX_PER_THREAD;
        int32_t v[NX_PER_THREAD];
#pragma unroll
        for (int t = NX_PER_THREAD - 1; t >= 0; --t) {
            const int64_t q = q0 + t;
            int32_t x = (q < n && cols[q] == sym) ? (int32_t)q + 2 : inf;
            v[t] = (t == NX_PER_THREAD - 1) ? x : min(x, v[t + 1]);
        }
        int32_t agg = v[0];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t o = __shfl_down_sync(0xffffffffu, agg, d);
            if (lane + d < 32) agg = min(agg, o);
        }
        int32_t excl = __shfl_down_sync(0xffffffffu, agg, 1);
        if (lane == 31) excl = inf;
        if (lane == 0) warp_min[wid] = agg;
        __syncthreads();
        int32_t right_warps = inf;
        for (int w = wid + 1; w < NX_THREADS / 32; ++w) right_warps = min(right_warps, warp_min[w]);
        const int32_t right = min(min(excl, right_warps), carry);
#pragma unroll
        for (int t = 0; t < NX_PER_THREAD; ++t) {
            const int64_t q = q0 + t;
            if (q < n) out[q] = min(v[t], right);
        }
        int32_t chunk_min = inf;
        for (int w = 0; w < NX_THREADS / 32; ++w) chunk_min = min(chunk_min, warp_min[w]);
        carry = min(carry, chunk_min);
        __syncthreads();
    }
}

int launch_base_case_row(const uint8_t *cols, int32_t n, uint8_t sym, int32_t *out,
                         cudaStream_t s) {
    base_case_row_kernel<<<1, NX_THREADS, 0, s>>>(cols, n, sym, out);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// Combine.  Packed first-wins key: (value << shift) | k.  The minimum key is
// the minimum value and, among ties, the smallest split weight k -- exactly
// the reference's strict-< linear scan (_kernel.pyx:38-44).
// ---------------------------------------------------------------------------
template <typename Key>
__device__ __forceinline__ Key pack(int32_t v, int32_t k, int shift) {
    return ((Key)(uint32_t)v << shift) | (Key)(uint32_t)k;
}
template <typename Key>
__device__ __forceinline__ int32_t key_val(Key key, int shift) {
    return (int32_t)(key >> shift);
}
template <typename Key>
__device__ __forceinline__ int32_t key_k(Key key, int shift) {
    return (int32_t)(key & (((Key)1 << shift) - 1));
}

__device__ __forceinline__ uint32_t warp_min(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t warp_min(uint64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}

// cell_value (_kernel.pyx:14-25) for start row i (0-based) with x = U[i,k].
__device__ __forceinline__ int32_t cell(const TabAcc &L, int32_t x, int32_t k, int32_t j,
                                        int32_t inf, int32_t wl) {
    if (k > j) return inf;
    if (x >= inf) return inf;
    if (j - k > wl) return inf;
    return tab_get(L, (int64_t)x - 1, j - k);
}

// Thread-per-row exact bisection (small tables): the reference's col_mins
// (_kernel.pyx:28-60) as an iterative DFS with an explicit right-sibling stack.
constexpr int STACK = 24;
constexpr int CT_THREADS = 64;

template <typename Key>
__global__ void __launch_bounds__(256) combine_thread_kernel(const CombineDesc *__restrict__ descs,
                                                             int32_t ndesc, Ctx c, int shift,
                                                             int64_t rows_pad, int32_t stride,
                                                             int32_t nrows) {
    // rows r = 0 .. nrows-1 map to i = r*stride, the last one to n (= n1-1)
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t di = gid / rows_pad;  // warp-uniform: rows_pad % 32 == 0
    if (di >= ndesc) return;
    const int64_t r = gid - di * rows_pad;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t i = (r == nrows - 1) ? n1 - 1 : r * stride;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    int32_t kfin = -1;
    if (r < nrows) {
        const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
        const int32_t w = d.w1 - 1, wl = L.w1 - 1;
        const int32_t kmaxU = tab_kmax(U, i, inf);
        const int32_t wstarL = *d.L.wstar;
        int32_t colhi = min(w, kmaxU + wstarL);
        int32_t *reach = d.out_reach + i * d.w1;
        int32_t *trace = d.out_trace ? d.out_trace + i * d.w1 : nullptr;
        uint64_t stk[STACK];
        int sp = 0;
        int32_t left = 0, right = colhi, top = 0, bottom = kmaxU;
        for (;;) {
            while (right >= left) {
                const int32_t mid = (left + right + 1) >> 1;
                Key best = ~(Key)0;
                for (int32_t k = top; k <= bottom; ++k) {
                    const int32_t x = tab_get(U, i, k);
                    const Key key = pack<Key>(cell(L, x, k, mid, inf, wl), k, shift);
                    best = key < best ? key : best;
                }
                const int32_t bv = key_val<Key>(best, shift), bk = key_k<Key>(best, shift);
                reach[mid] = bv;
                if (trace) trace[mid] = bk;
                if (bv != inf) {
                    kfin = max(kfin, mid);
                    if (mid + 1 <= right && sp < STACK)
                        stk[sp++] = ((uint64_t)(uint16_t)(mid + 1) << 48) |
                                    ((uint64_t)(uint16_t)right << 32) |
                                    ((uint64_t)(uint16_t)bk << 16) | (uint64_t)(uint16_t)bottom;
                    right = mid - 1;
                    bottom = bk;
                } else {
                    for (int32_t q = mid + 1; q <= right; ++q) {
                        reach[q] = inf;
                        if (trace) trace[q] = top;
                    }
                    right = mid - 1;
                }
            }
            if (sp == 0) break;
            const uint64_t e = stk[--sp];
            left = (int32_t)(uint16_t)(e >> 48);
            right = (int32_t)(uint16_t)(e >> 32);
            top = (int32_t)(uint16_t)(e >> 16);
            bottom = (int32_t)(uint16_t)e;
        }
        for (int32_t q = colhi + 1; q <= w; ++q) {
            reach[q] = inf;
            if (trace) trace[q] = 0;
        }
        d.out_kmax[i] = kfin;
    }
    // kfin == last finite column == kmax of the row (finite prefix property)
    const int32_t wmax = __reduce_max_sync(0xffffffffu, kfin);
    if ((threadIdx.x & 31) == 0 && wmax >= 0) atomicMax(d.out_wstar, wmax);
}

// Same exact bisection for narrow tables (w1 <= TS_W), all rows (stride 1):
// each thread's row goes to a shared-memory slot first, then every warp writes
// its 32 consecutive rows as ONE contiguous block.  Writing rows directly
// (lane-strided stores) made ncu count ~3x the compulsory DRAM traffic on
// these levels (partially written sectors).
constexpr int TS_W = 33;       // max table width staged
constexpr int TS_SLOT = 33;    // odd slot pitch: conflict-free per-lane writes
constexpr int TS_THREADS = 128;

template <typename Key>
__global__ void __launch_bounds__(TS_THREADS)
    combine_thread_staged_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c,
                                 int shift, int64_t rows_pad) {
    __shared__ int32_t s_reach[TS_THREADS * TS_SLOT];
    __shared__ uint16_t s_trace[TS_THREADS * TS_SLOT];
    const int lane = threadIdx.x & 31;
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t di = gid / rows_pad;  // warp-uniform: rows_pad % 32 == 0
    if (di >= ndesc) return;
    const int64_t i = gid - di * rows_pad;
    const int64_t n1 = (int64_t)c.n + 1;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const int32_t w1 = d.w1, w = w1 - 1;
    int32_t *sr = s_reach + threadIdx.x * TS_SLOT;
    uint16_t *st = s_trace + threadIdx.x * TS_SLOT;
    int32_t kfin = -1;
    if (i < n1) {
        const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
        const int32_t wl = L.w1 - 1;
        const int32_t kmaxU = tab_kmax(U, i, inf);
        const int32_t colhi = min(w, kmaxU + *d.L.wstar);
        uint64_t stk[STACK];
        int sp = 0;
        int32_t left = 0, right = colhi, top = 0, bottom = kmaxU;
        for (;;) {
            while (right >= left) {
                const int32_t mid = (left + right + 1) >> 1;
                Key best = ~(Key)0;
                for (int32_t k = top; k <= bottom; ++k) {
                    const int32_t x = tab_get(U, i, k);
                    const Key key = pack<Key>(cell(L, x, k, mid, inf, wl), k, shift);
                    best = key < best ? key : best;
                }
                const int32_t bv = key_val<Key>(best, shift), bk = key_k<Key>(best, shift);
                sr[mid] = bv;
                st[mid] = (uint16_t)bk;
                if (bv != inf) {
                    kfin = max(kfin, mid);
                    if (mid + 1 <= right && sp < STACK)
                        stk[sp++] = ((uint64_t)(uint16_t)(mid + 1) << 48) |
                                    ((uint64_t)(uint16_t)right << 32) |
                                    ((uint64_t)(uint16_t)bk << 16) | (uint64_t)(uint16_t)bottom;
                    right = mid - 1;
                    bottom = bk;
                } else {
                    for (int32_t q = mid + 1; q <= right; ++q) {
                        sr[q] = inf;
                        st[q] = (uint16_t)top;
                    }
                    right = mid - 1;
                }
            }
            if (sp == 0) break;
            const uint64_t e = stk[--sp];
            left = (int32_t)(uint16_t)(e >> 48);
            right = (int32_t)(uint16_t)(e >> 32);
            top = (int32_t)(uint16_t)(e >> 16);
            bottom = (int32_t)(uint16_t)e;
        }
        for (int32_t q = colhi + 1; q <= w; ++q) {
            sr[q] = inf;
            st[q] = 0;
        }
        d.out_kmax[i] = kfin;
    }
    __syncwarp();
    // coalesced copy-out of the warp's consecutive rows
    const int64_t i0 = i - lane;
    const int32_t nrow = (int32_t)min((int64_t)32, max((int64_t)0, n1 - i0));
    const int32_t total = nrow * w1;
    const int wb = threadIdx.x - lane;
    int32_t *gr = d.out_reach + i0 * w1;
    int32_t *gt = d.out_trace ? d.out_trace + i0 * w1 : nullptr;
    for (int32_t f = lane; f < total; f += 32) {
        const int32_t rr = f / w1, cc = f - rr * w1;
        gr[f] = s_reach[(wb + rr) * TS_SLOT + cc];
        if (gt) gt[f] = s_trace[(wb + rr) * TS_SLOT + cc];
    }
    const int32_t wmax = __reduce_max_sync(0xffffffffu, kfin);
    if (lane == 0 && wmax >= 0) atomicMax(d.out_wstar, wmax);
}

// Warp-per-row exact bisection: the warp evaluates one Alg. 1 node at a time,
// lanes striding over its row range [top..bottom] and reducing packed keys
// with a warp min (REDUX.MIN for 32-bit keys).  The DFS stack is warp-uniform
// and lives in shared memory.
constexpr int WARP_KERNEL_WARPS = 2;
constexpr int WSTACK = 34;  // > log2(max colhi) + 1 for colhi < 2^32

template <typename Key>
__global__ void __launch_bounds__(32 * WARP_KERNEL_WARPS)
    combine_warp_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                        int32_t stride, int32_t nrows) {
    __shared__ int4 stk_all[WARP_KERNEL_WARPS][WSTACK];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int4 *stk = stk_all[wid];
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t gw = blockIdx.x * (int64_t)WARP_KERNEL_WARPS + wid;
    const int64_t di = gw / nrows;
    if (di >= ndesc) return;
    const int64_t r = gw - di * nrows;
    const int64_t i = (r == nrows - 1) ? n1 - 1 : r * stride;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t w = d.w1 - 1, wl = L.w1 - 1;
    const int32_t kmaxU = tab_kmax(U, i, inf);
    const int32_t wstarL = *d.L.wstar;
    const int32_t colhi = min(w, kmaxU + wstarL);
    int32_t *reach = d.out_reach + i * d.w1;
    int32_t *trace = d.out_trace ? d.out_trace + i * d.w1 : nullptr;
    int sp = 0;
    int32_t kfin = -1;
    int32_t left = 0, right = colhi, top = 0, bottom = kmaxU;
    for (;;) {
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            Key best = ~(Key)0;
            for (int32_t k = top + lane; k <= bottom; k += 32) {
                const int32_t x = tab_get(U, i, k);
                const Key key = pack<Key>(cell(L, x, k, mid, inf, wl), k, shift);
                best = key < best ? key : best;
            }
            best = warp_min(best);
            const int32_t bv = key_val<Key>(best, shift), bk = key_k<Key>(best, shift);
            if (lane == 0) {
                reach[mid] = bv;
                if (trace) trace[mid] = bk;
            }
            if (bv != inf) {
                kfin = max(kfin, mid);
                if (mid + 1 <= right) {
                    if (lane == 0) stk[sp] = make_int4(mid + 1, right, bk, bottom);
                    ++sp;
                }
                right = mid - 1;
                bottom = bk;
            } else {
                for (int32_t q = mid + 1 + lane; q <= right; q += 32) {
                    reach[q] = inf;
                    if (trace) trace[q] = top;
                }
                right = mid - 1;
            }
        }
        if (sp == 0) break;
        __syncwarp();
        const int4 e = stk[--sp];
        __syncwarp();
        left = e.x;
        right = e.y;
        top = e.z;
        bottom = e.w;
    }
    for (int32_t q = colhi + 1 + lane; q <= w; q += 32) {
        reach[q] = inf;
        if (trace) trace[q] = 0;
    }
    if (lane == 0) {
        d.out_kmax[i] = kfin;
        atomicMax(d.out_wstar, kfin);
    }
}

int launch_combine_staged(const CombineDesc *descs, int32_t ndesc, Ctx c, int key_shift,
                          bool key64, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t rows_pad = (n1 + 31) / 32 * 32;
    const unsigned blocks = (unsigned)((rows_pad * ndesc + TS_THREADS - 1) / TS_THREADS);
    if (key64)
        combine_thread_staged_kernel<uint64_t><<<blocks, TS_THREADS, 0, s>>>(descs, ndesc, c, key_shift, rows_pad);
    else
        combine_thread_staged_kernel<uint32_t><<<blocks, TS_THREADS, 0, s>>>(descs, ndesc, c, key_shift, rows_pad);
    LCSG_LAUNCH_CHECK();
    return 0;
}

int launch_combine(int kind, const CombineDesc *descs, int32_t ndesc, Ctx c, int key_shift,
                   bool key64, cudaStream_t s, int32_t stride) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    // stride 1: every row; stride S: skeleton rows 0, S, 2S, ..., n
    const int32_t nrows = stride <= 1 ? (int32_t)n1 : (int32_t)((n1 - 1 + stride - 1) / stride) + 1;
    if (kind == 0) {
        const int64_t rows_pad = ((int64_t)nrows + 31) / 32 * 32;
        const int64_t threads = rows_pad * ndesc;
        // small CTAs: per-row DFS work is very uneven, and a CTA holds its
        // slot until its slowest row is done
        const unsigned blocks = (unsigned)((threads + CT_THREADS - 1) / CT_THREADS);
        if (key64)
            combine_thread_kernel<uint64_t><<<blocks, CT_THREADS, 0, s>>>(descs, ndesc, c, key_shift, rows_pad, stride, nrows);
        else
            combine_thread_kernel<uint32_t><<<blocks, CT_THREADS, 0, s>>>(descs, ndesc, c, key_shift, rows_pad, stride, nrows);
    } else {
        const int64_t warps = (int64_t)nrows * ndesc;
        const unsigned blocks = (unsigned)((warps + WARP_KERNEL_WARPS - 1) / WARP_KERNEL_WARPS);
        if (key64)
            combine_warp_kernel<uint64_t><<<blocks, 32 * WARP_KERNEL_WARPS, 0, s>>>(descs, ndesc, c, key_shift, stride, nrows);
        else
            combine_warp_kernel<uint32_t><<<blocks, 32 * WARP_KERNEL_WARPS, 0, s>>>(descs, ndesc, c, key_shift, stride, nrows);
    }
    LCSG_LAUNCH_CHECK();
    return 0;
}

// ---------------------------------------------------------------------------
// Extraction.  Recovery walk (solver.py:180-207), one launch per tree depth:
// node (i, jj) -> k = trace[i-1, jj] (or the low-memory first-wins retrace,
// solver.py:165-177), x = U.reach[i-1, k]; children get (i, k) and (x, jj-k);
// a leaf child records cols[top_row-1] = i.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void walk_children(const WalkNode &nd, const WalkNode *nodes, Ctx c,
                                              int32_t i, int32_t jj, int32_t k, int32_t *wi,
                                              int32_t *wj, int32_t *cols_out) {
    const TabAcc U = resolve(nd.U, c);
    const int32_t x = tab_get(U, (int64_t)i - 1, k);
    const WalkNode &up = nodes[nd.upper];
    const WalkNode &lo = nodes[nd.lower];
    if (up.is_leaf) cols_out[up.top_row - 1] = i;
    else { wi[nd.upper] = i; wj[nd.upper] = k; }
    if (lo.is_leaf) cols_out[lo.top_row - 1] = x;
    else { wi[nd.lower] = x; wj[nd.lower] = jj - k; }
}

__global__ void walk_trace_kernel(const WalkNode *__restrict__ nodes, const int32_t *__restrict__ ids,
                                  int32_t count, Ctx c, int32_t *wi, int32_t *wj, int32_t *cols_out) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int32_t id = ids[t];
    const WalkNode nd = nodes[id];
    const int32_t i = wi[id], jj = wj[id];
    int32_t k = 0;
    if (nd.trace) {
        k = nd.trace[((int64_t)i - 1) * nd.w1 + jj];
    } else {
        // a virtual node keeps no trace: first-wins retrace over its (at most
        // 3) splits (solver.py:165-177)
        const TabAcc U = resolve(nd.U, c), L = resolve(nd.L, c);
        const int32_t inf = c.inf;
        const int32_t hi = min(jj, tab_kmax(U, (int64_t)i - 1, inf));
        int32_t best = INT32_MAX;
        for (int32_t kk = 0; kk <= hi; ++kk) {
            const int32_t x = tab_get(U, (int64_t)i - 1, kk);
            const int32_t v = (x < inf && jj - kk < L.w1) ? tab_get(L, (int64_t)x - 1, jj - kk) : inf;
            if (v < best) {
                best = v;
                k = kk;
            }
        }
    }
    walk_children(nd, nodes, c, i, jj, k, wi, wj, cols_out);
}

template <typename Key>
__global__ void walk_retrace_kernel(const WalkNode *__restrict__ nodes, const int32_t *__restrict__ ids,
                                    int32_t count, Ctx c, int32_t *wi, int32_t *wj,
                                    int32_t *cols_out, int shift) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (t >= count) return;
    const int32_t id = ids[t];
    const WalkNode nd = nodes[id];
    const int32_t i = wi[id], jj = wj[id];
    const TabAcc U = resolve(nd.U, c), L = resolve(nd.L, c);
    const int32_t inf = c.inf;
    const int32_t hi = min(jj, tab_kmax(U, (int64_t)i - 1, inf));
    Key best = ~(Key)0;
    for (int32_t k = lane; k <= hi; k += 32) {
        // compose_cell (monotone.py:46-63)
        const int32_t x = tab_get(U, (int64_t)i - 1, k);
        int32_t v = inf;
        const int32_t dd = jj - k;
        if (x < inf && dd < L.w1) v = tab_get(L, (int64_t)x - 1, dd);
        const Key key = pack<Key>(v, k, shift);
        best = key < best ? key : best;
    }
    best = warp_min(best);
    if (lane == 0) walk_children(nd, nodes, c, i, jj, key_k<Key>(best, shift), wi, wj, cols_out);
}

int launch_walk_level(const WalkNode *nodes, const int32_t *ids, int32_t count, Ctx c,
                      int32_t *wi, int32_t *wj, int32_t *cols_out, bool retrace, int key_shift,
                      bool key64, cudaStream_t s) {
    if (count <= 0) return 0;
    if (!retrace) {
        walk_trace_kernel<<<(count + 127) / 128, 128, 0, s>>>(nodes, ids, count, c, wi, wj, cols_out);
    } else {
        const unsigned blocks = (unsigned)(((int64_t)count * 32 + 127) / 128);
        if (key64)
            walk_retrace_kernel<uint64_t><<<blocks, 128, 0, s>>>(nodes, ids, count, c, wi, wj, cols_out, key_shift);
        else
            walk_retrace_kernel<uint32_t><<<blocks, 128, 0, s>>>(nodes, ids, count, c, wi, wj, cols_out, key_shift);
    }
    LCSG_LAUNCH_CHECK();
    return 0;
}

// Root of the walk: j < 0 means "the LCS length" = kmax[0] of the root
// (solver.py:160-162), read on the device so no host round trip is needed.
// (i_start = 1 for lcs(); other start columns walk a band sub-tree for the
// multi-GPU schedule; WalkNode.top_row is relative to the slab's first row.)
__device__ __forceinline__ TabDev pair_root(TabDev t, int32_t p, const RootBatch &rb) {
    if (t.reach) {
        t.reach += p * rb.tab_stride;
        t.kmax += p * rb.tab_stride;
    } else {
        t.leaf_row += p * rb.pair_rows;
        t.pair = p;
    }
    return t;
}

__global__ void walk_root_kernel(const WalkNode *nodes, int32_t root0, Ctx c, TabDev root_tab,
                                 int32_t j, int32_t i_start, int32_t *wi, int32_t *wj,
                                 int32_t *cols_out, RootBatch rb) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;  // pair
    if (p >= rb.npairs) return;
    const int32_t root = root0 + p * rb.pair_nodes;
    const TabAcc R = resolve(pair_root(root_tab, p, rb), c);
    const int32_t jj = j >= 0 ? j : tab_kmax(R, i_start - 1, c.inf);
    wi[root] = i_start;
    wj[root] = jj;
    if (nodes[root].is_leaf) cols_out[nodes[root].top_row - 1] = i_start;
}

int launch_walk_root(const WalkNode *nodes, int32_t root, Ctx c, TabDev root_tab, int32_t j,
                     int32_t i_start, int32_t *wi, int32_t *wj, int32_t *cols_out, RootBatch rb,
                     cudaStream_t s) {
    walk_root_kernel<<<(rb.npairs + 127) / 128, 128, 0, s>>>(nodes, root, c, root_tab, j, i_start,
                                                             wi, wj, cols_out, rb);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// cols[m] = table.reach[i_start-1, j] (solver.py:206)
__global__ void walk_final_kernel(Ctx c, TabDev root_tab, int32_t m, int32_t i_start,
                                  int32_t root0, const int32_t *wj, int32_t *cols_out,
                                  RootBatch rb) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= rb.npairs) return;
    const TabAcc R = resolve(pair_root(root_tab, p, rb), c);
    cols_out[(int64_t)p * (m + 1) + m] = tab_get(R, i_start - 1, wj[root0 + p * rb.pair_nodes]);
}

int launch_walk_final(Ctx c, TabDev root_tab, int32_t i_start, int32_t m, int32_t root,
                      const int32_t *wj, int32_t *cols_out, RootBatch rb, cudaStream_t s) {
    walk_final_kernel<<<(rb.npairs + 127) / 128, 128, 0, s>>>(c, root_tab, m, i_start, root, wj,
                                                              cols_out, rb);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// assemble_lcs (solver.py:210-234): mark + block scan + compact, one CTA.
constexpr int ASM_THREADS = 1024;
__global__ void __launch_bounds__(ASM_THREADS)
    assemble_kernel(const uint8_t *__restrict__ rows, int32_t m, const uint8_t *__restrict__ cols,
                    int32_t n, const int32_t *__restrict__ path, int32_t *out_len,
                    int32_t *row_pos, int32_t *col_pos, uint8_t *subseq, int64_t out_stride,
                    int64_t sub_stride) {
    // one CTA per pair of a batch
    const int64_t p = blockIdx.x;
    rows += p * m;
    cols += p * n;
    path += p * (m + 1);
    out_len += p * out_stride;
    row_pos += p * out_stride;
    col_pos += p * out_stride;
    subseq += p * sub_stride;
    using Scan = cub::BlockScan<int32_t, ASM_THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    int32_t carry = 0;
    if (m > 0 && n > 0) {
        for (int32_t base = 0; base < m; base += ASM_THREADS) {
            const int32_t r = base + threadIdx.x;
            int32_t mark = 0, cur = 0;
            if (r < m) {
                const int32_t prev = path[r];
                cur = path[r + 1];
                int32_t land = cur - 2;
                land = land < 0 ? 0 : (land > n - 1 ? n - 1 : land);
                mark = (cur > prev) && (rows[r] == cols[land]);
            }
            int32_t pos, total;
            Scan(tmp).ExclusiveSum(mark, pos, total);
            if (mark) {
                subseq[carry + pos] = rows[r];
                row_pos[carry + pos] = r + 1;
                col_pos[carry + pos] = cur - 1;
            }
            carry += total;
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) *out_len = carry;
}

int launch_assemble(const uint8_t *rows, int32_t m, const uint8_t *cols, int32_t n,
                    const int32_t *path, int32_t *out_len, int32_t *row_pos, int32_t *col_pos,
                    uint8_t *subseq, cudaStream_t s, int32_t npairs, int64_t out_stride,
                    int64_t sub_stride) {
    assemble_kernel<<<npairs, ASM_THREADS, 0, s>>>(rows, m, cols, n, path, out_len, row_pos,
                                                   col_pos, subseq, out_stride, sub_stride);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
