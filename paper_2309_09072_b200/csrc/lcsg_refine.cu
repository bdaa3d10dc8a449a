// lcsg_refine.cu -- the fast combine for wide tables: skeleton + refinement.
//
// The reference evaluates every output row i of a combine with its own
// Alg. 1 bisection (_kernel.pyx:28-82): ~log2(w) rounds of dependent
// scattered gathers per row.  On the GPU that is a latency chain.  Here:
//
//  1. skeleton rows i = 0, S, 2S, ..., n (S = 16 by default) are computed by
//     the exact bisection, one CTA per row: the first rounds of Alg. 1 are
//     evaluated cooperatively by all 8 warps, then each warp runs the DFS of
//     one of the <= 8 resulting sub-trees (same outputs as the reference,
//     INF-cell traces included);
//  2. every other row c is then computed in log2(S) refinement passes
//     (delta = S/2 ... 1) from its two already-computed neighbours a = c-delta
//     and b = c+delta: with X(i,j) = U[i, k*(i,j)] the crossing column of the
//     first-wins argmin, X(a,j) <= X(c,j) <= X(b,j) (monotone argmin of a
//     Monge composition; verified on every finite cell of the parity suite),
//     so k*(c,j) lies in the short range of k with U[c,k] in [X(a,j), X(b,j)]
//     -- found with two tiny binary searches in the shared-memory copy of the
//     U row (interleave: U[a,k] <= U[c,k] <= U[a,k+delta]).  Lanes map to
//     consecutive output columns, so the L gathers of one warp hit a handful
//     of 128-B lines and all writes are coalesced.  The first-wins minimum over
//     that range equals the reference's value and trace (the global first-wins
//     argmin lies inside it).
//     Cells finite in row c but INF in row b (at most b - c per row) have no
//     upper bound and are scanned over [lower bound, min(j, kmax_c)] by a whole
//     warp; INF cells get the reference's bisection-artifact trace by
//     replaying Alg. 1's path over the INF suffix (O(log w) per row, no
//     gathers), and cells beyond colhi get (INF, 0) as in _kernel.pyx:79-82.
#include <cstdlib>

#include "lcsg_internal.cuh"

namespace lcsg {

#define LCSG_LAUNCH_CHECK()                         \
    do {                                            \
        cudaError_t e__ = cudaGetLastError();       \
        if (e__ != cudaSuccess) return (int)e__;    \
    } while (0)

template <typename Key>
__device__ __forceinline__ Key rpack(int32_t v, int32_t k, int shift) {
    return ((Key)(uint32_t)v << shift) | (Key)(uint32_t)k;
}
template <typename Key>
__device__ __forceinline__ int32_t rval(Key key, int shift) { return (int32_t)(key >> shift); }
template <typename Key>
__device__ __forceinline__ int32_t rk(Key key, int shift) {
    return (int32_t)(key & (((Key)1 << shift) - 1));
}
__device__ __forceinline__ uint32_t rwarp_min(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t rwarp_min(uint64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}
__device__ __forceinline__ void smem_min(uint32_t *p, uint32_t v) { atomicMin(p, v); }
__device__ __forceinline__ void smem_min(uint64_t *p, uint64_t v) {
    atomicMin((unsigned long long *)p, (unsigned long long)v);
}

// cell_value (_kernel.pyx:14-25) with x = U[i,k] already loaded.
__device__ __forceinline__ int32_t rcell(const TabAcc &L, int32_t x, int32_t k, int32_t j,
                                         int32_t inf, int32_t wl) {
    if (k > j || x >= inf || j - k > wl) return inf;
    return tab_get(L, (int64_t)x - 1, j - k);
}

// ---------------------------------------------------------------------------
// 1. skeleton rows: exact Alg. 1, one CTA (8 warps) per row.
// ---------------------------------------------------------------------------
constexpr int SK_WARPS = 8;
// per-warp stack of the batched DFS: a step pops up to 32 nodes and pushes
// <= 2 per node; within SK_SLACK of the top it pops one node at a time (plain
// DFS: the stack then grows by <= 1 per tree level, and the tree height is
// < 34), so it never overflows
constexpr int SK_STACK = 320;
constexpr int SK_SLACK = 40;
constexpr int SK_SERIAL = 12;  // ranges / fills up to this length: one lane (24/48 slower, 6/8 equal)

// Batched DFS of Alg. 1's bisection tree (_kernel.pyx:28-60) for one output
// row, by one warp: every node's (value, trace) depends only on its own
// (left, right, top, bottom), so the stack is consumed in batches -- lane l
// takes the l-th node, scans a short split range [top, bottom] serially, and
// long ranges / long INF fills are done cooperatively by the whole warp.
// Outputs equal the reference's node by node (order-independent writes to
// disjoint cells); the batch turns the one-node-at-a-time chain of dependent
// gathers (~colhi nodes per row) into ~colhi / 32 steps.  `stk` holds `sp`
// pending nodes on entry; each lane's kfin gets the largest finite mid it saw.
template <typename Key, typename Cell>
__device__ __forceinline__ void batched_dfs(int4 *stk, int sp, const Cell &cell, int32_t *reach,
                                            int32_t *trace, int32_t inf, int shift, int lane,
                                            int32_t &kfin) {
    while (sp > 0) {
        const int nb = min(min(sp, 32), max(1, SK_STACK - SK_SLACK - sp));
        const bool has = lane < nb;
        const int4 nd = has ? stk[sp - nb + lane] : make_int4(1, 0, 0, -1);
        __syncwarp();
        sp -= nb;
        const int32_t left = nd.x, right = nd.y, top = nd.z, bottom = nd.w;
        const int32_t mid = (left + right + 1) >> 1;
        const bool serial = has && bottom - top < SK_SERIAL;
        Key best = ~(Key)0;
        if (serial) {
#pragma unroll 4
            for (int32_t k = top; k <= bottom; ++k) {
                const Key key = rpack<Key>(cell(k, mid), k, shift);
                best = key < best ? key : best;
            }
        }
        unsigned lm = __ballot_sync(0xffffffffu, has && !serial);
        while (lm) {  // long split ranges: whole warp, one node at a time
            const int src = __ffs(lm) - 1;
            lm &= lm - 1;
            const int32_t t0 = __shfl_sync(0xffffffffu, top, src);
            const int32_t t1 = __shfl_sync(0xffffffffu, bottom, src);
            const int32_t mj = __shfl_sync(0xffffffffu, mid, src);
            Key b2 = ~(Key)0;
            for (int32_t k = t0 + lane; k <= t1; k += 32) {
                const Key key = rpack<Key>(cell(k, mj), k, shift);
                b2 = key < b2 ? key : b2;
            }
            b2 = rwarp_min(b2);
            if (lane == src) best = b2;
        }
        const int32_t bv = rval<Key>(best, shift), bk = rk<Key>(best, shift);
        const bool fin = has && bv != inf;
        if (has) {
            reach[mid] = bv;
            trace[mid] = bk;
        }
        if (fin) kfin = max(kfin, mid);
        // INF node: (mid, right] gets (INF, top); short fills serially
        const bool infn = has && !fin && right > mid;
        const bool longfill = infn && right - mid > SK_SERIAL;
        if (infn && !longfill)
            for (int32_t q = mid + 1; q <= right; ++q) {
                reach[q] = inf;
                trace[q] = top;
            }
        unsigned fm = __ballot_sync(0xffffffffu, longfill);
        while (fm) {
            const int src = __ffs(fm) - 1;
            fm &= fm - 1;
            const int32_t q0 = __shfl_sync(0xffffffffu, mid, src) + 1;
            const int32_t q1 = __shfl_sync(0xffffffffu, right, src);
            const int32_t tt = __shfl_sync(0xffffffffu, top, src);
            for (int32_t q = q0 + lane; q <= q1; q += 32) {
                reach[q] = inf;
                trace[q] = tt;
            }
        }
        // children: finite -> [left, mid-1] (bottom = bk), [mid+1, right]
        // (top = bk); INF -> [left, mid-1] with the node's own split range
        const bool cl = has && mid - 1 >= left;
        const bool cr = fin && right >= mid + 1;
        const int nc = (int)cl + (int)cr;
        int pos = nc;
    #pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, pos, o);
            if (lane >= o) pos += t;
        }
        const int tot = __shfl_sync(0xffffffffu, pos, 31);
        pos = sp + pos - nc;
        if (cr) stk[pos++] = make_int4(mid + 1, right, bk, bottom);
        if (cl) stk[pos] = make_int4(left, mid - 1, top, fin ? bk : bottom);
        sp += tot;
        __syncwarp();
    }
}

template <typename Key>
__global__ void __launch_bounds__(32 * SK_WARPS)
    skeleton_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                    int32_t stride, int32_t nsk) {
    __shared__ int4 front[2][SK_WARPS];
    __shared__ int nfront[2];
    __shared__ Key node_key;
    extern __shared__ int4 stk_all[];  // SK_WARPS x SK_STACK
    __shared__ int kfin_sh;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t di = blockIdx.x / nsk;
    if (di >= ndesc) return;
    const int32_t r = (int32_t)(blockIdx.x - di * nsk);
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t i = (r == nsk - 1) ? n1 - 1 : (int64_t)r * stride;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    // skeleton combines always have materialised (slab) children, and every
    // refined table has n1 * w1 < 2^32 (lcsg_api.cu): plain rows, 32-bit offsets
    const int32_t *__restrict__ Urow = d.U.reach + (uint32_t)i * (uint32_t)d.U.w1;
    const int32_t *__restrict__ Lr = d.L.reach;
    const uint32_t lw1 = (uint32_t)d.L.w1;
    const int32_t w = d.w1 - 1, wl = d.L.w1 - 1;
    const int32_t kmaxU = __ldg(d.U.kmax + i);
    const int32_t colhi = min(w, kmaxU + *d.L.wstar);
    int32_t *reach = d.out_reach + (uint32_t)i * (uint32_t)d.w1;
    int32_t *trace = d.out_trace + (uint32_t)i * (uint32_t)d.w1;
    // cell_value (_kernel.pyx:14-25) of split k at column j
    auto cell = [&](int32_t k, int32_t j) -> int32_t {
        const int32_t x = __ldg(Urow + k);
        if (k > j || x >= inf || j - k > wl) return inf;
        return __ldg(Lr + ((uint32_t)(x - 1) * lw1 + (uint32_t)(j - k)));
    };
    if (threadIdx.x == 0) {
        front[0][0] = make_int4(0, colhi, 0, kmaxU);
        nfront[0] = 1;
        nfront[1] = 0;
        kfin_sh = -1;
    }
    int cur = 0;
    int32_t kfin = -1;
    // --- cooperative rounds (all 256 threads per node) ---
    for (;;) {
        __syncthreads();
        const int nf = nfront[cur];
        if (nf == 0 || nf > SK_WARPS / 2) break;
        __syncthreads();
        if (threadIdx.x == 0) nfront[cur ^ 1] = 0;
        for (int f = 0; f < nf; ++f) {
            const int4 nd = front[cur][f];  // (left, right, top, bottom)
            const int32_t mid = (nd.x + nd.y + 1) >> 1;
            if (threadIdx.x == 0) node_key = ~(Key)0;
            __syncthreads();
            Key best = ~(Key)0;
            for (int32_t k = nd.z + (int32_t)threadIdx.x; k <= nd.w; k += 32 * SK_WARPS) {
                const Key key = rpack<Key>(cell(k, mid), k, shift);
                best = key < best ? key : best;
            }
            best = rwarp_min(best);
            if (lane == 0) smem_min(&node_key, best);
            __syncthreads();
            const Key key = node_key;
            __syncthreads();
            const int32_t bv = rval<Key>(key, shift), bk = rk<Key>(key, shift);
            if (bv == inf) {
                for (int32_t q = mid + 1 + (int32_t)threadIdx.x; q <= nd.y; q += 32 * SK_WARPS) {
                    reach[q] = inf;
                    trace[q] = nd.z;
                }
            }
            if (threadIdx.x == 0) {
                reach[mid] = bv;
                trace[mid] = bk;
                int &nn = nfront[cur ^ 1];
                if (bv != inf) {
                    kfin = max(kfin, mid);
                    if (mid - 1 >= nd.x) front[cur ^ 1][nn++] = make_int4(nd.x, mid - 1, nd.z, bk);
                    if (nd.y >= mid + 1) front[cur ^ 1][nn++] = make_int4(mid + 1, nd.y, bk, nd.w);
                } else if (mid - 1 >= nd.x) {
                    front[cur ^ 1][nn++] = make_int4(nd.x, mid - 1, nd.z, nd.w);
                }
            }
        }
        cur ^= 1;
    }
    // --- one warp per remaining sub-tree: batched DFS (up to 32 nodes a step)
    const int nf = nfront[cur];
    if (wid < nf) {
        int4 *stk = stk_all + wid * SK_STACK;
        int sp = 0;
        if (lane == 0) stk[0] = front[cur][wid];
        sp = 1;
        __syncwarp();
        batched_dfs<Key>(stk, sp, cell, reach, trace, inf, shift, lane, kfin);
    }
    // the batched DFS leaves each lane with the largest finite mid IT visited
    kfin = __reduce_max_sync(0xffffffffu, kfin);
    if (lane == 0 && kfin >= 0) atomicMax(&kfin_sh, kfin);
    for (int32_t q = colhi + 1 + (int32_t)threadIdx.x; q <= w; q += 32 * SK_WARPS) {
        reach[q] = inf;
        trace[q] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        d.out_kmax[i] = kfin_sh;
        atomicMax(d.out_wstar, kfin_sh);
    }
}

// ---------------------------------------------------------------------------
// 2. refinement pass: rows c = (2t+1)*delta from rows a = c-delta, b = c+delta.
// One warp per row, rows fully independent (no CTA barriers): a profile of a
// CTA-synchronised variant showed a quarter of all stall samples parked at the
// barrier behind the slowest row.  U rows are read straight from HBM/L2 with
// the read-only path: consecutive lanes touch consecutive k, so each warp
// load is one or two 128-B lines.  Each lane owns RF_NB columns per step
// (j = j0 + lane + 32q) so several independent gathers are in flight.
// ---------------------------------------------------------------------------
constexpr int RF_SEGS = 40;
constexpr int RF_NB = 4;
constexpr int RF_WARPS = 8;

template <typename Key>
__global__ void __launch_bounds__(32 * RF_WARPS)
    refine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                  int32_t delta, int32_t cnt) {
    __shared__ int4 seg_all[RF_WARPS][RF_SEGS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t gw = blockIdx.x * (int64_t)RF_WARPS + wid;
    const int64_t di = gw / cnt;
    if (di >= ndesc) return;  // warp-uniform
    const int32_t slot = (int32_t)(gw - di * cnt);
    int4 *seg = seg_all[wid];
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t inf = c.inf;
    const CombineDesc &d = descs[di];
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t w = d.w1 - 1, wl = L.w1 - 1;
    const int64_t cr = (2 * (int64_t)slot + 1) * delta;
    const int64_t ar = cr - delta;
    const int64_t br = min(cr + delta, n1 - 1);
    const int32_t db = (int32_t)(br - cr);
    const int32_t kmaxc = tab_kmax(U, cr, inf);
    const int32_t colhi = min(w, kmaxc + *d.L.wstar);
    const int32_t Ka = d.out_kmax[ar], Kb = d.out_kmax[br];
    int32_t *reach = d.out_reach + cr * d.w1;
    int32_t *trace = d.out_trace + cr * d.w1;
    const int32_t *trace_a = d.out_trace + ar * d.w1;
    const int32_t *trace_b = d.out_trace + br * d.w1;
    const int32_t *Ur = U.reach + cr * (int64_t)U.w1;  // U is never a leaf here (w1 > 17)
    const int32_t *Ua = U.reach + ar * (int64_t)U.w1;
    const int32_t *Ub = U.reach + br * (int64_t)U.w1;

    // ---- main cells: (b, j) finite => (c, j) finite, bounded k-range ----
    for (int32_t j0 = 0; j0 <= Kb; j0 += 32 * RF_NB) {
        int32_t Ta[RF_NB], Tb[RF_NB], klo[RF_NB], khi[RF_NB];
#pragma unroll
        for (int q = 0; q < RF_NB; ++q) {
            const int32_t j = j0 + lane + 32 * q;
            Ta[q] = j <= Kb ? __ldg(trace_a + j) : 0;
            Tb[q] = j <= Kb ? __ldg(trace_b + j) : 0;
        }
        int32_t Xa[RF_NB], Xb[RF_NB];
#pragma unroll
        for (int q = 0; q < RF_NB; ++q) {
            Xa[q] = __ldg(Ua + Ta[q]);
            Xb[q] = __ldg(Ub + Tb[q]);
        }
        int32_t maxlen = 0;
#pragma unroll
        for (int q = 0; q < RF_NB; ++q) {
            const int32_t j = j0 + lane + 32 * q;
            // klo = first k with U[c,k] >= X(a,j), in [Ta - delta, Ta]
            int32_t hi = min(Ta[q], kmaxc);
            int32_t lo = min(max(0, Ta[q] - (int32_t)delta), hi);
            while (lo < hi) {
                const int32_t md = (lo + hi) >> 1;
                if (__ldg(Ur + md) >= Xa[q]) hi = md; else lo = md + 1;
            }
            int32_t kl = max(lo, j - wl);
            // khi = last k with U[c,k] <= X(b,j), in [Tb, Tb + (b - c)]
            lo = min(Tb[q], kmaxc);
            hi = min(Tb[q] + db, kmaxc);
            while (lo < hi) {
                const int32_t md = (lo + hi + 1) >> 1;
                if (__ldg(Ur + md) <= Xb[q]) lo = md; else hi = md - 1;
            }
            int32_t kh = min(lo, j);
            if (kl > kh) {  // safety net: never taken when the bounds hold
                kl = max(0, j - wl);
                kh = min(j, kmaxc);
            }
            if (j > Kb) { kl = 1; kh = 0; }
            klo[q] = kl;
            khi[q] = kh;
            maxlen = max(maxlen, kh - kl + 1);
        }
        Key best[RF_NB];
#pragma unroll
        for (int q = 0; q < RF_NB; ++q) best[q] = ~(Key)0;
        for (int32_t t = 0; t < maxlen; ++t) {
#pragma unroll
            for (int q = 0; q < RF_NB; ++q) {
                const int32_t k = klo[q] + t;
                if (k <= khi[q]) {
                    const int32_t j = j0 + lane + 32 * q;
                    const Key key = rpack<Key>(rcell(L, __ldg(Ur + k), k, j, inf, wl), k, shift);
                    best[q] = key < best[q] ? key : best[q];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RF_NB; ++q) {
            const int32_t j = j0 + lane + 32 * q;
            if (j <= Kb) {
                reach[j] = best[q] == ~(Key)0 ? inf : rval<Key>(best[q], shift);
                trace[j] = rk<Key>(best[q], shift);
            }
        }
    }
    // ---- tail: finite in a, INF in b -> lower bound only; whole warp per cell ----
    int32_t K = Kb;
    const int32_t jt_hi = min(min(Ka, Kb + db), colhi);
    for (int32_t j = Kb + 1; j <= jt_hi; ++j) {
        const int32_t Ta = __ldg(trace_a + j);
        const int32_t Xa = __ldg(Ua + Ta);
        int32_t hi = min(Ta, kmaxc);
        int32_t lo = min(max(0, Ta - (int32_t)delta), hi);
        while (lo < hi) {
            const int32_t md = (lo + hi) >> 1;
            if (__ldg(Ur + md) >= Xa) hi = md; else lo = md + 1;
        }
        const int32_t kl = max(lo, j - wl), kh = min(j, kmaxc);
        Key best = ~(Key)0;
        for (int32_t k = kl + lane; k <= kh; k += 32) {
            const Key key = rpack<Key>(rcell(L, __ldg(Ur + k), k, j, inf, wl), k, shift);
            best = key < best ? key : best;
        }
        best = rwarp_min(best);
        const int32_t bv = best == ~(Key)0 ? inf : rval<Key>(best, shift);  // empty range: INF
        if (bv == inf) break;  // finite cells form a prefix
        if (lane == 0) {
            reach[j] = bv;
            trace[j] = rk<Key>(best, shift);
        }
        K = j;
    }
    // ---- replay Alg. 1 over the INF suffix (K, colhi]: trace = `top` of the
    // covering node.  Lane 0 walks the path positions (no loads); the `top`
    // values (traces at finite mids of the path) are then fetched in parallel.
    int ns = 0;
    if (lane == 0) {
        int32_t left = 0, right = colhi, fm = -1;
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            if (mid <= K) {
                fm = mid;
                left = mid + 1;
            } else {
                if (ns < RF_SEGS) seg[ns++] = make_int4(mid, right, fm, 0);
                right = mid - 1;
            }
        }
    }
    ns = __shfl_sync(0xffffffffu, ns, 0);
    __syncwarp();
    for (int s = lane; s < ns; s += 32) {
        const int32_t fm = seg[s].z;
        seg[s].w = fm >= 0 ? trace[fm] : 0;
    }
    __syncwarp();
    for (int32_t q = K + 1 + lane; q <= w; q += 32) {
        int32_t tv = 0;
        if (q <= colhi)
            for (int s = 0; s < ns; ++s) {
                const int4 sg = seg[s];
                if (q >= sg.x && q <= sg.y) { tv = sg.w; break; }
            }
        reach[q] = inf;
        trace[q] = tv;
    }
    if (lane == 0) {
        d.out_kmax[cr] = K;
        atomicMax(d.out_wstar, K);
    }
}

int launch_skeleton(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                    int32_t stride, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t nsk = (int32_t)((n1 - 1 + stride - 1) / stride) + 1;
    const unsigned blocks = (unsigned)(nsk * (int64_t)ndesc);
    const size_t smem = (size_t)SK_WARPS * SK_STACK * sizeof(int4);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(skeleton_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(skeleton_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    {
        // shared-memory carveout: 75% leaves L1 room for the U rows every DFS
        // node re-reads (cfg5 26.85 -> 26.54 ms vs the default split)
        const char *e = getenv("LCSG_SKEL_CARVEOUT");
        const int carve = e ? atoi(e) : 75;
        cudaFuncSetAttribute(skeleton_kernel<uint64_t>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        cudaFuncSetAttribute(skeleton_kernel<uint32_t>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    }
    if (key64)
        skeleton_kernel<uint64_t><<<blocks, 32 * SK_WARPS, smem, s>>>(descs, ndesc, c, shift, stride, nsk);
    else
        skeleton_kernel<uint32_t><<<blocks, 32 * SK_WARPS, smem, s>>>(descs, ndesc, c, shift, stride, nsk);
    LCSG_LAUNCH_CHECK();
    return 0;
}

// Skeleton rows of the narrower wide tables (w1 <= 257): one warp per row,
// the whole Alg. 1 tree by the batched DFS (the per-node chain of
// combine_warp_kernel took ~colhi dependent steps per row).
constexpr int SKW_WARPS = 4;

template <typename Key>
__global__ void __launch_bounds__(32 * SKW_WARPS)
    skeleton_warp_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                         int32_t stride, int32_t nsk) {
    extern __shared__ int4 stkw_all[];  // SKW_WARPS x SK_STACK
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t gw = blockIdx.x * (int64_t)SKW_WARPS + wid;
    const int64_t di = gw / nsk;
    if (di >= ndesc) return;  // warp-uniform
    const int32_t r = (int32_t)(gw - di * nsk);
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t i = (r == nsk - 1) ? n1 - 1 : (int64_t)r * stride;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const int32_t *__restrict__ Urow = d.U.reach + (uint32_t)i * (uint32_t)d.U.w1;
    const int32_t *__restrict__ Lr = d.L.reach;
    const uint32_t lw1 = (uint32_t)d.L.w1;
    const int32_t w = d.w1 - 1, wl = d.L.w1 - 1;
    const int32_t kmaxU = __ldg(d.U.kmax + i);
    const int32_t colhi = min(w, kmaxU + *d.L.wstar);
    int32_t *reach = d.out_reach + (uint32_t)i * (uint32_t)d.w1;
    int32_t *trace = d.out_trace + (uint32_t)i * (uint32_t)d.w1;
    auto cell = [&](int32_t k, int32_t j) -> int32_t {
        const int32_t x = __ldg(Urow + k);
        if (k > j || x >= inf || j - k > wl) return inf;
        return __ldg(Lr + ((uint32_t)(x - 1) * lw1 + (uint32_t)(j - k)));
    };
    int4 *stk = stkw_all + wid * SK_STACK;
    if (lane == 0) stk[0] = make_int4(0, colhi, 0, kmaxU);
    __syncwarp();
    int32_t kfin = -1;
    batched_dfs<Key>(stk, 1, cell, reach, trace, inf, shift, lane, kfin);
    for (int32_t q = colhi + 1 + lane; q <= w; q += 32) {
        reach[q] = inf;
        trace[q] = 0;
    }
    kfin = __reduce_max_sync(0xffffffffu, kfin);
    if (lane == 0) {
        d.out_kmax[i] = kfin;
        atomicMax(d.out_wstar, kfin);
    }
}

int launch_skeleton_warp(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                         int32_t stride, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t nsk = (int32_t)((n1 - 1 + stride - 1) / stride) + 1;
    const int64_t warps = (int64_t)nsk * ndesc;
    const unsigned blocks = (unsigned)((warps + SKW_WARPS - 1) / SKW_WARPS);
    const size_t smem = (size_t)SKW_WARPS * SK_STACK * sizeof(int4);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(skeleton_warp_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(skeleton_warp_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    if (key64)
        skeleton_warp_kernel<uint64_t><<<blocks, 32 * SKW_WARPS, smem, s>>>(descs, ndesc, c, shift, stride, nsk);
    else
        skeleton_warp_kernel<uint32_t><<<blocks, 32 * SKW_WARPS, smem, s>>>(descs, ndesc, c, shift, stride, nsk);
    LCSG_LAUNCH_CHECK();
    return 0;
}

int refine_rows(int64_t n1, int32_t delta) {
    // rows c = delta, 3*delta, ... < n1 - 1
    if (n1 - 1 <= delta) return 0;
    return (int32_t)((n1 - 1 - delta + 2 * (int64_t)delta - 1) / (2 * (int64_t)delta));
}

int launch_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t delta, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t cnt = refine_rows(n1, delta);
    if (cnt <= 0) return 0;
    const int64_t warps = (int64_t)cnt * ndesc;
    const unsigned blocks = (unsigned)((warps + RF_WARPS - 1) / RF_WARPS);
    if (key64)
        refine_kernel<uint64_t><<<blocks, 32 * RF_WARPS, 0, s>>>(descs, ndesc, c, shift, delta, cnt);
    else
        refine_kernel<uint32_t><<<blocks, 32 * RF_WARPS, 0, s>>>(descs, ndesc, c, shift, delta, cnt);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
