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
constexpr int SK_STACK = 34;

template <typename Key>
__global__ void __launch_bounds__(32 * SK_WARPS)
    skeleton_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                    int32_t stride, int32_t nsk) {
    __shared__ int4 front[2][SK_WARPS];
    __shared__ int nfront[2];
    __shared__ Key node_key;
    __shared__ int4 stk_all[SK_WARPS][SK_STACK];
    __shared__ int kfin_sh;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t di = blockIdx.x / nsk;
    if (di >= ndesc) return;
    const int32_t r = (int32_t)(blockIdx.x - di * nsk);
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t i = (r == nsk - 1) ? n1 - 1 : (int64_t)r * stride;
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t w = d.w1 - 1, wl = L.w1 - 1;
    const int32_t kmaxU = tab_kmax(U, i, inf);
    const int32_t colhi = min(w, kmaxU + *d.L.wstar);
    int32_t *reach = d.out_reach + i * d.w1;
    int32_t *trace = d.out_trace + i * d.w1;
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
                const Key key = rpack<Key>(rcell(L, tab_get(U, i, k), k, mid, inf, wl), k, shift);
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
    // --- one warp per remaining sub-tree: DFS as in combine_warp_kernel ---
    const int nf = nfront[cur];
    if (wid < nf) {
        int4 *stk = stk_all[wid];
        int sp = 0;
        int4 nd = front[cur][wid];
        int32_t left = nd.x, right = nd.y, top = nd.z, bottom = nd.w;
        for (;;) {
            while (right >= left) {
                const int32_t mid = (left + right + 1) >> 1;
                Key best = ~(Key)0;
                for (int32_t k = top + lane; k <= bottom; k += 32) {
                    const Key key = rpack<Key>(rcell(L, tab_get(U, i, k), k, mid, inf, wl), k, shift);
                    best = key < best ? key : best;
                }
                best = rwarp_min(best);
                const int32_t bv = rval<Key>(best, shift), bk = rk<Key>(best, shift);
                if (lane == 0) {
                    reach[mid] = bv;
                    trace[mid] = bk;
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
                        trace[q] = top;
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
    }
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
// A CTA of 8 warps holds R = 8 / wpr rows; wpr warps share one row.  Shared
// memory holds the U rows of the R rows and of their R+1 neighbours (row b of
// slot t is row a of slot t+1), so the crossing columns X(a,j) = U[a,T(a,j)],
// X(b,j) and both binary searches are shared-memory only: per column the
// dependent global traffic is the two coalesced trace loads and the L
// gathers.  Each lane handles RF_NB columns at once (independent loads in
// flight) to cover HBM latency.
// ---------------------------------------------------------------------------
constexpr int RF_SEGS = 40;
constexpr int RF_NB = 4;

template <typename Key>
__global__ void __launch_bounds__(256, 2)
    refine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                  int32_t delta, int32_t cnt, int wpr_log2, int32_t ustride) {
    extern __shared__ int32_t sm[];
    __shared__ int32_t g_kfin[8];
    __shared__ int4 g_seg[8][RF_SEGS];
    __shared__ int32_t g_nseg[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wpr = 1 << wpr_log2, R = 8 >> wpr_log2;
    const int grp = warp >> wpr_log2, gw = warp & (wpr - 1);
    const int gt = gw * 32 + lane, gthreads = wpr * 32;
    const int32_t bpd = (cnt + R - 1) / R;
    const int64_t di = blockIdx.x / bpd;
    const int32_t slot0 = (int32_t)(blockIdx.x - di * bpd) * R;
    const int32_t slot = slot0 + grp;
    const bool active = di < ndesc && slot < cnt;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t inf = c.inf;
    int32_t *Uc = sm + grp * ustride;
    const int32_t *Ua = sm + (R + grp) * ustride;
    const int32_t *Ub = sm + (R + grp + 1) * ustride;

    const CombineDesc &d = descs[di < ndesc ? di : 0];
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t w = d.w1 - 1, wl = L.w1 - 1;
    const int64_t cr = (2 * (int64_t)slot + 1) * delta;
    const int64_t ar = cr - delta;
    const int64_t br = min(cr + delta, n1 - 1);
    const int32_t db = (int32_t)(br - cr);
    int32_t kmaxc = 0, colhi = 0, Ka = 0, Kb = 0;
    int32_t *reach = nullptr, *trace = nullptr;
    const int32_t *trace_a = nullptr, *trace_b = nullptr;
    // ---- stage U rows: own row, neighbour a (= slot's even row), and b for the last group ----
    if (di < ndesc && slot0 + grp <= cnt) {
        const int64_t nb = min(2 * (int64_t)slot * delta, n1 - 1);
        int32_t *Un = sm + (R + grp) * ustride;
        const int32_t kn = tab_kmax(U, nb, inf);
        for (int32_t k = gt; k <= kn; k += gthreads) Un[k] = tab_get(U, nb, k);
        if (grp == R - 1) {
            const int64_t nb2 = min(2 * (int64_t)(slot + 1) * delta, n1 - 1);
            int32_t *Un2 = sm + (R + grp + 1) * ustride;
            const int32_t kn2 = tab_kmax(U, nb2, inf);
            for (int32_t k = gt; k <= kn2; k += gthreads) Un2[k] = tab_get(U, nb2, k);
        }
    }
    if (active) {
        kmaxc = tab_kmax(U, cr, inf);
        colhi = min(w, kmaxc + *d.L.wstar);
        Ka = d.out_kmax[ar];
        Kb = d.out_kmax[br];
        reach = d.out_reach + cr * d.w1;
        trace = d.out_trace + cr * d.w1;
        trace_a = d.out_trace + ar * d.w1;
        trace_b = d.out_trace + br * d.w1;
        for (int32_t k = gt; k <= kmaxc; k += gthreads) Uc[k] = tab_get(U, cr, k);
        if (gt == 0) g_kfin[grp] = Kb;
    }
    __syncthreads();
    if (active) {
        // ---- main cells: (b, j) finite => (c, j) finite, bounded k-range ----
        for (int32_t j0 = gt; j0 <= Kb; j0 += gthreads * RF_NB) {
            int32_t Ta[RF_NB], Tb[RF_NB], klo[RF_NB], khi[RF_NB];
#pragma unroll
            for (int q = 0; q < RF_NB; ++q) {
                const int32_t j = j0 + q * gthreads;
                Ta[q] = j <= Kb ? __ldg(trace_a + j) : 0;
                Tb[q] = j <= Kb ? __ldg(trace_b + j) : 0;
            }
            int32_t maxlen = 0;
#pragma unroll
            for (int q = 0; q < RF_NB; ++q) {
                const int32_t j = j0 + q * gthreads;
                const int32_t Xa = Ua[Ta[q]], Xb = Ub[Tb[q]];
                int32_t hi = min(Ta[q], kmaxc);
                int32_t lo = min(max(0, Ta[q] - (int32_t)delta), hi);
                while (lo < hi) {  // first k with Uc[k] >= Xa
                    const int32_t md = (lo + hi) >> 1;
                    if (Uc[md] >= Xa) hi = md; else lo = md + 1;
                }
                int32_t kl = max(lo, j - wl);
                lo = min(Tb[q], kmaxc);
                hi = min(Tb[q] + db, kmaxc);
                while (lo < hi) {  // last k with Uc[k] <= Xb
                    const int32_t md = (lo + hi + 1) >> 1;
                    if (Uc[md] <= Xb) lo = md; else hi = md - 1;
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
                        const int32_t j = j0 + q * gthreads;
                        const Key key = rpack<Key>(rcell(L, Uc[k], k, j, inf, wl), k, shift);
                        best[q] = key < best[q] ? key : best[q];
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < RF_NB; ++q) {
                const int32_t j = j0 + q * gthreads;
                if (j <= Kb) {
                    reach[j] = rval<Key>(best[q], shift);
                    trace[j] = rk<Key>(best[q], shift);
                }
            }
        }
        // ---- tail: finite in a, INF in b -> lower bound only; one warp per cell ----
        const int32_t jt_hi = min(min(Ka, Kb + db), colhi);
        for (int32_t j = Kb + 1 + gw; j <= jt_hi; j += wpr) {
            const int32_t Ta = __ldg(trace_a + j);
            const int32_t Xa = Ua[Ta];
            int32_t hi = min(Ta, kmaxc);
            int32_t lo = min(max(0, Ta - (int32_t)delta), hi);
            while (lo < hi) {
                const int32_t md = (lo + hi) >> 1;
                if (Uc[md] >= Xa) hi = md; else lo = md + 1;
            }
            const int32_t kl = max(lo, j - wl), kh = min(j, kmaxc);
            Key best = ~(Key)0;
            for (int32_t k = kl + lane; k <= kh; k += 32) {
                const Key key = rpack<Key>(rcell(L, Uc[k], k, j, inf, wl), k, shift);
                best = key < best ? key : best;
            }
            best = rwarp_min(best);
            const int32_t bv = rval<Key>(best, shift);
            if (lane == 0 && bv != inf) {
                reach[j] = bv;
                trace[j] = rk<Key>(best, shift);
                atomicMax(&g_kfin[grp], j);
            }
        }
    }
    __syncthreads();
    // ---- replay Alg. 1 over the INF suffix: trace = `top` of the covering node ----
    if (active && gt == 0) {
        const int32_t K = g_kfin[grp];
        int32_t left = 0, right = colhi, top = 0, ns = 0;
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            if (mid <= K) {
                top = trace[mid];
                left = mid + 1;
            } else {
                if (ns < RF_SEGS) g_seg[grp][ns++] = make_int4(mid, right, top, 0);
                right = mid - 1;
            }
        }
        g_nseg[grp] = ns;
    }
    __syncthreads();
    if (active) {
        const int32_t K = g_kfin[grp];
        const int ns = g_nseg[grp];
        for (int32_t q = K + 1 + gt; q <= w; q += gthreads) {
            int32_t tv = 0;
            if (q <= colhi)
                for (int s = 0; s < ns; ++s) {
                    const int4 sg = g_seg[grp][s];
                    if (q >= sg.x && q <= sg.y) { tv = sg.z; break; }
                }
            reach[q] = inf;
            trace[q] = tv;
        }
        if (gt == 0) {
            d.out_kmax[cr] = K;
            atomicMax(d.out_wstar, K);
        }
    }
}

int launch_skeleton(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                    int32_t stride, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t nsk = (int32_t)((n1 - 1 + stride - 1) / stride) + 1;
    const unsigned blocks = (unsigned)(nsk * (int64_t)ndesc);
    if (key64)
        skeleton_kernel<uint64_t><<<blocks, 32 * SK_WARPS, 0, s>>>(descs, ndesc, c, shift, stride, nsk);
    else
        skeleton_kernel<uint32_t><<<blocks, 32 * SK_WARPS, 0, s>>>(descs, ndesc, c, shift, stride, nsk);
    LCSG_LAUNCH_CHECK();
    return 0;
}

int refine_rows(int64_t n1, int32_t delta) {
    // rows c = delta, 3*delta, ... < n1 - 1
    if (n1 - 1 <= delta) return 0;
    return (int32_t)((n1 - 1 - delta + 2 * (int64_t)delta - 1) / (2 * (int64_t)delta));
}

int launch_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                  int32_t delta, int wpr_log2, int32_t ustride, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int32_t cnt = refine_rows(n1, delta);
    if (cnt <= 0) return 0;
    const int R = 8 >> wpr_log2;
    const int64_t bpd = (cnt + R - 1) / R;
    const unsigned blocks = (unsigned)(bpd * ndesc);
    const size_t smem = (size_t)(2 * R + 1) * ustride * 4;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(refine_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(refine_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr_set = true;
    }
    if (key64)
        refine_kernel<uint64_t><<<blocks, 256, smem, s>>>(descs, ndesc, c, shift, delta, cnt, wpr_log2, ustride);
    else
        refine_kernel<uint32_t><<<blocks, 256, smem, s>>>(descs, ndesc, c, shift, delta, cnt, wpr_log2, ustride);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
