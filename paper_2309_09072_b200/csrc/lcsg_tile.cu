// lcsg_tile.cu -- tiled refinement of the wide combines (the fast path).
//
// After the skeleton rows i = 0, S, 2S, ..., n of a combine are known (exact
// Alg. 1, lcsg_refine.cu), every interior row is derived by refinement:
// X(c,j) = U[c, k*(c,j)] is monotone in the start row c (Monge argmin), so
// k*(c,j) lies between bounds read off rows c-delta and c+delta AT THE SAME
// COLUMN j.  Column tiles are therefore independent: one CTA owns a block of
// S+1 consecutive rows (two skeleton rows bracketing S-1 interior rows) times
// TJ columns, keeps the block's (reach, trace) in shared memory, stages the
// window of U rows the block can touch once, and runs all log2(S) refinement
// passes with only the L gathers going to L2/HBM.  Finite cells are written
// once, coalesced; the per-row finalize kernel then writes the INF suffix
// (replaying Alg. 1 for the reference's INF-cell traces) and kmax / wstar.
//
// Cells finite in row a but INF in row b (at most 2*delta per row and pass)
// have no upper bound; they are queued and scanned warp-cooperatively over
// [lower bound, min(j, kmax_c)].
#include <climits>

#include "lcsg_internal.cuh"

namespace lcsg {

#define LCSG_LAUNCH_CHECK()                         \
    do {                                            \
        cudaError_t e__ = cudaGetLastError();       \
        if (e__ != cudaSuccess) return (int)e__;    \
    } while (0)

constexpr int BT_THREADS = 256;
constexpr int BT_MAXS = 64;
constexpr int BT_TAILCAP = 512;
constexpr int FN_SEGS = 40;
constexpr int FN_WARPS = 8;

template <typename Key>
__device__ __forceinline__ Key tpack(int32_t v, int32_t k, int shift) {
    return ((Key)(uint32_t)v << shift) | (Key)(uint32_t)k;
}
template <typename Key>
__device__ __forceinline__ int32_t tval(Key key, int shift) { return (int32_t)(key >> shift); }
template <typename Key>
__device__ __forceinline__ int32_t tk(Key key, int shift) {
    return (int32_t)(key & (((Key)1 << shift) - 1));
}
__device__ __forceinline__ uint32_t twarp_min(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t twarp_min(uint64_t v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
        v = o < v ? o : v;
    }
    return v;
}

// cell_value (_kernel.pyx:14-25) with x = U[i,k] already loaded.
__device__ __forceinline__ int32_t tcell(const TabAcc &L, int32_t x, int32_t k, int32_t j,
                                         int32_t inf, int32_t wl) {
    if (k > j || x >= inf || j - k > wl) return inf;
    return tab_get(L, (int64_t)x - 1, j - k);
}

struct TileGeo {
    int32_t S;      // rows per block (power of two, <= BT_MAXS)
    int32_t TJ;     // columns per tile
    int32_t WK;     // staged U-window width (k entries per row)
    int32_t nblk;   // row blocks per combine
    int32_t ntile;  // column tiles per combine
};

template <typename Key>
__global__ void __launch_bounds__(BT_THREADS)
    block_refine_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int shift,
                        TileGeo g) {
    extern __shared__ int32_t smem[];
    __shared__ int32_t s_kwlo;
    __shared__ int32_t s_kmaxc[BT_MAXS + 1];
    __shared__ int32_t s_rowmax[BT_MAXS + 1];
    __shared__ int32_t s_ntail[2];
    __shared__ int2 s_tail[BT_TAILCAP];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int64_t per_desc = (int64_t)g.nblk * g.ntile;
    const int64_t di = blockIdx.x / per_desc;
    if (di >= ndesc) return;
    const int64_t rem = blockIdx.x - di * per_desc;
    const int32_t blk = (int32_t)(rem / g.ntile), tile = (int32_t)(rem - (int64_t)blk * g.ntile);
    const CombineDesc &d = descs[di];
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t i0 = (int64_t)blk * g.S;
    const int32_t rb = (int32_t)min((int64_t)g.S, n1 - 1 - i0);  // local index of the bottom skeleton row
    const int32_t w1 = d.w1;
    const int32_t j0 = tile * g.TJ;
    if (j0 >= w1 || rb <= 1) return;  // block-uniform: nothing interior here
    const int32_t tw = min(g.TJ, w1 - j0);
    const int32_t TJ = g.TJ, WK = g.WK;
    int32_t *tR = smem;
    int32_t *tT = tR + (g.S + 1) * TJ;
    int32_t *Uw = tT + (g.S + 1) * TJ;
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c), L = resolve(d.L, c);
    const int32_t wl = L.w1 - 1;

    // 1. the two skeleton rows of the block, per-row kmax of U
    for (int e = tid; e < 2 * tw; e += BT_THREADS) {
        const int32_t r = e < tw ? 0 : rb, jj = e < tw ? e : e - tw;
        const int64_t off = (i0 + r) * w1 + j0 + jj;
        tR[r * TJ + jj] = __ldg(d.out_reach + off);
        tT[r * TJ + jj] = __ldg(d.out_trace + off);
    }
    for (int r = tid; r <= rb; r += BT_THREADS) {
        s_kmaxc[r] = tab_kmax(U, i0 + r, inf);
        s_rowmax[r] = -1;
    }
    if (tid == 0) {
        s_kwlo = INT_MAX;
        s_ntail[0] = s_ntail[1] = 0;
    }
    __syncthreads();
    // 2. U window: k >= min_j T(top skeleton, j) - S covers every bound of the block
    int32_t m = INT_MAX;
    for (int jj = tid; jj < tw; jj += BT_THREADS)
        if (tR[jj] < inf) m = min(m, tT[jj]);
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m != INT_MAX) atomicMin(&s_kwlo, m);
    __syncthreads();
    if (s_kwlo == INT_MAX) return;  // top row INF on the whole tile => every row is
    const int32_t kwlo = max(0, s_kwlo - g.S);
    for (int e = tid; e < (rb + 1) * WK; e += BT_THREADS) {
        const int32_t r = e / WK, kk = e - r * WK;
        const int32_t k = kwlo + kk;
        if (k <= s_kmaxc[r]) Uw[e] = tab_get(U, i0 + r, k);
    }
    __syncthreads();
    auto uget = [&](int32_t r, int32_t k) -> int32_t {
        const int32_t kk = k - kwlo;
        if ((unsigned)kk < (unsigned)WK) return Uw[r * WK + kk];
        return tab_get(U, i0 + r, k);
    };

    // 3. refinement passes, all in shared memory
    int pass = 0;
    for (int32_t dl = g.S >> 1; dl >= 1; dl >>= 1, ++pass) {
        if (rb <= dl) continue;  // block-uniform
        const int32_t nr = (rb - dl + 2 * dl - 1) / (2 * dl);
        const int32_t total = nr * tw;
        int32_t *ntail = &s_ntail[pass & 1];
        if (tid == 0) s_ntail[(pass + 1) & 1] = 0;
        for (int32_t e = tid; e < total; e += BT_THREADS) {
            const int32_t t = e / tw, jj = e - t * tw;
            const int32_t r = dl * (2 * t + 1), a = r - dl, b = min(r + dl, rb);
            const int32_t j = j0 + jj;
            if (tR[a * TJ + jj] >= inf) {  // (a, j) INF => (c, j) INF
                tR[r * TJ + jj] = inf;
                continue;
            }
            if (tR[b * TJ + jj] >= inf) {  // no upper bound: queue for the warps
                const int q = atomicAdd(ntail, 1);
                if (q < BT_TAILCAP) {
                    s_tail[q] = make_int2(r, jj);
                    continue;
                }
            }
            const int32_t kmc = s_kmaxc[r];
            const int32_t Ta = tT[a * TJ + jj];
            const int32_t Xa = uget(a, Ta);
            int32_t hi = min(Ta, kmc);
            int32_t lo = min(max(0, Ta - dl), hi);
            while (lo < hi) {  // first k with U[c,k] >= X(a,j)
                const int32_t md = (lo + hi) >> 1;
                if (uget(r, md) >= Xa) hi = md; else lo = md + 1;
            }
            int32_t kl = max(lo, j - wl), kh;
            if (tR[b * TJ + jj] < inf) {
                const int32_t Tb = tT[b * TJ + jj];
                const int32_t Xb = uget(b, Tb);
                lo = min(Tb, kmc);
                hi = min(Tb + (b - r), kmc);
                while (lo < hi) {  // last k with U[c,k] <= X(b,j)
                    const int32_t md = (lo + hi + 1) >> 1;
                    if (uget(r, md) <= Xb) lo = md; else hi = md - 1;
                }
                kh = min(lo, j);
                if (kl > kh) {  // safety net: never taken when the bounds hold
                    kl = max(0, j - wl);
                    kh = min(j, kmc);
                }
            } else {
                kh = min(j, kmc);  // tail cell, queue overflowed
            }
            Key best = ~(Key)0;
            for (int32_t k = kl; k <= kh; ++k) {
                const Key key = tpack<Key>(tcell(L, uget(r, k), k, j, inf, wl), k, shift);
                best = key < best ? key : best;
            }
            tR[r * TJ + jj] = tval<Key>(best, shift);
            tT[r * TJ + jj] = tk<Key>(best, shift);
        }
        __syncthreads();
        const int32_t nt = min(*ntail, BT_TAILCAP);
        for (int32_t q = wid; q < nt; q += BT_THREADS / 32) {
            const int2 tc = s_tail[q];
            const int32_t r = tc.x, jj = tc.y, a = r - dl, j = j0 + jj;
            const int32_t kmc = s_kmaxc[r];
            const int32_t Ta = tT[a * TJ + jj];
            const int32_t Xa = uget(a, Ta);
            int32_t hi = min(Ta, kmc);
            int32_t lo = min(max(0, Ta - dl), hi);
            while (lo < hi) {
                const int32_t md = (lo + hi) >> 1;
                if (uget(r, md) >= Xa) hi = md; else lo = md + 1;
            }
            const int32_t kl = max(lo, j - wl), kh = min(j, kmc);
            Key best = ~(Key)0;
            for (int32_t k = kl + lane; k <= kh; k += 32) {
                const Key key = tpack<Key>(tcell(L, uget(r, k), k, j, inf, wl), k, shift);
                best = key < best ? key : best;
            }
            best = twarp_min(best);
            if (lane == 0) {
                tR[r * TJ + jj] = tval<Key>(best, shift);
                tT[r * TJ + jj] = tk<Key>(best, shift);
            }
        }
        __syncthreads();
    }
    // 4. write the finite cells of the interior rows; per-row max finite column
    for (int32_t e = tid; e < (rb - 1) * tw; e += BT_THREADS) {
        const int32_t r = 1 + e / tw, jj = e - (r - 1) * tw;
        const int32_t v = tR[r * TJ + jj];
        if (v < inf) {
            const int64_t off = (i0 + r) * w1 + j0 + jj;
            d.out_reach[off] = v;
            d.out_trace[off] = tT[r * TJ + jj];
            atomicMax(&s_rowmax[r], j0 + jj);
        }
    }
    __syncthreads();
    for (int r = 1 + tid; r < rb; r += BT_THREADS)
        if (s_rowmax[r] >= 0) atomicMax(d.out_kmax + i0 + r, s_rowmax[r]);
}

// Per interior row: kmax is final (max over tiles); write the INF suffix
// (K, w] -- reach INF, trace = `top` of the Alg. 1 node covering the column
// (replay of the reference bisection, _kernel.pyx:53-60) or 0 beyond colhi
// (_kernel.pyx:79-82) -- and fold kmax into wstar.
__global__ void __launch_bounds__(32 * FN_WARPS)
    finalize_rows_kernel(const CombineDesc *__restrict__ descs, int32_t ndesc, Ctx c, int32_t S) {
    __shared__ int4 seg_all[FN_WARPS][FN_SEGS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t gw = blockIdx.x * (int64_t)FN_WARPS + wid;
    const int64_t di = gw / n1;
    if (di >= ndesc) return;
    const int64_t i = gw - di * n1;
    if (i % S == 0 || i == n1 - 1) return;  // skeleton rows are complete
    int4 *seg = seg_all[wid];
    const CombineDesc &d = descs[di];
    const int32_t inf = c.inf;
    const TabAcc U = resolve(d.U, c);
    const int32_t w = d.w1 - 1;
    const int32_t colhi = min(w, tab_kmax(U, i, inf) + *d.L.wstar);
    const int32_t K = d.out_kmax[i];
    int32_t *reach = d.out_reach + i * d.w1;
    int32_t *trace = d.out_trace + i * d.w1;
    int ns = 0;
    if (lane == 0) {
        int32_t left = 0, right = colhi, fm = -1;
        while (right >= left) {
            const int32_t mid = (left + right + 1) >> 1;
            if (mid <= K) {
                fm = mid;
                left = mid + 1;
            } else {
                if (ns < FN_SEGS) seg[ns++] = make_int4(mid, right, fm, 0);
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
    if (lane == 0) atomicMax(d.out_wstar, K);
}

int launch_block_refine(const CombineDesc *descs, int32_t ndesc, Ctx c, int shift, bool key64,
                        int32_t S, int32_t TJ, int32_t WK, int32_t maxw1, cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    if (S < 2 || S > BT_MAXS) return (int)cudaErrorInvalidValue;
    TileGeo g;
    g.S = S;
    g.TJ = TJ;
    g.WK = WK;
    g.nblk = (int32_t)((n1 - 1 + S - 1) / S);
    g.ntile = (maxw1 + TJ - 1) / TJ;
    if (g.nblk <= 0) return 0;
    const size_t smem = (size_t)(S + 1) * (2 * TJ + WK) * 4;
    const unsigned blocks = (unsigned)((int64_t)g.nblk * g.ntile * ndesc);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(block_refine_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(block_refine_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    if (key64)
        block_refine_kernel<uint64_t><<<blocks, BT_THREADS, smem, s>>>(descs, ndesc, c, shift, g);
    else
        block_refine_kernel<uint32_t><<<blocks, BT_THREADS, smem, s>>>(descs, ndesc, c, shift, g);
    LCSG_LAUNCH_CHECK();
    return 0;
}

int launch_finalize_rows(const CombineDesc *descs, int32_t ndesc, Ctx c, int32_t S,
                         cudaStream_t s) {
    if (ndesc <= 0) return 0;
    const int64_t n1 = (int64_t)c.n + 1;
    const int64_t warps = n1 * ndesc;
    const unsigned blocks = (unsigned)((warps + FN_WARPS - 1) / FN_WARPS);
    finalize_rows_kernel<<<blocks, 32 * FN_WARPS, 0, s>>>(descs, ndesc, c, S);
    LCSG_LAUNCH_CHECK();
    return 0;
}

}  // namespace lcsg
